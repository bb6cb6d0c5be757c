"""Markdown tables for profiles/README.md from a workloads.jsonl of bench lines."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/workloads.jsonl") if l.startswith("{")]
print("| workload | workers | sparsifier | µs/iter | density | K1a µs | K1a frac | step frac | e2e µs |")
print("|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    rf = d["roofline"]
    w = c.get("workers", 1)
    e2e = d["e2e"]["value"] if d.get("e2e") else None
    print(f"| {c['workload'].split(' (')[0]} | {w} | {c.get('sparsifier', 'micro')} | {d['value']:.1f} | "
          f"{d['density'] * 100:.3f} % | {rf['avg_launch_ms'] * 1000:.1f} | {rf['frac']:.2f} | {rf['step_frac']:.2f} | "
          f"{e2e:.0f} |" if e2e else "| — |")
