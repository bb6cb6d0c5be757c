"""Markdown tables for profiles/README.md from a workloads.jsonl of bench lines."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/workloads.jsonl")
        if l.startswith("{")]
print("| workload | workers | sparsifier | dtype (gradient) | dense g/n | µs/iter | density | K1a µs | K1a frac | step frac | "
      "f64 on f64 gradients µs/iter (K1a frac, step frac) | f32 µs/iter (K1a frac, step frac) | e2e µs |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    rf = d["roofline"]
    w = c.get("workers", 1)
    e2e = d["e2e"]["value"] if d.get("e2e") else None
    o = d.get("other_dtype")
    ot = (f"{o['dtype']}: {o['value']:.1f} ({o['roofline']['frac']:.2f}, {o['roofline']['step_frac']:.2f})"
          if o else "—")
    g = d.get("other_gradient")
    gt = f"{g['value']:.1f} ({g['roofline']['frac']:.2f}, {g['roofline']['step_frac']:.2f})" if g else "—"
    grad = "f32" if "f32 gradients" in d.get("data", "") else "f64"
    name = c["workload"].split(" (")[0].replace("C3 per-GPU slice (n=1): ", "")
    print(f"| {name} | {w} | {c.get('sparsifier', 'micro')} | {d['dtype']} ({grad}) | "
          f"{'yes' if c.get('dense_g_over_n') else 'no'} | "
          f"{d['value']:.1f} | {d['density'] * 100:.3f} % | {rf['avg_launch_ms'] * 1000:.1f} | {rf['frac']:.2f} | "
          f"{rf['step_frac']:.2f} | {gt} | {ot} | " + (f"{e2e:.0f} |" if e2e else "— |"))
