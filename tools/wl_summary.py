"""One line per bench JSON line: workload, dtype, dense, µs/iter, K1a frac, step frac (+ the other dtype)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        try:
            d = json.loads(line)
        except ValueError:
            continue
        c, r, o = d["config"], d["roofline"], d.get("other_dtype") or {}
        orf = o.get("roofline", {})
        print(f"{c['workload'][:34]:34s} W={c.get('workers')} {d['dtype']} dense={int(c.get('dense_g_over_n', 0))} "
              f"{d['value']:9.1f} us  K1a {r['avg_launch_ms'] * 1e3:8.1f} us frac {r['frac']:.3f} step {r['step_frac']:.3f}"
              + (f" | {o['dtype']} {o['value']:9.1f} us K1a {orf['avg_launch_ms'] * 1e3:8.1f} frac {orf['frac']:.3f} "
                 f"step {orf['step_frac']:.3f}" if o else ""))
