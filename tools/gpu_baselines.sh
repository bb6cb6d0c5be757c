# The comparison sparsifiers vs MiCRO, measured (the paper's Table 1 comparison).
cd $GRAFT_REPO_ROOT
for k in micro topk hard dense; do
  timeout 600 python bench.py --sparsifier $k --steps 30 --warmup 3 --prime 200 --no-cpu-baseline >> gpurun_out/baselines.jsonl 2> gpurun_out/bl_$k.err
  echo "c3 $k rc=$?"
done
for k in micro topk cltk hard; do
  timeout 600 python bench.py --workload c1 --cluster-workers 8 --sparsifier $k --steps 30 --warmup 3 --prime 200 --no-cpu-baseline >> gpurun_out/baselines.jsonl 2> gpurun_out/bl8_$k.err
  echo "c1x8 $k rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/baselines.jsonl"):
    d = json.loads(l); c = d["config"]
    print(c["workload"][:12], c.get("parallelism")[:14], c["sparsifier"], round(d["value"], 1), "us/iter density", round(d["density"] * 100, 4), "%")
PY
