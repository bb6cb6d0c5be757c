cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_baselines.py -x -q > gpurun_out/pytest_bl.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_bl.log
rm -f gpurun_out/baselines.jsonl
for k in topk dense; do
  timeout 600 python bench.py --sparsifier $k --steps 30 --warmup 3 --prime 200 --no-cpu-baseline >> gpurun_out/baselines.jsonl 2> gpurun_out/bl_$k.err
  echo "c3 $k rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/baselines.jsonl"):
    d = json.loads(l); c = d["config"]
    print(c["workload"][:12], c["sparsifier"], round(d["value"], 1), "us/iter density", round(d["density"] * 100, 4), "%")
PY
