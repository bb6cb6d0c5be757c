cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/val
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/val/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/val/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/val/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/val/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/val/bench.log > gpurun_out/val/bench.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/val/ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/val/ref.log > gpurun_out/val/ref.json
if [ -n "$WORKLOADS" ]; then
  rm -f gpurun_out/val/workloads.jsonl
  run() { timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/val/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/val/wl.log >> gpurun_out/val/workloads.jsonl; }
  run --workload c5_d1 --steps 20 --warmup 3
  run --workload c1 --steps 200
  for k in topk cltk hard; do run --workload c1 --cluster-workers 8 --sparsifier $k --steps 30 --prime 200 --dtype f32 --no-dense; done
  for k in topk hard; do run --workload c3 --sparsifier $k --steps 20 --prime 200 --dtype f32 --no-dense; done
fi
