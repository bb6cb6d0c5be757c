# GPU call: the whole -m gpu suite, then C1 / C3 / C5 d=0.1 bench lines (k1_stream changes)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
run() { timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/wl.log >> gpurun_out/k1_wl.jsonl; }
rm -f gpurun_out/k1_wl.jsonl
run --workload c1 --steps 200
run --workload c1 --steps 200 --no-dense
run --workload c3 --steps 100
run --workload c3 --steps 100 --no-dense
run --workload c5_d1 --steps 20 --warmup 3
