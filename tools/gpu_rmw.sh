set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 120 tools/build/rmw_probe 138000000 0.0109 > gpurun_out/rmw.log 2>&1; cat gpurun_out/rmw.log
timeout 120 tools/build/rmw_probe 1500000000 0.1 >> gpurun_out/rmw.log 2>&1; tail -8 gpurun_out/rmw.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log
timeout 600 python bench.py --workload c1 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c1.log
