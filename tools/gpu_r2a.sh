cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_bench.py -m gpu -q -x --durations=20 > gpurun_out/pytest_cfg.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_cfg.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench_default.log
timeout 300 python bench.py --workload c1 --steps 50 --warmup 5 --no-cpu-baseline --no-other-dtype --dtype f32 > gpurun_out/c1_f32.log 2>&1; echo c1 rc=$?
tail -c 1500 gpurun_out/c1_f32.log
