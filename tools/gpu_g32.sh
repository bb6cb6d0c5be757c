# GPU call: fp32 gradients into the fp64 engine — parity (small + at size), then the default bench line
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp32_gradients or f64_matches" > gpurun_out/pytest_g32.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_g32.log
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "fp32_gradients" > gpurun_out/pytest_g32c.log 2>&1; echo pytest configs rc=$?; tail -2 gpurun_out/pytest_g32c.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_g32.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_g32.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref_g32.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/ref_g32.log
