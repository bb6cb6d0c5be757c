# GPU call: smoke, the whole -m gpu suite, the default bench line
set -x
nvidia-smi -L
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench.log
