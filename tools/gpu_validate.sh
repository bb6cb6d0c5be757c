cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/val
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/val/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/val/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/val/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/val/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/val/bench.log > gpurun_out/val/bench.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/val/ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/val/ref.log > gpurun_out/val/ref.json
