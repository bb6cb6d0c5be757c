# GPU call: the whole -m gpu suite (+ smoke), log under gpurun_out/
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x --durations=25 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_gpu.log
