# compute-sanitizer over small parity / baseline / value-API cases (bugs, not timing)
cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
S="/usr/local/cuda/bin/compute-sanitizer --error-exitcode 99 --print-limit 20"
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "stream and (10000-1 or 10007-2 or 4095-1 or 5-5)" > gpurun_out/san_mem_parity.log 2>&1; echo memcheck parity rc=$?
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_baselines.py -q -x -k "f32 and (10000 or 8192)" > gpurun_out/san_mem_bl.log 2>&1; echo memcheck baselines rc=$?
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_sparsim.py -q -x -k "topk or error_metric or select_examples" > gpurun_out/san_mem_sp.log 2>&1; echo memcheck sparsim rc=$?
timeout 1500 $S --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "stream and (10007-2 or 65537-4)" > gpurun_out/san_race.log 2>&1; echo racecheck rc=$?
timeout 1500 $S --tool racecheck python -m pytest tests/test_gpu_baselines.py -q -x -k "f32 and 8192 and topk" > gpurun_out/san_race_bl.log 2>&1; echo racecheck baselines rc=$?
timeout 1500 $S --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "stream and 10007-2" > gpurun_out/san_sync.log 2>&1; echo synccheck rc=$?
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|Invalid|Race|Hazard" $f | head -5; done
