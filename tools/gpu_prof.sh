# GPU call: parity tests, the default bench line (with the CPU reference), the
# launch list and one full ncu capture of the per-step kernels
# (run under gpurun; outputs in gpurun_out/).
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log
# profiling command: converged threshold (prime), then a few timed steps
P="python bench.py --steps 5 --warmup 3 --prime 400 --no-cpu-baseline ${PROF_ARGS}"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1190 -c 40 --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_stream|k1_gather|k_finalize" -s 806 -c 4 -o gpurun_out/k1_full $P > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
