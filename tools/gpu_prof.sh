# GPU call: parity tests, the default bench line, the launch list and one
# full ncu capture of K1 (tools/, run under gpurun; outputs in gpurun_out/).
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log
P="python bench.py --steps 5 --warmup 3 --prime 20 --no-cpu-baseline ${PROF_ARGS}"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 300 $P > gpurun_out/prof_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_fused -s 10 -c 1 -o gpurun_out/k1_full $P > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
