cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for v in "" "--dense" "--dense --no-model" "--no-model"; do
  timeout 300 python bench.py --steps 60 --no-cpu-baseline $v > gpurun_out/bv.log 2>&1
  tail -1 gpurun_out/bv.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', 'us/iter', round(j['value'],1), 'K1 us', round(j['roofline']['avg_launch_ms']*1e3,1), 'frac', round(j['roofline']['frac'],3), 'density', round(j['density'],5))"
done
P="python bench.py --steps 5 --warmup 3 --prime 400 --no-cpu-baseline"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1610 -c 40 --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_|k_finalize" -s 1203 -c 3 -o gpurun_out/k1_full $P > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
