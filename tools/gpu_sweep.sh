# K1 configuration sweep: parity subset + short bench per MICRO_K1_CFG.
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-0 1 2 3 4}; do
  MICRO_K1_CFG=$c timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "matches_restatement and tma" > gpurun_out/sweep_test_$c.log 2>&1
  echo "cfg $c tests rc=$? $(tail -1 gpurun_out/sweep_test_$c.log)"
  MICRO_K1_CFG=$c timeout 300 python bench.py --steps 40 --warmup 5 --prime 600 --no-cpu-baseline > gpurun_out/sweep_bench_$c.log 2>&1
  echo "cfg $c bench rc=$?"
  tail -1 gpurun_out/sweep_bench_$c.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('cfg', $c, 'us/iter', round(j['value'],1), 'K1 us', round(j['roofline']['avg_launch_ms']*1e3,1), 'frac', round(j['roofline']['frac'],3))"
done
