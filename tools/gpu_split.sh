cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for sp in 2 1; do
  for w in c3 c1 c5_d1 c4; do
    MICRO_SPLIT=$sp timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --prime 300 --no-cpu-baseline | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('split=$sp', d['config']['workload'][:14], round(d['value'],1), round(d['roofline']['avg_launch_ms']*1000,1))"
  done
done
