cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for pdl in 1 0; do
  for w in c1 c3; do
    MICRO_PDL=$pdl timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --prime 500 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['config']['workload'][:12], round(d['value'],1), round(d['roofline']['avg_launch_ms']*1000,1))"
  done
done
MICRO_PDL=1 python tools/host_overhead.py
