cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for pdl in 1 0; do
  MICRO_PDL=$pdl timeout 600 python bench.py --workload c1 --cluster-workers 8 --steps 50 --warmup 5 --no-cpu-baseline --prime 300 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl=$pdl c1x8', round(d['value'],1))"
done
