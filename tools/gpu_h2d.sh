cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py -q -x -k "step_host or cpp" 2>&1 | tail -1
for p in 1 0; do
  MICRO_H2D_PIPELINE=$p timeout 600 python bench.py --steps 20 --warmup 3 --prime 300 --no-cpu-baseline | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pipeline=$p', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['h2d_gbs_effective'],2))"
done
