cd $GRAFT_REPO_ROOT
cp paper_2310_00967_b200/lib/libmicro_b200.so /tmp/lib_d2.so
for L in 2 4 8; do
  if [ $L != 2 ]; then cp gpurun_variants/lib_d$L.so paper_2310_00967_b200/lib/libmicro_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stream and (10000-1 or 4095-1 or 5-5)" 2>&1 | tail -1
  timeout 600 python bench.py --dense --steps 50 --warmup 5 --prime 500 --no-cpu-baseline | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('lanes=$L', round(d['value'],1), round(d['roofline']['avg_launch_ms']*1000,1))"
done
cp /tmp/lib_d2.so paper_2310_00967_b200/lib/libmicro_b200.so
