cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py -q -x 2>&1 | tail -1
for args in "--workload c3" "--workload c5_d1 --steps 10 --prime 300" "--workload c3 --sparsifier dense --prime 5" "--workload c3 --sparsifier hard --prime 50" "--workload c1 --cluster-workers 8"; do
  timeout 900 python bench.py $args --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ilp.log 2>&1
  echo "$args rc=$? $(tail -1 gpurun_out/ilp.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["avg_launch_ms"]*1000,1), round(d["density"]*100,4))')"
done
