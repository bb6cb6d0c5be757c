cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_baselines.py -x -q > gpurun_out/pytest_red.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_red.log
for args in "--workload c1 --cluster-workers 8" "--workload c1 --cluster-workers 2" "--workload c3 --cluster-workers 8"; do
  timeout 600 python bench.py $args --steps 30 --warmup 3 --prime 300 --no-cpu-baseline > gpurun_out/red.log 2>&1
  echo "$args rc=$? $(tail -1 gpurun_out/red.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["avg_launch_ms"]*1000,1), round(d["roofline"]["step_frac"],3), round(d["density"]*100,4))')"
done
P8="python bench.py --workload c1 --cluster-workers 8 --steps 4 --warmup 3 --prime 100 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_reduce" -s 100 -c 1 -o gpurun_out/reduce_full2 $P8 > gpurun_out/reduce_ncu.log 2>&1; echo ncu rc=$?
