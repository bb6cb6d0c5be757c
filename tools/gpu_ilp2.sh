cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for args in "--workload c3" "--workload c5_d1 --steps 10 --prime 300" "--workload c5_d01 --steps 10 --prime 300" "--workload c3 --sparsifier dense --prime 5" "--workload c1 --cluster-workers 8 --sparsifier cltk"; do
  timeout 900 python bench.py $args --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ilp.log 2>&1
  echo "$args rc=$? $(tail -1 gpurun_out/ilp.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["avg_launch_ms"]*1000,1), round(d["density"]*100,4))')"
done
