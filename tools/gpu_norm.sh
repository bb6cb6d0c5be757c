cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
for w in c3 c1; do
  for f in "" "--error-norm"; do
    timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --prime 600 $f > gpurun_out/norm_$w$f.log 2>&1
    echo "$w $f rc=$? $(tail -1 gpurun_out/norm_$w$f.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["avg_launch_ms"]*1000,1), round(d["density"]*100,4))')"
  done
done
