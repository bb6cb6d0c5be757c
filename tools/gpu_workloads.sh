# Bench lines for the other BASELINE configs and the in-process cluster mode.
cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/wl.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(json.dumps({k: j[k] for k in ['value','density','config']} | {'frac': j['roofline']['frac'], 'step_frac': j['roofline']['step_frac'], 'k1a_ms': j['roofline']['avg_launch_ms'], 'e2e': j['e2e']['value'] if j['e2e'] else None}))" | tee -a gpurun_out/workloads.jsonl; }
rm -f gpurun_out/workloads.jsonl
run --workload c1 --steps 200
run --workload c3 --steps 100
run --workload c4 --steps 50
run --workload c5_d001 --steps 20 --warmup 3 --prime 300
run --workload c5_d01 --steps 20 --warmup 3 --prime 300
run --workload c5_d1 --steps 20 --warmup 3 --prime 300
run --workload c1 --cluster-workers 2 --steps 100
run --workload c1 --cluster-workers 8 --steps 100
run --workload c3 --cluster-workers 8 --steps 20 --prime 300
