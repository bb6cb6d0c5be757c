cd $GRAFT_REPO_ROOT
run() { timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/wl.log >> gpurun_out/workloads_c5.jsonl; }
rm -f gpurun_out/workloads_c5.jsonl
run --workload c5_d001 --steps 20 --warmup 3
run --workload c5_d01 --steps 20 --warmup 3
run --workload c5_d1 --steps 20 --warmup 3
run --workload c5_d1 --steps 20 --warmup 3 --no-dense
python tools/make_tables.py gpurun_out/workloads_c5.jsonl
