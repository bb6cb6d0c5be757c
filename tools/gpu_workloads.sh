# Bench lines for the other BASELINE configs, the in-process cluster mode and
# the comparison sparsifiers (tables: python tools/make_tables.py).
# Default: f64 arithmetic (the reference's own) on fp32 gradients (BASELINE's
# "fp32 gradient", widened exactly), with the f32-arithmetic line and the
# f64-gradient line beside it; the dense g/n and the model update in every step.
cd $GRAFT_REPO_ROOT
run() { timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/wl.log >> gpurun_out/workloads.jsonl; }
rm -f gpurun_out/workloads.jsonl
run --workload c1 --steps 200
run --workload c1 --steps 200 --no-dense
run --workload c3 --steps 100
run --workload c3 --steps 100 --no-dense
run --workload c4 --steps 50
run --workload c5_d001 --steps 20 --warmup 3
run --workload c5_d01 --steps 20 --warmup 3
run --workload c5_d1 --steps 20 --warmup 3
run --workload c5_d1 --steps 20 --warmup 3 --no-dense
run --workload c1 --cluster-workers 2 --steps 100
run --workload c1 --cluster-workers 8 --steps 100
run --workload c3 --cluster-workers 8 --steps 20 --prime 3000
for k in topk hard dense; do run --workload c3 --sparsifier $k --steps 20 --prime 200 --dtype f32 --no-dense; done
for k in topk cltk hard; do run --workload c1 --cluster-workers 8 --sparsifier $k --steps 30 --prime 200 --dtype f32 --no-dense; done
