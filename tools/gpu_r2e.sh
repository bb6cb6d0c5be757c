cd $GRAFT_REPO_ROOT
# the driver's two arms, as it runs them
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_default.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/ref_default.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_default.log
bash tools/gpu_workloads.sh
python tools/make_tables.py gpurun_out/workloads.jsonl
