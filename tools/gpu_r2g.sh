cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py "tests/test_gpu_configs.py::test_c5_gpt2xl_density_sweep" tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_r2g.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_r2g.log
run() { timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/wl.log 2>&1; echo "== $* rc=$?"; tail -1 gpurun_out/wl.log >> gpurun_out/w_r2g.jsonl; }
rm -f gpurun_out/w_r2g.jsonl
run --workload c5_d1 --steps 20 --warmup 3 --no-dense
run --workload c5_d1 --steps 20 --warmup 3
run --workload c3 --steps 50 --no-dense
run --workload c3 --steps 50
python tools/make_tables.py gpurun_out/w_r2g.jsonl
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5k.csv python tools/prof_step.py --workload c5_d1 --steps 2 --prime 300 > /dev/null 2>&1
python - <<'P'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/c5k.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    print(r[ki][:60], r[mi], r[vi])
P
