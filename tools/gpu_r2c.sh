cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_dist.py tests/test_gpu_acceptance.py tests/test_gpu_cpp.py "tests/test_gpu_configs.py::test_c2_partitioned_cluster_and_group" -m gpu -q -x > gpurun_out/pytest_r2c.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_r2c.log
python tools/c1_exp.py > gpurun_out/c1_exp2.txt 2>&1; cat gpurun_out/c1_exp2.txt
for w in c1 c3; do
timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --dtype f32 --no-dense --no-other-dtype > gpurun_out/b_$w.log 2>&1; echo $w rc=$?
python -c "import json;j=json.loads([l for l in open('gpurun_out/b_$w.log') if l.startswith('{')][-1]);print(j['value'], j['roofline']['frac'], j['roofline']['step_frac'], j['protocol'])"
done
python tools/prof_step.py --workload c3 --mode group --n 8 --steps 3 --prime 300
python tools/prof_step.py --workload c1 --mode group --n 8 --steps 3 --prime 300
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8.csv python tools/prof_step.py --workload c3 --mode group --n 8 --steps 1 --prime 300 > /dev/null 2>&1
python tools/launches.py gpurun_out/g8.csv
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c8.csv python tools/prof_step.py --workload c3 --mode cluster --n 8 --steps 1 --prime 300 > /dev/null 2>&1
python tools/launches.py gpurun_out/c8.csv
