cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_full.log 2>&1; echo pytest rc=$?
tail -22 gpurun_out/pytest_full.log
for m in group cluster; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_$m.csv python tools/prof_step.py --workload c3 --mode $m --n 8 --steps 1 --prime 300 > /dev/null 2>&1
python tools/launches.py gpurun_out/x_$m.csv
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x1_$m.csv python tools/prof_step.py --workload c1 --mode $m --n 8 --steps 1 --prime 300 > /dev/null 2>&1
python tools/launches.py gpurun_out/x1_$m.csv
done
