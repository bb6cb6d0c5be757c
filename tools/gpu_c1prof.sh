cd $GRAFT_REPO_ROOT
P1="python bench.py --workload c1 --steps 20 --warmup 3 --prime 300 --no-cpu-baseline"
P8="python bench.py --workload c1 --cluster-workers 8 --steps 10 --warmup 3 --prime 100 --no-cpu-baseline"
timeout 300 $P1 > gpurun_out/c1.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k_fin|k_clu" -s 606 -c 40 --csv --log-file gpurun_out/c1_launches.csv $P1 > /dev/null 2>&1; echo c1 rc=$?
timeout 300 $P8 > gpurun_out/c1x8.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k_fin|k_clu" -s 1800 -c 54 --csv --log-file gpurun_out/c1x8_launches.csv $P8 > /dev/null 2>&1; echo c1x8 rc=$?
tail -1 gpurun_out/c1.log | cut -c1-200; tail -1 gpurun_out/c1x8.log | cut -c1-200
