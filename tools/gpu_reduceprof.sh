cd $GRAFT_REPO_ROOT
P8="python bench.py --workload c1 --cluster-workers 8 --steps 4 --warmup 3 --prime 100 --no-cpu-baseline"
timeout 300 $P8 > gpurun_out/c1x8.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_reduce" -s 100 -c 1 -o gpurun_out/reduce_full $P8 > gpurun_out/reduce_ncu.log 2>&1; echo rc=$?
