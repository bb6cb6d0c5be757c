cd $GRAFT_REPO_ROOT
P8="python bench.py --workload c1 --cluster-workers 8 --steps 4 --warmup 3 --prime 300 --no-cpu-baseline"
timeout 300 $P8 > gpurun_out/c1x8.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__sectors_read.sum,dram__sectors_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum --clock-control none -k regex:"k_cluster_reduce" -s 301 -c 2 --csv --log-file gpurun_out/reduce_metrics.csv $P8 > gpurun_out/reduce_ncu.log 2>&1; echo rc=$?
tail -1 gpurun_out/c1x8.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("density", d["density"], "K", d["density"]*11700000)'
