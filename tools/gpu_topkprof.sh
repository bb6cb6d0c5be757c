cd $GRAFT_REPO_ROOT
P="python bench.py --sparsifier topk --steps 3 --warmup 3 --prime 20 --no-cpu-baseline"
timeout 300 $P > gpurun_out/topk.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_t|^k1_|^k_b|^k_f|^k_u|^k_w|^Device" -s 414 -c 36 --csv --log-file gpurun_out/topk_launches.csv $P > /dev/null 2>&1; echo rc=$?
