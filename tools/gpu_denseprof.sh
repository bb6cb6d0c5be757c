cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_baselines.py -q -x 2>&1 | tail -1
P="python bench.py --sparsifier dense --steps 3 --warmup 3 --prime 5 --no-cpu-baseline"
timeout 300 $P > gpurun_out/dense.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|^k1_" -s 12 -c 8 --csv --log-file gpurun_out/dense_launches.csv $P > /dev/null 2>&1; echo rc=$?
tail -1 gpurun_out/dense.log | cut -c1-150
P="python bench.py --sparsifier hard --steps 3 --warmup 3 --prime 5 --no-cpu-baseline"
timeout 300 $P > gpurun_out/hard.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_u|^k_f|^k1_" -s 20 -c 8 --csv --log-file gpurun_out/hard_launches.csv $P > /dev/null 2>&1; echo rc=$?
tail -1 gpurun_out/hard.log | cut -c1-150
