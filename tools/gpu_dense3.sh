cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_baselines.py -q -x -k dense 2>&1 | tail -1
timeout 600 python bench.py --sparsifier dense --steps 10 --warmup 3 --prime 3 --no-cpu-baseline > gpurun_out/dense.log 2>&1; tail -1 gpurun_out/dense.log | cut -c1-160
P="python bench.py --sparsifier dense --steps 2 --warmup 3 --prime 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dense_all" -s 5 -c 1 --csv $P 2>/dev/null | grep -v "^==" | tail -3
