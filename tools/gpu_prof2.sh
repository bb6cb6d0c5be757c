# ncu --set full captures of the secondary kernels (cluster reduce, finalize, top-k histogram, dense pass)
cd $GRAFT_REPO_ROOT
P8="python bench.py --workload c3 --cluster-workers 8 --steps 2 --warmup 3 --prime 300 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k regex:"k_cluster_reduce|k_finalize" -s 606 -c 2 -o gpurun_out/sec_cluster $P8 > gpurun_out/sec1.log 2>&1; echo cluster rc=$?
PT="python bench.py --sparsifier topk --steps 2 --warmup 3 --prime 10 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k regex:"k_topk_hist|k1_stream" -s 39 -c 4 -o gpurun_out/sec_topk $PT > gpurun_out/sec2.log 2>&1; echo topk rc=$?
PD="python bench.py --sparsifier dense --steps 2 --warmup 3 --prime 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k regex:"k_dense_all" -s 5 -c 1 -o gpurun_out/sec_dense $PD > gpurun_out/sec3.log 2>&1; echo dense rc=$?
