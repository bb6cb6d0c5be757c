cd $GRAFT_REPO_ROOT
P="python bench.py --sparsifier dense --steps 2 --warmup 3 --prime 3 --no-cpu-baseline"
timeout 300 $P > gpurun_out/dense.log 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:"k_dense_all" -s 5 -c 1 -o gpurun_out/dense_full $P > /dev/null 2>&1; echo rc=$?
