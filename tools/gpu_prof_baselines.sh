# ncu --set full of the comparison sparsifiers' batched / fused kernels at C1 x 8 (f32):
# the union by words (hard threshold, 35 % union) and the batched top-k pass + union gather
cd $GRAFT_REPO_ROOT
B="python bench.py --workload c1 --cluster-workers 8 --steps 1 --warmup 3 --prime 3 --dtype f32 --no-dense --no-cpu-baseline --no-other-dtype"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_union_words|k_union_reduce" -s 2 -c 2 \
  -o gpurun_out/bl_hard_full -f $B --sparsifier hard > gpurun_out/bl_hard_full.log 2>&1; echo "hard rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_topk_hist_b|k_union_reduce|k_union_words" -s 6 -c 4 \
  -o gpurun_out/bl_topk_full -f $B --sparsifier topk > gpurun_out/bl_topk_full.log 2>&1; echo "topk rc=$?"
