# Code-path check of bench.py at N = 2 with both ranks on one GPU (gloo); numbers are not valid.
cd $GRAFT_REPO_ROOT
for tr in peer peer_pull nccl; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --dist-backend gloo --transport $tr --workload c1 --steps 5 --warmup 3 --prime 50 > gpurun_out/distbench_$tr.log 2>&1
  echo "$tr rc=$? $(tail -1 gpurun_out/distbench_$tr.log | cut -c1-150)"
done
