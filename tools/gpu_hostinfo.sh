# GPU call: host facts the oracle-at-size tests and the reference arm depend on
cd $GRAFT_REPO_ROOT
{ nproc; free -g; lscpu | grep -E 'Model name|Socket|Core|Thread|L3|NUMA node\(s\)'; nvidia-smi --query-gpu=name,memory.total --format=csv; df -h /tmp | tail -1; } > gpurun_out/hostinfo.txt 2>&1
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/c1_bench.log 2>&1
timeout 300 python bench.py --workload c1 --steps 50 --warmup 5 --no-cpu-baseline --flush-l2 off > gpurun_out/c1_bench_noflush.log 2>&1
cat gpurun_out/hostinfo.txt gpurun_out/host_overhead.txt
tail -c 600 gpurun_out/c1_bench.log
