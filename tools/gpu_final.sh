# GPU call (round 2, final build): the -m gpu suite, the default bench line
# and the reference arm, the launch list of the bench command (ncu
# gpu__time_duration), ncu --set full summaries of the profiled steps, and
# the workloads table.  Outputs in gpurun_out/final/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
if [ -z "$SKIP_TESTS" ]; then
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q --durations=20 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
fi
timeout 900 python bench.py --steps 50 --warmup 5 > $O/bench.log 2>&1; echo bench rc=$?; tail -1 $O/bench.log > $O/bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.log 2>&1; echo ref rc=$?; tail -1 $O/ref.log > $O/ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-other-dtype > $O/ncu_launch.log 2>&1; echo launches rc=$?
P="python tools/prof_step.py"
prof() {  # name, args...
  name=$1; shift
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
     -k regex:"k1_" -c 4 -o $O/$name $P "$@" > $O/$name.ncu.log 2>&1; echo "$name full rc=$?"
  python tools/summarize_ncu.py $O/$name.ncu-rep $O/$name.summary.json > /dev/null 2>&1
  [ "$KEEP" = 1 ] || rm -f $O/$name.ncu-rep
}
KEEP=1 prof c3_f64_g32_dense --workload c3 --dtype f64 --grad f32 --dense --steps 2
prof c3_f64_dense --workload c3 --dtype f64 --dense --steps 2
prof c3_f32_dense --workload c3 --dtype f32 --dense --steps 2
prof c1_f64_g32_dense --workload c1 --dtype f64 --grad f32 --dense --steps 2 --flush --prime 3000
prof c5_d1_f64_g32_dense --workload c5_d1 --dtype f64 --grad f32 --dense --steps 1 --prime 3000
if [ -n "$WORKLOADS" ]; then bash tools/gpu_workloads.sh; cp gpurun_out/workloads.jsonl $O/; fi
du -sh $O
