# GPU call (round 2): one launch list + one ncu --set full capture per
# profiled workload, the profiled steps only (tools/prof_step.py brackets
# them with cudaProfilerStart/Stop).  Outputs in gpurun_out/r2prof/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2prof; mkdir -p $O
P="python tools/prof_step.py"
run() {  # name, args...
  name=$1; shift
  timeout 300 $P "$@" > $O/$name.plain.txt 2>&1; echo "$name plain rc=$?"; tail -1 $O/$name.plain.txt
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $O/$name.launches.csv $P "$@" > /dev/null 2>&1; echo "$name launches rc=$?"
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
     -k regex:"${KREGEX:-k1_|k_[a-rt-z]}" -c ${NCU_COUNT:-6} -o $O/$name $P "$@" > $O/$name.ncu.log 2>&1; echo "$name full rc=$?"
  # summaries only travel back (gpurun_out is capped at 64 MiB); keep the report when KEEP=1
  python tools/summarize_ncu.py $O/$name.ncu-rep $O/$name.summary.json > /dev/null 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
  [ "$KEEP" = 1 ] || rm -f $O/$name.ncu-rep
}
if [ -n "$ONLY_XCHG" ]; then
KREGEX="k1_gather|k_peer|k_cluster|k_finalize|k_dist" NCU_COUNT=12 run c3_group8 --workload c3 --dtype f32 --mode group --n 8 --steps 1 --prime 300
KREGEX="k1_gather|k_peer|k_cluster|k_finalize|k_dist" NCU_COUNT=12 run c3_cluster8 --workload c3 --dtype f32 --mode cluster --n 8 --steps 1 --prime 300
KREGEX="k1_gather|k_peer|k_cluster|k_finalize|k_dist" NCU_COUNT=12 run c1_group8 --workload c1 --dtype f32 --mode group --n 8 --steps 1 --prime 300
KREGEX="k1_gather|k_peer|k_cluster|k_finalize|k_dist" NCU_COUNT=12 run c1_cluster8 --workload c1 --dtype f32 --mode cluster --n 8 --steps 1 --prime 300
python tools/c1_exp.py > $O/c1_exp.txt 2>&1; cat $O/c1_exp.txt
python tools/c1_exp.py --dense > $O/c1_exp_dense.txt 2>&1; cat $O/c1_exp_dense.txt
du -sh $O; exit 0
fi
KEEP=1 run c3_f64_dense --workload c3 --dtype f64 --dense --steps 3
run c3_f32_dense --workload c3 --dtype f32 --dense --steps 3
run c3_f32 --workload c3 --dtype f32 --steps 3
run c1_f32_flush --workload c1 --dtype f32 --steps 5 --flush --prime 1000
KREGEX="k1_|k_" run c5_d1_f32 --workload c5_d1 --dtype f32 --steps 2 --prime 300
run c3_group8 --workload c3 --dtype f32 --mode group --n 8 --steps 2 --prime 60
run c3_cluster8 --workload c3 --dtype f32 --mode cluster --n 8 --steps 2 --prime 60
run c1_group8 --workload c1 --dtype f32 --mode group --n 8 --steps 3 --prime 300
du -sh $O; ls -la $O
