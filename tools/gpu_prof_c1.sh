# GPU call: ncu --set full with source of the C1 step (f64 + dense, the
# bench's default arithmetic; f32 beside it), reports kept in gpurun_out/c1prof
cd $GRAFT_REPO_ROOT
O=gpurun_out/c1prof; mkdir -p $O
P="python tools/prof_step.py"
for cfg in "c1_f64_dense --dtype f64 --dense" "c1_f32 --dtype f32"; do
  set -- $cfg; name=$1; shift
  timeout 300 $P --workload c1 --steps 4 --flush --prime 1000 "$@" > $O/$name.plain.txt 2>&1; echo "$name plain rc=$?"; tail -2 $O/$name.plain.txt
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
     -k regex:"k1_" -c 4 -o $O/$name $P --workload c1 --steps 2 --flush --prime 1000 "$@" > $O/$name.ncu.log 2>&1; echo "$name full rc=$?"
done
ls -la $O
