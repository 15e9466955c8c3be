# usage: capture_profiles.sh TAG ["model system" ...] — launch lists + one-step ncu --set full captures
TAG=$1
shift
CFGS=("$@")
[ ${#CFGS[@]} -eq 0 ] && CFGS=("dpa3 1YRF" "dpa2 1YRF" "dpa3 2PTC" "dpa2 2PTC")
mkdir -p gpurun_out
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  # kernels per MD step (search + network + force)
  case $1 in dpa3|repformer|repflow) n=7 ;; *) n=3 ;; esac
  # 60 steps: the Verlet-row rebuilds (every ~20-40 steps at dt 1 fs, skin 0.1 nm) are in the list
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s $((n*6)) -c $((n*60)) --csv \
      --log-file gpurun_out/launches_${TAG}_$1_$2.csv python tools/ncu_target.py $1 $2 70 > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none --cache-control none -s $((n*4+2)) -c $n \
      -o gpurun_out/full_${TAG}_$1_$2 python tools/ncu_target.py $1 $2 8 > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
