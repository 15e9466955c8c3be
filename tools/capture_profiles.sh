# usage: capture_profiles.sh TAG — launch lists + one-step ncu --set full captures
TAG=$1
mkdir -p gpurun_out
for cfg in "dpa3 1YRF" "dpa2 1YRF" "dpa3 2PTC" "dpa2 2PTC"; do
  set -- $cfg
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 70 --csv \
      --log-file gpurun_out/launches_${TAG}_$1_$2.csv python tools/ncu_target.py $1 $2 20 > /dev/null 2>&1
  n=$([ "$1" = dpa3 ] && echo 7 || echo 3)
  ncu --set full --import-source on --clock-control none --cache-control none -s $((n*4+2)) -c $n \
      -o gpurun_out/full_${TAG}_$1_$2 python tools/ncu_target.py $1 $2 8 > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
