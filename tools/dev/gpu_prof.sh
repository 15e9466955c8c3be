set -x
bash tools/capture_and_summarize.sh r2b "dpa3 2PTC" "dpa2 2PTC" "dpa3 1YRF" "dpa2 1YRF" > gpurun_out/cap.log 2>&1; echo "cap rc=$?"
for p in 0 1 2; do
  HMDP_PULL=$p ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 42 -c 21 --csv --log-file gpurun_out/traffic_pull$p.csv python tools/ncu_target.py dpa3 2PTC 12 > /dev/null 2>&1
done
ls gpurun_out/profiles/round2
