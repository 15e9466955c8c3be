bash tools/capture_and_summarize.sh r2c "dpa3 2PTC" "dpa2 2PTC" "dpa3 1YRF" "dpa2 1YRF" "dpa3 1UBQ" "dpa3 3LZM" > gpurun_out/cap.log 2>&1; echo "cap rc=$?"
bash tools/run_all_systems.sh 2>&1 | tee gpurun_out/all_systems.md
