# full GPU suite + smoke + default bench + fresh launch lists/summaries + every paper box
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --junitxml=gpurun_out/gpu_all.xml > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/capture_and_summarize.sh r2g "dpa3 2PTC" "dpa2 2PTC" "dpa3 1YRF" "dpa2 1YRF" "dpa3 1UBQ" "dpa3 3LZM" > gpurun_out/cap.log 2>&1; echo "cap rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
bash tools/run_all_systems.sh 2>&1 | tee gpurun_out/all_systems.md
