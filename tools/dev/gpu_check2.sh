timeout 900 python -m pytest tests/test_gpu_skin.py tests/test_gpu_md.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t.log
for m in dpa3 dpa2; do HMDP_E2E_PROBE=1 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python tools/show_bench.py gpurun_out/bench_default.json | grep -v event
