# full GPU suite + smoke + default bench (session re-entry check)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python tools/show_bench.py gpurun_out/bench_default.json 2>/dev/null | head -20
for m in dpa3 dpa2; do HMDP_E2E_PROBE=1 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; done
