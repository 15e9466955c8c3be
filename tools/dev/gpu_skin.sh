# Verlet-skin MD loop: parity tests, MD tests, default bench with and without the skin
timeout 900 python -m pytest tests/test_gpu_skin.py tests/test_gpu_md.py -q -x -p no:cacheprovider > gpurun_out/skin_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/skin_tests.log
for sk in 0 0.1 0.05 0.15; do
  HMDP_SKIN=$sk timeout 600 python bench.py > gpurun_out/bench_skin_$sk.json 2> gpurun_out/bench_skin_$sk.err; echo "bench skin=$sk rc=$?"
  python tools/show_bench.py gpurun_out/bench_skin_$sk.json 2>&1 | grep -v "^ *event"
done
