# Verlet skin on the MD loop + hmdp_compute graph path: skin tests, full GPU suite, bench
timeout 900 python -m pytest tests/test_gpu_skin.py -q -x -p no:cacheprovider > gpurun_out/skin_tests.log 2>&1; echo "skin pytest rc=$?"; tail -15 gpurun_out/skin_tests.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_all.log
for sk in 0 0.1; do
  HMDP_SKIN=$sk timeout 600 python bench.py > gpurun_out/bench_skin_$sk.json 2> gpurun_out/bench_skin_$sk.err; echo "bench skin=$sk rc=$?"
  python tools/show_bench.py gpurun_out/bench_skin_$sk.json 2>&1 | grep -v "^ *event"
done
