set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_md.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
AB_REPS=2 AB_CFGS="${CFGS:-dpa3:2PTC dpa3:1YRF dpa3:1UBQ dpa2:2PTC dpa2:1YRF}" timeout 1500 bash tools/ab_env.sh $AB_ENVS 2>&1 | tee gpurun_out/ab.txt
