set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_md.py -q -x -p no:cacheprovider > gpurun_out/pull2_tests.log 2>&1; echo "pull2 rc=$?"; tail -3 gpurun_out/pull2_tests.log
HMDP_PULL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pull1_tests.log 2>&1; echo "pull1 rc=$?"; tail -3 gpurun_out/pull1_tests.log
AB_REPS=2 AB_CFGS="dpa3:2PTC dpa3:1YRF dpa3:1UBQ" timeout 1200 bash tools/ab_env.sh HMDP_PULL=0 HMDP_PULL=1 HMDP_PULL=2 2>&1 | tee gpurun_out/ab_pull.txt
