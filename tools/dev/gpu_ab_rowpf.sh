# A/B: Verlet filter's row loads issued before the count arrives (rowpf) vs base
timeout 600 python -m pytest tests/test_gpu_skin.py -q -x -p no:cacheprovider 2>&1 | tail -2
AB_REPS=3 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:1YRF dpa2:1UBQ" timeout 1500 bash tools/ab_env.sh lib_alt/base.so@- lib_alt/rowpf.so@- 2>&1 | tee gpurun_out/ab_rowpf.txt
