# Verlet-row mirror tables for k_embed's rev (mtab) vs the per-step mirror search (base)
timeout 900 python -m pytest tests/test_gpu_skin.py tests/test_gpu_md.py tests/test_gpu_parity.py tests/test_dpfamily.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
AB_REPS=2 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:1YRF dpa2:1UBQ" timeout 1500 bash tools/ab_env.sh lib_alt/base.so@- lib_alt/mtab.so@- 2>&1 | tee gpurun_out/ab_mtab.txt
