# A/B: contiguous force / per-atom stores in k_force (fstore) x hmdp_compute output path (copy node vs mapped)
timeout 900 python -m pytest tests/test_gpu_skin.py tests/test_gpu_parity.py tests/test_gpu_md.py tests/test_gpu_halo.py -q -x -p no:cacheprovider 2>&1 | tail -2
AB_REPS=2 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:1YRF dpa2:1UBQ" timeout 2000 bash tools/ab_env.sh lib_alt/base.so@- lib_alt/fstore.so@- lib_alt/fstore.so@HMDP_CGRAPH_MAPPED_OUT=1 lib_alt/base.so@HMDP_CGRAPH_MAPPED_OUT=1 2>&1 | tee gpurun_out/ab_fstore.txt
