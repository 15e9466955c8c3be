# A/B of the Verlet filter's blocks in flight per warp (HMDP_FILTER_U builds in lib_alt/)
AB_REPS=2 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:1YRF dpa2:1UBQ" timeout 1500 bash tools/ab_env.sh lib_alt/u4.so@- lib_alt/u2.so@- lib_alt/u5.so@- 2>&1 | tee gpurun_out/ab_filter.txt
