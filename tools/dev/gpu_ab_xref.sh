# A/B: Verlet reference position loaded with the MD state at the top of the force kernel
AB_REPS=3 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:1YRF" timeout 1500 bash tools/ab_env.sh lib_alt/base.so@- lib_alt/xref.so@- 2>&1 | tee gpurun_out/ab_xref.txt
