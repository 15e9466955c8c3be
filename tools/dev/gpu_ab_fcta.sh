# force-kernel CTA size (HMDP_FORCE_CTA builds): 128 (base) vs 64 vs 256
AB_REPS=2 AB_STEPS=800 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa2:1YRF dpa2:3LZM dpa2:2PTC:2,2,2" timeout 1700 bash tools/ab_env.sh lib_alt/base.so@- lib_alt/fcta64.so@- lib_alt/fcta256.so@- 2>&1 | tee gpurun_out/ab_fcta.txt
