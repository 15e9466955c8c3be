# force-kernel lanes per atom on the small and the replicated boxes
AB_REPS=2 AB_STEPS=600 AB_CFGS="dpa3:1YRF dpa3:1UBQ dpa2:1UBQ dpa2:1YRF dpa3:2PTC:2,2,2 dpa2:2PTC:2,2,2" timeout 1700 bash tools/ab_env.sh - HMDP_FORCE_FG=16 HMDP_FORCE_FG=8 2>&1 | tee gpurun_out/ab_fg2.txt
