# Verlet filter / search team size (warps per atom) by box
AB_REPS=2 AB_STEPS=800 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa2:3LZM dpa2:1UBQ dpa2:1YRF" timeout 1700 bash tools/ab_env.sh - HMDP_SEARCH_G=1 HMDP_SEARCH_G=2 HMDP_SEARCH_G=4 2>&1 | tee gpurun_out/ab_sg.txt
