# Verlet filter CTA shape at 2PTC / 3LZM: teams (warps, G=1) per CTA
AB_REPS=2 AB_STEPS=800 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa2:3LZM" timeout 1500 bash tools/ab_env.sh - HMDP_SEARCH_T=8 HMDP_SEARCH_T=16 HMDP_SEARCH_T=4 2>&1 | tee gpurun_out/ab_st.txt
