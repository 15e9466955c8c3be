# network team size / CTA build re-check after the Verlet rows and the force re-sweep
AB_REPS=2 AB_STEPS=800 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:3LZM" timeout 1700 bash tools/ab_env.sh - HMDP_TEAM=1 HMDP_TEAM=4 HMDP_WIDE=0 HMDP_SKIN=0.08 HMDP_SKIN=0.12 2>&1 | tee gpurun_out/ab_team.txt
