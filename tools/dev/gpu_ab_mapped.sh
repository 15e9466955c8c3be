# hmdp_compute output path re-check on another box: host-mapped writes (default) vs D2H copy node
AB_REPS=3 AB_STEPS=600 AB_CFGS="dpa3:2PTC dpa2:2PTC" timeout 1500 bash tools/ab_env.sh - HMDP_CGRAPH_MAPPED_OUT=0 2>&1 | tee gpurun_out/ab_mapped.txt
for m in dpa3 dpa2; do HMDP_E2E_PROBE=1 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; HMDP_CGRAPH_MAPPED_OUT=0 HMDP_E2E_PROBE=1 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; done
