for m in dpa3 dpa2; do HMDP_E2E_PROBE=1 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; done
for m in dpa3 dpa2; do HMDP_E2E_PROBE=1 HMDP_SKIN=0 python tools/dev/e2e_breakdown.py $m 2>&1 | tail -2; done
