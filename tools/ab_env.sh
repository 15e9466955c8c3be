# usage: ab_env.sh "HMDP_PULL=0" "HMDP_PULL=2" ... — interleaved bench of environment
# settings of the in-tree libhmdp.so (dev aid for the A/B switches in hmdp_net.cu).
# AB_CFGS="dpa3:2PTC dpa2:2PTC" selects the configs, AB_REPS the interleaved repetitions.
CFGS=${AB_CFGS:-"dpa3:2PTC dpa3:1YRF"}
for rep in $(seq ${AB_REPS:-2}); do for envs in "$@"; do
  for c in $CFGS; do m=${c%%:*}; s=${c##*:}
    env $envs python bench.py --model $m --system $s --also "" --no-cpu-baseline --steps ${AB_STEPS:-1000} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$envs', '$m', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']), round(d['e2e']['value']), {k: round(v, 1) for k, v in d.get('kernels_event_us', {}).items()})"
  done
done; done
