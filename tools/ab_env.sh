# usage: ab_env.sh SPEC... — interleaved bench of library builds x environment settings
# (dev aid for the A/B switches in hmdp_net.cu).  SPEC = [LIB@]ENV[,ENV...]: LIB is an
# alternative libhmdp.so (e.g. lib_alt/base.so, copied over the in-tree library for
# the run and restored after); ENV e.g. HMDP_PULL=1 ("-" = none).
# AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:2PTC:2,2,2" selects the configs (model:system[:replicas]), AB_REPS the repetitions.
CFGS=${AB_CFGS:-"dpa3:2PTC dpa3:1YRF"}
LIBF=paper_2602_02234_b200/lib/libhmdp.so
cp $LIBF /tmp/ab_cur.so
for rep in $(seq ${AB_REPS:-2}); do for spec in "$@"; do
  lib=/tmp/ab_cur.so; envs=$spec
  case "$spec" in *@*) lib=${spec%%@*}; envs=${spec#*@};; esac
  cp $lib $LIBF
  envs=$(echo "$envs" | tr ',' ' '); [ "$envs" = "-" ] && envs=""
  for c in $CFGS; do IFS=: read m s r <<< "$c"; r=${r:-1,1,1}
    env $envs python bench.py --model $m --system $s --replicas $r --also "" --no-cpu-baseline --steps ${AB_STEPS:-1000} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$spec', '$m', '$s', '$r', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']), round(d['e2e']['value']), {k: round(v, 1) for k, v in d.get('kernels_event_us', {}).items()})"
  done
done; done
cp /tmp/ab_cur.so $LIBF
