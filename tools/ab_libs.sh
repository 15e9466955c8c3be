# usage: ab_libs.sh A.so B.so ... — interleaved bench of the in-tree libhmdp.so ("cur")
# against alternative builds (dev aid; the in-tree lib is restored at the end).
# AB_CFGS="dpa3:2PTC dpa2:2PTC" selects the configs, AB_REPS the interleaved repetitions.
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/cur.so
CFGS=${AB_CFGS:-"dpa3:2PTC dpa2:2PTC dpa3:1YRF dpa2:1YRF"}
for rep in $(seq ${AB_REPS:-2}); do for lib in /tmp/cur.so "$@"; do
  cp $lib paper_2602_02234_b200/lib/libhmdp.so
  python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1 || echo "$lib SMOKE FAILED"
  for c in $CFGS; do m=${c%%:*}; s=${c##*:}
    python bench.py --model $m --system $s --also "" --no-cpu-baseline --steps 1000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$(basename $lib)', '$m', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']), round(d['e2e']['value']))"
  done
done; done
cp /tmp/cur.so paper_2602_02234_b200/lib/libhmdp.so
