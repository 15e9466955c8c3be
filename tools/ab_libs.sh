# usage: ab_libs.sh A.so B.so ... — interleaved bench of the in-tree libhmdp.so ("cur")
# against alternative builds (dev aid; the in-tree lib is restored at the end)
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/cur.so
for rep in 1 2; do for lib in /tmp/cur.so "$@"; do
  cp $lib paper_2602_02234_b200/lib/libhmdp.so
  python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1 || echo "$lib SMOKE FAILED"
  for m in dpa3 dpa2; do for s in 1YRF 2PTC; do
    python bench.py --model $m --system $s --no-cpu-baseline --steps 1000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$(basename $lib)', '$m', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))"
  done; done
done; done
cp /tmp/cur.so paper_2602_02234_b200/lib/libhmdp.so
