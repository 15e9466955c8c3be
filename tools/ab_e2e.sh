# usage: ab_e2e.sh ALT.so — interleaved hmdp_compute e2e probe: in-tree lib vs ALT.so (dev aid)
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/cur.so
for rep in 1 2; do for lib in /tmp/cur.so $1; do
  cp $lib paper_2602_02234_b200/lib/libhmdp.so
  for c in "dpa3 582" "dpa2 582" "dpa2 4114"; do
    echo "$(basename $lib) $c $(python tools/e2e_probe.py $c 2>/dev/null | grep raw)"
  done
done; done
cp /tmp/cur.so paper_2602_02234_b200/lib/libhmdp.so
