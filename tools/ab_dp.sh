# usage: ab_dp.sh ALT.so "models" "systems" — A/B the in-tree libhmdp.so against ALT.so on
# the DeePMD-style families (dev aid; interleaved runs)
ALT=$1; MODELS=${2:-"repformer repflow"}; SYSTEMS=${3:-"1YRF 2PTC"}
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/cur.so
for rep in 1 2; do for lib in cur alt; do
  if [ $lib = alt ]; then cp $ALT paper_2602_02234_b200/lib/libhmdp.so; else cp /tmp/cur.so paper_2602_02234_b200/lib/libhmdp.so; fi
  for m in $MODELS; do for s in $SYSTEMS; do
    python bench.py --model $m --system $s --no-cpu-baseline --steps 500 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', '$m', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))"
  done; done
done; done
cp /tmp/cur.so paper_2602_02234_b200/lib/libhmdp.so
