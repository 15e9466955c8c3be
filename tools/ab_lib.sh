# usage: ab_lib.sh ALT.so — bench the in-tree libhmdp.so against ALT.so (dev aid)
ALT=$1
run() { for m in dpa3 dpa2; do for s in 1YRF 2PTC; do
  python bench.py --model $m --system $s --no-cpu-baseline --steps 1000 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$1', '$m', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))"
done; done; }
run base
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/base.so
cp $ALT paper_2602_02234_b200/lib/libhmdp.so
run alt
cp /tmp/base.so paper_2602_02234_b200/lib/libhmdp.so
