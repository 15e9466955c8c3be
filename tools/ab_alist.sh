# A/B: in-tree libhmdp.so (base) vs lib_alt/libhmdp_noalist.so, DPA3 1YRF/2PTC
run() { for k in 1 2; do for s in 1YRF 2PTC; do
  python bench.py --model dpa3 --system $s --no-cpu-baseline --steps 1500 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$1', '$s', round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))"
done; done; }
run base
cp paper_2602_02234_b200/lib/libhmdp.so /tmp/base.so
cp lib_alt/libhmdp_noalist.so paper_2602_02234_b200/lib/libhmdp.so
run alt
cp /tmp/base.so paper_2602_02234_b200/lib/libhmdp.so
