for sys in 1UBQ 3LZM 2PTC; do for t in 1 2 4; do
r=$(HMDP_TEAM=$t python bench.py --model dpa3 --system $sys --no-cpu-baseline --steps 500 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))")
r2=$(HMDP_TEAM=$t python bench.py --model dpa2 --system $sys --no-cpu-baseline --steps 500 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']), round(d['warm_l2_graph100']['steps_per_s']))")
echo "$sys G=$t dpa3 $r dpa2 $r2"
done; done
