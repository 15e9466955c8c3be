for mode in dd dd-gather dd-allreduce; do for g in 2 4; do
  BENCH_DD_BACKEND=gloo timeout 600 python bench.py --gpus $g --steps 30 --warmup 3 --mode $mode --no-cpu-baseline > gpurun_out/dry_${mode}_$g.json 2> gpurun_out/dry_${mode}_$g.err
  python -c "import json; d=json.load(open('gpurun_out/dry_${mode}_$g.json')); print('$mode', $g, round(d['value'],1), round(d['ms_per_step'],3), d.get('extensivity',{}).get('rel_diff'))" || tail -3 gpurun_out/dry_${mode}_$g.err
done; done
for m in se_a repformer repflow; do
  timeout 600 python bench.py --model $m --system 2PTC --also "" --no-cpu-baseline --steps 200 > gpurun_out/fam_$m.json 2> gpurun_out/fam_$m.err
  python -c "import json; d=json.load(open('gpurun_out/fam_$m.json')); print('$m', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/fam_$m.err
done
timeout 900 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/ref.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/ref.json')); print('ref', d['value'], d['impl'])"
