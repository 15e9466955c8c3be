# headline + config benches (1 GPU): DPA3 / DPA2 x 1YRF / 2PTC
for m in dpa3 dpa2; do for s in 1YRF 2PTC; do
  python bench.py --model $m --system $s > gpurun_out/main_${m}_${s}.json 2> gpurun_out/main_${m}_${s}.err
  python -c "import json;d=json.load(open('gpurun_out/main_${m}_${s}.json'));r=d['roofline'];print('$m $s', round(d['value']), round(d['ms_per_step']*1000,1), round(d['warm_l2_graph100']['steps_per_s']), round(d['e2e']['value']), r['kernel'], round(r['frac'],4), r['traffic'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['clocks'])"
done; done
