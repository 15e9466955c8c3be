# every paper box x {DPA2, DPA3} (1 GPU): steps/s, ns/day, roofline, CPU reference beside it
for m in dpa3 dpa2; do for s in 1YRF 1UBQ 3LZM 2PTC; do
  python bench.py --model $m --system $s --also "" --steps 1000 --cpu-seconds 8 > gpurun_out/sys_${m}_${s}.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/sys_${m}_${s}.json'));r=d['roofline'];c=d['cpu_baseline'];print('| $m | $s | %d | %.0f | %.0f | %.1f %% (%s) | %.1f (%d thr) |' % (d['config']['atoms'], d['value'], d['ns_per_day'], 100*r['frac'], r['kernel'], c['value'], c['cores']))"
done; done
# weak-scaled replicas of the 2PTC box on one GPU
for m in dpa3 dpa2; do for r in 2,2,2 4,4,4; do
  python bench.py --model $m --system 2PTC --replicas $r --also "" --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/rep_${m}_${r}.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/rep_${m}_${r}.json'));r=d['roofline'];print('| $m | 2PTC x($r) | %d | %.1f | %.2f ms | %.1f %% (%s) |' % (d['config']['atoms'], d['value'], d['ms_per_step'], 100*r['frac'], r['kernel']))"
done; done
