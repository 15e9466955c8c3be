# every paper box x {DPA2, DPA3} (1 GPU): steps/s, ns/day, roofline, CPU reference beside it
for m in dpa3 dpa2; do for s in 1YRF 1UBQ 3LZM 2PTC; do
  python bench.py --model $m --system $s --steps 1000 --cpu-seconds 8 > gpurun_out/sys_${m}_${s}.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/sys_${m}_${s}.json'));r=d['roofline'];c=d['cpu_baseline'];print('| $m | $s | %d | %.0f | %.0f | %.1f %% (%s) | %.1f (%d thr) |' % (d['config']['atoms'], d['value'], d['ns_per_day'], 100*r['frac'], r['kernel'], c['value'], c['cores']))"
done; done
