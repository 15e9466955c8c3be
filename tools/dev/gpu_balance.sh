# per-kernel SM activity spread (min/avg/max active cycles vs elapsed) for DPA3/DPA2 2PTC
for m in dpa3 dpa2; do
 case $m in dpa3) n=7 ;; *) n=3 ;; esac
 ncu --metrics sm__cycles_active.min,sm__cycles_active.avg,sm__cycles_active.max,gpc__cycles_elapsed.max,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__cycles_active.avg,sm__ctas_launched.max,sm__ctas_launched.min \
   --clock-control none --cache-control none -s $((n*4+2)) -c $n --csv --log-file gpurun_out/balance_$m.csv python tools/ncu_target.py $m 2PTC 8 > /dev/null 2>&1
done
python - <<'PY'
import csv,collections
for m in ("dpa3","dpa2"):
    rows=list(csv.DictReader(l for l in open(f"gpurun_out/balance_{m}.csv") if l.startswith('"')))
    d=collections.OrderedDict()
    for r in rows:
        d.setdefault((r["ID"],r["Kernel Name"][:40]),{})[r["Metric Name"]]=r["Metric Value"]
    for k,v in d.items(): print(m,k,{a.split('.',1)[0][:12]+'.'+a.split('.',1)[1][:14]:b for a,b in v.items()})
PY
