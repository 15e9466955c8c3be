for mode in dd dd-gather; do for g in 2 4; do
  BENCH_DD_BACKEND=gloo timeout 600 python bench.py --gpus $g --steps 30 --warmup 3 --mode $mode --no-cpu-baseline > gpurun_out/dry_${mode}_$g.json 2> gpurun_out/dry_${mode}_$g.err
  python -c "import json; d=json.load(open('gpurun_out/dry_${mode}_$g.json')); print('$mode', $g, round(d['value'],1), round(d['ms_per_step'],3), d['halo'], d['extensivity']['rel_diff'])"
done; done
