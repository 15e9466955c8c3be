# N>1 bench path dry runs (gloo, ranks sharing the GPU) + the reference arm at N=2
for g in 2 4; do
  BENCH_DD_BACKEND=gloo timeout 600 python bench.py --gpus $g --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/dry_dd_$g.json 2> gpurun_out/dry_dd_$g.err; echo "dd $g rc=$?"
  tail -c 600 gpurun_out/dry_dd_$g.json; echo
done
BENCH_DD_BACKEND=gloo timeout 600 python bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo "ref2 rc=$?"; tail -c 400 gpurun_out/ref2.json
