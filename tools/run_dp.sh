# DeePMD-style families: GPU parity tests + short benches (usage: bash tools/run_dp.sh [models] [systems])
MODELS=${1:-"se_a repformer"}
SYSTEMS=${2:-"1YRF 2PTC"}
timeout 900 python -m pytest tests/test_dpfamily.py -x -q -m gpu > gpurun_out/dp_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/dp_tests.log
for m in $MODELS; do for sys in $SYSTEMS; do
timeout 300 python bench.py --model $m --system $sys --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/b_${m}_${sys}.json 2> gpurun_out/b_${m}_${sys}.err
python -c "import json;d=json.load(open('gpurun_out/b_${m}_${sys}.json'));print('$m $sys',round(d['value']),round(d['warm_l2_graph100']['steps_per_s']),{k:round(v,1) for k,v in d['kernels_us'].items()},round(d['roofline']['frac'],4),round(d['e2e']['value']))" || tail -5 gpurun_out/b_${m}_${sys}.err
done; done
