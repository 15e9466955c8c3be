# usage: run_bench.sh TAG  — tests + 4 bench configs + warm launch list
TAG=$1
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/tests_$TAG.log 2>&1; tail -1 gpurun_out/tests_$TAG.log
for s in 1YRF 2PTC; do for m in dpa3 dpa2; do
python bench.py --model $m --system $s --no-cpu-baseline --steps 1000 2>&1 | tail -1 > gpurun_out/b_${TAG}_${m}_$s.log
python -c "
import json; d=json.load(open('gpurun_out/b_${TAG}_${m}_$s.log')); print('$m $s', round(d['value']), round(d['ms_per_step']*1e3,1), round(d['warm_l2_graph100']['steps_per_s']), round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done; done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 80 --csv --log-file gpurun_out/launches_${TAG}.csv python tools/ncu_target.py dpa3 1YRF 20 > /dev/null 2>&1
