set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench rc=$?"
tail -2 gpurun_out/gputests.log
python -c "
import json;d=json.loads(open('gpurun_out/bench_c5.json').read().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],d['clocks'],'e2e',d['e2e']['value'])
for s in d['sweep']: print(s['workload'], round(s['ms_per_launch'],3), round(s['raw_gbps']), round(s['frac'],3))
print(d['parity'], d['cpu_baseline']['value'])"
