set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
for w in paper c4p c2p c3; do timeout 300 python bench.py --workload $w --steps 10 --no-cpu > gpurun_out/b_$w.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/b_$w.json').read().splitlines()[-1]);r=d['roofline'];print('$w', round(d['ms_per_step'],4), round(r['frac'],3), d['parity']['mismatches'], d['e2e']['value'])"; done
tail -3 gpurun_out/gputests.log
