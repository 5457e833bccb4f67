mkdir -p gpurun_out
for w in c4p paper; do
  for kb in 24 36 48 72 96; do
    BX_TMA_BUDGET_KB=$kb timeout 300 python bench.py --workload $w --steps 10 --no-cpu --e2e-steps 1 --e2e-warmup 0 > gpurun_out/tma_${w}_${kb}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/tma_${w}_${kb}.json').read().splitlines()[-1]);r=d['roofline'];print('$w', $kb, round(d['ms_per_step'],4), round(r['frac'],3), r['launch'], d['parity']['mismatches'])"
  done
done
