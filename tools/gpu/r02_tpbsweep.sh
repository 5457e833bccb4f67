# tpb target x TMA budget sweep for the planner shapes (A/B; tools/gpu/r02_tpbsweep.sh)
mkdir -p gpurun_out/tpb
for w in c4p paper; do
  for tg in 8 16 32; do
    for kb in 72 112 160 200; do
      f=gpurun_out/tpb/${w}_${tg}_${kb}.json
      BX_TPB_TARGET=$tg BX_TMA_BUDGET_KB=$kb timeout 300 python bench.py --workload $w --steps 10 --no-cpu --e2e-steps 1 --e2e-warmup 0 > $f 2>/dev/null
      python -c "import json;d=json.loads(open('$f').read().splitlines()[-1]);r=d['roofline'];print('$w', 'target', $tg, 'kb', $kb, round(d['ms_per_step'],4), round(r['frac'],3), r['launch'], d['parity']['mismatches'])"
    done
  done
done 2>&1 | tee gpurun_out/tpb/sweep.txt
