set -x
mkdir -p gpurun_out
for v in default wide4; do
  if [ $v = default ]; then L=""; else L=$PWD/_exp/$v/libbx_b200.so; fi
  for r in 1 2; do
    BX_LIB=$L timeout 600 python bench.py --workload c3w --steps 20 --no-cpu > gpurun_out/ab_${v}_${r}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_${r}.json').read().splitlines()[-1]);print('$v', d['ms_per_step'], d['parity'])"
  done
done
