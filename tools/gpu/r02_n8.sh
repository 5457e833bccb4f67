mkdir -p gpurun_out
BX_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/n8_c5.json 2> gpurun_out/n8_c5.err
echo "n8 c5 rc=$?"
BX_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 4 --workload c2 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/n4_c2.json 2> gpurun_out/n4_c2.err
echo "n4 c2 rc=$?"
for f in n8_c5 n4_c2; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().splitlines()[-1]);print('$f', d['n_gpus'], d['value'], d['parity'], d['e2e']['error'], d['e2e']['bit_exact_vs_device_run'], d['config']['blocks_this_rank0'])"; done
grep -v "^W10" gpurun_out/n8_c5.err | tail -5
