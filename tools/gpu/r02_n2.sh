set -x
mkdir -p gpurun_out
timeout 300 python tools/api_overhead.py > gpurun_out/api_overhead.json 2> gpurun_out/api_overhead.err
BX_BENCH_TRACE=1 BX_BENCH_ONE_GPU=1 timeout 300 python bench.py --gpus 2 --workload c2 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/n2_c2.json 2> gpurun_out/n2_c2.err
echo "rc=$?"
BX_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/n2_c5.json 2> gpurun_out/n2_c5.err
echo "rc=$?"
cat gpurun_out/api_overhead.json
grep -v "^W1020\|^W10" gpurun_out/n2_c2.err | grep -v "^\[bench" | head -30; tail -c 1200 gpurun_out/n2_c2.json; tail -c 1200 gpurun_out/n2_c5.json
