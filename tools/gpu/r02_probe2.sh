set -x
mkdir -p gpurun_out
./tools/microbench/tmem_ld > gpurun_out/tmem_ld.txt 2>&1
timeout 300 python tools/api_overhead.py > gpurun_out/api_overhead.json 2> gpurun_out/api_overhead.err
BX_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/bench_n2_functional.json 2> gpurun_out/bench_n2_functional.err
echo "n2 rc=$?"
cat gpurun_out/tmem_ld.txt gpurun_out/api_overhead.json; tail -c 1500 gpurun_out/bench_n2_functional.json; tail -20 gpurun_out/bench_n2_functional.err
