set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_capi.py tests/test_gpu_parity.py -q -x > gpurun_out/t_wide.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --workload c3w --steps 10 > gpurun_out/bench_c3w.json 2> gpurun_out/bench_c3w.err
echo "bench rc=$?"
timeout 600 python bench.py --workload c3 --steps 10 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eq_wide256 -s 3 -c 1 -o gpurun_out/ncu_c3w -f python bench.py --workload c3w --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c3w.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/t_wide.log; tail -c 1500 gpurun_out/bench_c3w.json; tail -5 gpurun_out/bench_c3w.err; python -c "import json;d=json.loads(open('gpurun_out/bench_c3.json').read().splitlines()[-1]);print('c3 mapped',d['value'],d['ms_per_step'])"
