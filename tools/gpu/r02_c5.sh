set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_c5_fullsize.py -x -q 2>&1 | tail -15 > gpurun_out/t_c5.log
timeout 600 python -m pytest tests/test_gpu_peer_gather.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15 > gpurun_out/t_par.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -3 gpurun_out/t_c5.log gpurun_out/t_par.log; tail -c 3000 gpurun_out/bench_c5.json; tail -20 gpurun_out/bench_c5.err
