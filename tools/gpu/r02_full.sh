# Round-2 full GPU pass: GPU suite, default bench line, launch list of the bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -5 gpurun_out/gputests.log; tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
