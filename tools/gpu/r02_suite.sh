# full GPU suite + pipe throughput
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
timeout 600 python tools/pipe_bw.py > gpurun_out/pipe_bw.json 2> gpurun_out/pipe_bw.err
BX_PIPE_THREADS=0 timeout 600 python tools/pipe_bw.py > gpurun_out/pipe_bw_t0.json 2>> gpurun_out/pipe_bw.err
tail -4 gpurun_out/gputests.log; cat gpurun_out/pipe_bw.json gpurun_out/pipe_bw_t0.json; tail -3 gpurun_out/pipe_bw.err
