set -x
mkdir -p gpurun_out
timeout 300 python tools/api_overhead.py > gpurun_out/api_overhead.json 2> gpurun_out/api_overhead.err
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
BX_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -x -k "not c5_fullsize and not fullsize" > gpurun_out/gputests_checked.log 2>&1
echo "checked rc=$?"
cat gpurun_out/api_overhead.json; tail -3 gpurun_out/gputests.log; tail -3 gpurun_out/gputests_checked.log
