# Packer (bx_pack) parity + bench + ncu
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_parity.py tests/test_gpu_sources.py -q -x > gpurun_out/t_pack.log 2>&1
echo "pytest rc=$?"
for w in pack_b1 pack_b6 pack_b12 pack_b14; do
  timeout 300 python bench.py --workload $w --cpu-seconds 4 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pack --csv --log-file gpurun_out/ncu_pack_launches.csv python bench.py --workload pack_b6 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_pack.log 2>&1
for w in pack_b1 pack_b6 pack_b12 pack_b14; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_tile -s 3 -c 1 -o gpurun_out/ncu_$w python bench.py --workload $w --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full_$w.log 2>&1
done
tail -5 gpurun_out/t_pack.log; for w in pack_b1 pack_b6 pack_b12 pack_b14; do tail -c 600 gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err; done
