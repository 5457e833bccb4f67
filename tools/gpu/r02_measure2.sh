# round-2 final measurement pass: bench line, reference arm, launch list, ncu --set full of every C5 leg
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-warmup 0 > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:eq_direct_kernel -s 15 -c 5 -o gpurun_out/ncu_c5_r02 -f python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --e2e-warmup 0 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
for w in pack_b1 pack_b6 pack_b12 pack_b14 c3w paper; do timeout 300 python bench.py --workload $w --cpu-seconds 4 > gpurun_out/bench_$w.json 2>/dev/null; done
ls gpurun_out
