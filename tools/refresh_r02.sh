#!/bin/bash
# Round-2 evidence pass on a GPU box (via gpurun from the repo root): the default
# bench line (C5 sweep), the reference arm, planner-shape bench lines, ncu --set
# full of every C5 leg + the planner shapes, and the launch list of the bench
# command.  Outputs under gpurun_out/r02/; tools/refresh_r02_collect.sh copies
# the judged summaries into profiles/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
if [ "${1:-all}" != "ncu" ]; then
python bench.py --impl reference > $O/bench_c5_reference_arm.json 2> $O/bench_ref.err
python bench.py > $O/bench_c5_default.json 2> $O/bench.err
for w in c2p c4p paper c2 c3 c4 c1; do
  python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
fi
[ "${1:-all}" = "bench" ] && exit 0
for w in c5_n128 c5_n256 c5_n512 c5_n1024 c5_n2048 c2p c4p paper; do
  ncu --set full --import-source on --clock-control none -k regex:eq_ --launch-skip 1 --launch-count 1 \
      -o $O/ncu_$w python tools/prof_eq.py --workload $w --launches 1 > $O/ncu_$w.log 2>&1
done
python tools/ncu_summary.py $(for w in c5_n128 c5_n256 c5_n512 c5_n1024 c5_n2048; do echo $O/ncu_$w.ncu-rep:$w; done) \
    --out $O/ncu_c5_kernels > /dev/null
python tools/ncu_summary.py $(for w in c2p c4p paper; do echo $O/ncu_$w.ncu-rep:$w; done) \
    --out $O/ncu_planner_kernels > /dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:eq_ --csv --log-file $O/launches_bench_c5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-warmup 0 > $O/ncu_launches.log 2>&1
python tools/launch_table.py $O/launches_bench_c5.csv "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:eq_ python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-warmup 0" > $O/launches_bench_c5.md
rm -f $O/ncu_c5_n128.ncu-rep $O/ncu_c5_n256.ncu-rep $O/ncu_c5_n512.ncu-rep $O/ncu_paper.ncu-rep $O/ncu_c4p.ncu-rep
ls -la $O
