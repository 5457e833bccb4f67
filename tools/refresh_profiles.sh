#!/bin/bash
# Regenerate the round's evidence on a GPU box (run via gpurun from the repo root):
# bench lines for every config, ncu --set full of every config's extraction
# kernel, and the launch list of the default bench command.  Outputs go to
# gpurun_out/refresh/; copy what is judged into profiles/.
set -u
O=gpurun_out/refresh
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for w in c1 c3 c4 c5_n128 c5_n256 c5_n512 c5_n1024 c5_n2048 c2p c4p paper; do
  python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --impl reference > $O/bench_c2_reference.json 2> $O/bench_c2_reference.err
for w in c2 c3 c4 c5_n128 c5_n256 c5_n512 c5_n1024 c5_n2048 c2p c4p paper; do
  ncu --set full --import-source on --clock-control none -k regex:eq_ --launch-skip 1 --launch-count 1 \
      -o $O/ncu_$w python tools/prof_eq.py --workload $w --launches 1 > $O/ncu_$w.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_launches.log 2>&1
# summaries on the box (full .ncu-rep files are ~7 MB each; gpurun returns <= 64 MiB)
python tools/ncu_summary.py $(for w in c2 c3 c4 c5_n128 c5_n256 c5_n512 c5_n1024 c5_n2048 c2p c4p paper; do echo $O/ncu_$w.ncu-rep:$w; done) \
    --out $O/ncu_kernels > /dev/null
for w in c3 c4 c5_n128 c5_n256 c5_n512 c4p paper; do rm -f $O/ncu_$w.ncu-rep; done
ls $O
