mkdir -p gpurun_out
for w in c2p c4p paper; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eq_ -s 1 -c 1 -o gpurun_out/ncu_$w -f python tools/prof_eq.py --workload $w --launches 2 > gpurun_out/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
