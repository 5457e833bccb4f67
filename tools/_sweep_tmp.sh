cd $GRAFT_REPO_ROOT
python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
for w in c5_n1024; do
 for t in 1 2 4 8; do
  echo -n "$w tpb16=$t "; BX_DIRECT16_TPB=$t timeout 120 python tools/prof_eq.py --workload $w --launches 10 2>&1 | tail -1 | sed 's/, .family.*//'
 done
done
for n in 16 32 128 256; do
 for t in 1 8; do
  echo -n "q16 n=$n tpb16=$t "; BX_DIRECT16_TPB=$t timeout 120 python tools/prof_eq.py --q 16 --n $n --blocks $((2**35 / (32*n))) --launches 10 2>&1 | tail -1 | sed 's/, .family.*//'
 done
done
