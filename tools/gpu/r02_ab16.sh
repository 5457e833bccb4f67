mkdir -p gpurun_out
for r in 1 2 3; do
for v in default pf16 pf16c4 c4only; do
  if [ $v = default ]; then L=""; else L=$PWD/_exp/$v/libbx_b200.so; fi
  for w in c5_n1024; do
    echo -n "$v $w r$r: "; BX_LIB=$L timeout 300 python tools/prof_eq.py --workload $w --launches 20 2>/dev/null | cut -c1-80
  done
done
done
# correctness of the winner candidates on the full suite of direct variants
BX_LIB=$PWD/_exp/pf16c4/libbx_b200.so timeout 600 python -m pytest tests/test_gpu_direct_variants.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
