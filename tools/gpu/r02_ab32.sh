mkdir -p gpurun_out
for r in 1 2 3; do
for v in base16 pf32; do
  L=$PWD/_exp/$v/libbx_b200.so
  for w in c5_n2048 c1 c3; do
    echo -n "$v $w r$r: "; BX_LIB=$L timeout 300 python tools/prof_eq.py --workload $w --launches 20 2>/dev/null | cut -c1-80
  done
done
done
BX_LIB=$PWD/_exp/pf32/libbx_b200.so timeout 600 python -m pytest tests/test_gpu_direct_variants.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
