for r in 1 2 3; do
for v in default u2bpt2 u2bpt4; do
  if [ $v = default ]; then L=""; else L=$PWD/_exp/$v/libbx_b200.so; fi
  for w in c5_n256 c5_n128; do
  echo -n "$v $w r$r: "; BX_LIB=$L timeout 300 python tools/prof_eq.py --workload $w --launches 20 2>/dev/null | cut -c1-75
  done
done
done
timeout 900 python -m pytest tests/test_gpu_direct_variants.py tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x 2>&1 | tail -1
for v in u2bpt2 u2bpt4; do BX_LIB=$PWD/_exp/$v/libbx_b200.so timeout 600 python -m pytest tests/test_gpu_direct_variants.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done
