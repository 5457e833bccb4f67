for r in 1 2 3 4; do
for v in default splitimad; do
  if [ $v = default ]; then L=""; else L=$PWD/_exp/$v/libbx_b200.so; fi
  echo -n "$v c5_n1024 r$r: "; BX_LIB=$L timeout 300 python tools/prof_eq.py --workload c5_n1024 --launches 20 2>/dev/null | cut -c1-72
done
done
BX_LIB=$PWD/_exp/splitimad/libbx_b200.so timeout 600 python -m pytest tests/test_gpu_direct_variants.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
