for r in 1 2 3; do
for v in default q8m5 q8m6; do
  if [ $v = default ]; then L=""; else L=$PWD/_exp/$v/libbx_b200.so; fi
  echo -n "$v c5_n512 r$r: "; BX_LIB=$L timeout 300 python tools/prof_eq.py --workload c5_n512 --launches 20 2>/dev/null | cut -c1-70
done
done
