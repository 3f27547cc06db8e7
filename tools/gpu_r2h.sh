for v in default t512 t512l4 l16 l4; do
  if [ $v = default ]; then L=paper_2508_10076_b200/libtk_b200.so; else L=_variants/libtk_$v.so; fi
  echo "== $v"; TK_LIB_PATH=$L timeout 300 python tools/bench_svd.py --reps 3 2>/dev/null | cut -c1-120
done
