# small-tile GEMM ring depth after the instruction-count cut: default (BK 16 x 3 stages) against 4 / 5 stages
# and BK 32 x 3 stages (_variants/libtk_st4.so, libtk_st5.so, libtk_bk32.so); chains + per-phase GEMM times
for v in default st4 st5 bk32 default st4 bk32; do
  if [ $v = default ]; then unset TK_LIB_PATH; else export TK_LIB_PATH=_variants/libtk_$v.so; fi
  python tools/bench_configs.py --cfgs 2,3,7,8 --reps 30 --phases 2>/dev/null | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('$v', {r['cfg']: (r['us_per_chain_graph'], [p[2] for p in r['phase_us_per_step']]) for r in rows})"
done
