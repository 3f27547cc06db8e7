# small-tile GEMM residency after the instruction cut: default (128 registers, 2 CTAs/SM) against
# _variants/libtk_minb3.so (-DTK_SMALL_MINB=3: 80 registers, 8 B spilled) and libtk_minb4.so (64 registers,
# 312 B spilled); pairwise chains with per-phase GEMM times, then the tk_ncon chains
for v in default minb3 minb4 default minb3; do
  if [ $v = default ]; then unset TK_LIB_PATH; else export TK_LIB_PATH=_variants/libtk_$v.so; fi
  python tools/bench_configs.py --cfgs 2,3,7,8 --reps 30 --phases 2>/dev/null | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('$v', {r['cfg']: (r['us_per_chain_graph'], [p[2] for p in r['phase_us_per_step']]) for r in rows})"
done
for v in default minb3 default minb3; do
  if [ $v = default ]; then unset TK_LIB_PATH; else export TK_LIB_PATH=_variants/libtk_$v.so; fi
  python tools/bench_chains.py 2,3,5,6,7,8 2>/dev/null | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('ncon $v', {r['cfg']: (r['us_per_chain'], r['us_per_chain_pairwise']) for r in rows})"
done
