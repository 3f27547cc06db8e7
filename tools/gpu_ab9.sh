# A/B: small-GEMM pipeline depth (3 default / 4 / 5 stages)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run st3
TK_LIB_PATH=$PWD/_variants/libtk_st4.so run st4
TK_LIB_PATH=$PWD/_variants/libtk_st5.so run st5
