# A/B: seg variants on the latency configs
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[0] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run general
TK_SEG_DSTLEG=1 run general-dstleg
TK_SEG_PERSIST=1 TK_SEG_DIV=1776 run persist
TK_NO_SEG=1 run noseg
