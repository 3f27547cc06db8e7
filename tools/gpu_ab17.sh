# A/B: seg job size cap (TK_SEG_MAX) at the default TK_SEG_DIV = 296
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3,7,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[0] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run max8192
TK_SEG_MAX=16384 run max16384
TK_SEG_MAX=32768 run max32768
