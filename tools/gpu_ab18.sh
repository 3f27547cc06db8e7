# A/B: job size of the recoupling jobs (TK_JOB_DIV jobs per permute)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 5,6,7,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[0] for x in d['phase_us_per_step']], [x[3] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run div1184
TK_JOB_DIV=592 run div592
TK_JOB_DIV=296 run div296
