# A/B: minimum split-K slice (64 default / 32 / 16 k) on the latency configs
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 50 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run chunk64
TK_SPLIT_CHUNK=32 run chunk32
TK_SPLIT_CHUNK=16 run chunk16
