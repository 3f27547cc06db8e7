# A/B: persistent small-tile GEMM (default) vs one tile per CTA (TK_GEMM_NO_PERS=1), then parity
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run pers
TK_GEMM_NO_PERS=1 run nopers
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
