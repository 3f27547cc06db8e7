# A/B: split-K target (tiles per SM) and small-K threshold for the latency configs
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3,7 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run default
TK_SPLIT_TARGET=2 run split2
TK_SPLIT_TARGET=8 run split8
TK_NO_SPLITK=1 run nosplit
TK_GEMM_SMALL_K=512 run smallk512
