# A/B: small-K threshold (K <= small_k -> 64x64 tiles) on the latency configs
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3,7 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run default128
TK_GEMM_SMALL_K=0 run smallk0
TK_GEMM_SMALL_K=32 run smallk32
