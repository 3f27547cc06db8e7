# A/B: skinny GEMM at 3 CTAs/SM (launch bounds 3) vs 2 (82 registers), cfg7 / cfg8 W-steps
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 50 --phases --cfgs 7,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: pass"
}
run minb1
TK_LIB_PATH=$PWD/_variants/libtk_sk3.so run minb3
