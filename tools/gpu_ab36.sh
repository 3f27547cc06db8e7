# A/B: general permute kernel at 5 CTAs/SM (launch bounds 5) vs 4 on the latency configs
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 50 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'])
  except Exception: pass"
}
run minb4
TK_LIB_PATH=$PWD/_variants/libtk_pm5.so run minb5
