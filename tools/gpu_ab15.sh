# A/B: gathered GEMM occupancy (launch bounds 3 / 5 / 6) and tile rows (256 / 512)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run default
TK_GATHER_ROWS=256 run rows256
TK_LIB_PATH=$PWD/_variants/libtk_gm5.so TK_GATHER_ROWS=256 run gm5_256
TK_LIB_PATH=$PWD/_variants/libtk_gm6.so TK_GATHER_ROWS=256 run gm6_256
TK_LIB_PATH=$PWD/_variants/libtk_gm5.so run gm5_512
