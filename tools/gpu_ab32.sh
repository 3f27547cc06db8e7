# A/B: seg-job coefficient cached in a register (TK_SEG_CCACHE)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 50 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[0] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run base
TK_LIB_PATH=$PWD/_variants/libtk_cc1.so run ccache
run base2
