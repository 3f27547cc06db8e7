# A/B: small-tile GEMM with double-buffered DMMA fragments
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run base
TK_LIB_PATH=$PWD/_variants/libtk_fp.so run fragpipe
TK_LIB_PATH=$PWD/_variants/libtk_fp.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k chain 2>&1 | tail -1
