# A/B: small-tile GEMM warp tile 32x16 (8 warps, default) vs 32x32 (4 warps) at 4 / 3 CTAs per SM
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run wn16
TK_LIB_PATH=$PWD/_variants/libtk_wn32.so run wn32_m4
TK_LIB_PATH=$PWD/_variants/libtk_wn32m3.so run wn32_m3
TK_LIB_PATH=$PWD/_variants/libtk_wn32.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain" 2>&1 | tail -1
