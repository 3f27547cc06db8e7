# A/B: skinny GEMM variants (templated per launch; MINB 4 build; staged)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run templated
TK_LIB_PATH=$PWD/_variants/libtk_sk2.so run minb2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
