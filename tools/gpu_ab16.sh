# A/B: gathered GEMM rows per thread 2 (default) vs 4 (1024-row tiles)
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run default
TK_LIB_PATH=$PWD/_variants/libtk_rpt4.so run rpt4
timeout 900 python -m pytest tests/test_gpu_edge.py -q -k gather 2>&1 | tail -1
TK_LIB_PATH=$PWD/_variants/libtk_rpt4.so timeout 900 python -m pytest tests/test_gpu_edge.py -q -k gather 2>&1 | tail -1
