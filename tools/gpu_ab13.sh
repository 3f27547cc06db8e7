# A/B: recoupling groups of <= 4 sources inside the general permute launch vs their own launch
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_anyon.py tests/test_gpu_trace.py -q -x 2>&1 | tail -1
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d['phase_us_per_step'])
  except Exception: print(l.rstrip()[:300])"
}
run direct
TK_NO_DIRECT_MULTI=1 run separate
