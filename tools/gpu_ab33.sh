# gathered GEMM with general coefficients and recoupled subblocks from the workspace (cfg7 / cfg8 W-steps)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_ncon.py -q -x 2>&1 | tail -2
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 50 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d['phase_us_per_step'])
  except Exception: print(l.rstrip()[:300])"
}
run hybrid
