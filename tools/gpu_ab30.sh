# gathered GEMM with per-tile descriptor slots: parity, then cfg2 / cfg3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_ncon.py -q -x 2>&1 | tail -1
python tools/bench_configs.py --reps 50 --phases --cfgs 2,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
