# GEMM tiles carrying their group descriptors (one dependent load per CTA instead of two)
python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
