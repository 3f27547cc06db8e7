# A/B: big-GEMM rasterisation band (cfg4) and skinny-tile rows (cfg7 / cfg8 W-steps)
b() { python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['frac'], d['phase_ms']['gemm'])"; }
b band12
TK_GEMM_BAND=24 b band24
TK_GEMM_BAND=48 b band48
b band12again
c() { python tools/bench_configs.py --reps 50 --phases --cfgs 2,3,7,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print('$1', d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: pass"; }
c rows2048
TK_SKINNY_ROWS=1024 c rows1024
TK_SKINNY_ROWS=512 c rows512
