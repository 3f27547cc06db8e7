# A/B: persistent gathered GEMM (default) vs one tile per CTA (TK_GATHER_SIMPLE=1); parity first
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "chain or gather" 2>&1 | tail -1
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases --cfgs 2,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])
  except Exception: print(l.rstrip()[:300])"
}
run pers
TK_GATHER_SIMPLE=1 run simple
