# A/B: gathered skinny GEMM (A~ permute folded into the T.W GEMM) vs permute + skinny; parity first
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain" 2>&1 | tail -2
run() {
  echo "== $1"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d['phase_us_per_step'])
  except Exception: print(l.rstrip()[:300])"
}
run gather
TK_NO_GATHER=1 run nogather
