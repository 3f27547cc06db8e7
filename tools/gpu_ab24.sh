# group leg table in shared memory for the rows decode: cfg4 permutes + parity of the permute paths
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('smemlegs', d['value'], d['permute']['GB_s'], d['phase_ms'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or permute" 2>&1 | tail -1
python tools/bench_configs.py --reps 30 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'])
  except Exception: pass"
