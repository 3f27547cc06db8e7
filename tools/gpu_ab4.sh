# A/B: seg jobs (default) vs TK_NO_SEG=1 on the latency configs, then parity
for v in seg noseg; do
  if [ $v = noseg ]; then export TK_NO_SEG=1; else unset TK_NO_SEG; fi
  echo "== $v"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['phase_us_per_step'])
  except Exception: print(l.rstrip())"
done
unset TK_NO_SEG
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
