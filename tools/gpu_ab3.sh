# A/B: small-GEMM occupancy variants on the latency configs
for v in default s3m2 s2m4; do
  if [ $v = default ]; then unset TK_LIB_PATH; else export TK_LIB_PATH=$PWD/_variants/libtk_$v.so; fi
  echo "== $v"
  python tools/bench_configs.py --reps 30 --phases 2>&1 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], [x[2] for x in d['phase_us_per_step']])"
done
