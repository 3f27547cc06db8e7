# A/B: permute CTA size 256 (default) vs 128 / 512 threads on the cfg4 permutes and the latency configs
b() { python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['permute']['GB_s'], d['phase_ms'])"; }
c() { python tools/bench_configs.py --reps 30 --cfgs 2,3,7 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print('$1', d['cfg'], d['us_per_chain_graph'])
  except Exception: pass"; }
b t256; c t256
export TK_LIB_PATH=$PWD/_variants/libtk_t128.so; b t128; c t128
export TK_LIB_PATH=$PWD/_variants/libtk_t512.so; b t512; c t512
