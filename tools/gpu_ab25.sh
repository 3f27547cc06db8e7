# A/B: prefetch distance of the big-tile GEMM's 6-stage ring (2 default / 3 / 4) on cfg4
b() { python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['phase_ms']['gemm'])"; }
b pd2
TK_LIB_PATH=$PWD/_variants/libtk_pd3.so b pd3
TK_LIB_PATH=$PWD/_variants/libtk_pd4.so b pd4
b pd2again
