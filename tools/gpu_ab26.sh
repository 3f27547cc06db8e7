# A/B: big-tile GEMM k-step (BK 16 x 6 stages, prefetch 2) vs BK 32 x 3 stages (prefetch 1 / 2)
b() { python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['phase_ms']['gemm'])"; }
b bk16
TK_LIB_PATH=$PWD/_variants/libtk_bk32.so b bk32_s3_pd1
TK_LIB_PATH=$PWD/_variants/libtk_bk32s3p2.so b bk32_s3_pd2
