# A/B: loads in flight per thread in the rows kernel (TK_ROWS_U) at 512-row jobs
b() { python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['permute']['GB_s'], d['phase_ms'])"; }
b u8
TK_LIB_PATH=$PWD/_variants/libtk_u6.so b u6
TK_LIB_PATH=$PWD/_variants/libtk_u12.so b u12
