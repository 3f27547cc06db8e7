# A/B: ComplexF64 rows-only permute instances at 5 CTAs/SM vs 4
b() { python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --dtype c64 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['permute']['GB_s'], d['phase_ms'])"; }
b c_minb4
TK_LIB_PATH=$PWD/_variants/libtk_rc5.so b c_minb5
