# A/B: rows-job size on the cfg4 permutes (rows per job cap x element cap)
b() { python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['permute']['GB_s'], d['phase_ms'])"; }
b r256
TK_LIB_PATH=$PWD/_variants/libtk_r512.so b r512
TK_LIB_PATH=$PWD/_variants/libtk_r1024.so TK_JOB_MAX=16384 b r1024_16k
TK_LIB_PATH=$PWD/_variants/libtk_r1024.so TK_JOB_MAX=32768 b r1024_32k
TK_LIB_PATH=$PWD/_variants/libtk_r512.so TK_JOB_MAX=16384 b r512_16k
