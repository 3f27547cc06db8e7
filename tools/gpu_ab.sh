# A/B: GEMM big-tile variants (8 vs 16 warps) + permute; then parity tests
set -x
TK_PERM_TILE_ALL=1 TK_GEMM_BIG_WARPS=16 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_w16.json 2>gpurun_out/bench_w16.err
TK_GEMM_BIG_WARPS=16 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_w8.json 2>gpurun_out/bench_w8.err
for f in gpurun_out/bench_w16.json gpurun_out/bench_w8.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['phase_ms'], d['permute']['GB_s'], [ (k,v['GB_s']) for k,v in d['permute']['phases'].items()])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
