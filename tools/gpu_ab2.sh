for v in 2 5 6; do
TK_GEMM_BIG_WARPS=$v python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_v$v.json 2>gpurun_out/bench_v$v.err
python -c "
import json; d=json.load(open('gpurun_out/bench_v$v.json')); print('v$v', d['value'], d['roofline']['frac'], d['phase_ms'])"
done
#TK_GEMM_BIG_WARPS=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
