# round 2: TMA GEMM correctness + A/B against the cp.async kernel (knob build), bench line with chains
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_capture.py -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a_pytest.log
python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2a_bench_tma.json 2> gpurun_out/r2a_bench_tma.err; echo "bench rc=$?"
TK_LIB_PATH=_variants/libtk_knobs.so TK_NO_TMA=1 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-chains > gpurun_out/r2a_bench_notma.json 2> gpurun_out/r2a_bench_notma.err; echo "bench notma rc=$?"
python -c "
import json
for f in ['r2a_bench_tma','r2a_bench_notma']:
    try:
        d=json.load(open('gpurun_out/'+f+'.json'))
        print(f, d['value'], d['roofline']['achieved'], d['roofline']['peak'], d['roofline']['frac'], d['phase_ms'], d['roofline']['fp64_peaks_this_run'])
    except Exception as e: print(f, 'ERR', e)
"
