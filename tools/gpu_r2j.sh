python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_capture.py -x -q > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2j_pytest.log
python bench.py --steps 10 --warmup 3 --e2e-steps 4 --no-cpu-baseline > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2j_bench.err
python -c "
import json
d=json.load(open('gpurun_out/r2j_bench.json'))
print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['phase_ms'], d['e2e'])
for k,v in (d.get('chains') or {}).items(): print(k, v['us_per_chain'], v['roofline_frac'])
"
CMD1="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-chains"
ncu -k regex:gemm_tma_kernel -c 1 --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r2j_traffic_gemm.csv $CMD1 > gpurun_out/r2j_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"; grep -o '"dram__bytes_[a-z]*.sum","byte","[0-9]*"' gpurun_out/r2j_traffic_gemm.csv
