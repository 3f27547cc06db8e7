python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_g.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_g.json')); print(d['value'], d['roofline']['frac'], d['phase_ms'], d['clocks'])"
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_t.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none -k regex:gemm_mbar -s 1 -c 1 --csv --log-file gpurun_out/ncu_traffic_r01.csv $CMD > gpurun_out/ncu_t.log 2>&1; echo "ncu rc=$?"; cut -d, -f13- gpurun_out/ncu_traffic_r01.csv | tail -5
