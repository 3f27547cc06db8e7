set -x
python bench.py --dtype c64 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2c_bench_c64.json 2> gpurun_out/r2c_bench_c64.err; echo "c64 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-chains"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv $CMD > gpurun_out/r2c_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-chains"
ncu -k regex:gemm_tma_kernel -c 1 --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum --csv --log-file gpurun_out/r2c_traffic_gemm.csv $CMD1 > gpurun_out/r2c_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
ncu -k regex:gemm_tma_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/r2c_gemm_full python bench.py --d-leg 192 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-chains > gpurun_out/r2c_ncu_full.log 2>&1; echo "ncu full rc=$?"
