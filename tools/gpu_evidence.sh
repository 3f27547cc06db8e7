# round evidence (round 2): GPU tests, smoke, bench lines (f64 with chains + SVD + e2e + CPU baseline, c64),
# config latencies, SVD, ncu launch list of the bench step, DRAM traffic of the big GEMM, ncu captures
set -x
python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ev_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/ev_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench_f64.json 2> gpurun_out/ev_bench_f64.err; echo "bench rc=$?"
python bench.py --dtype c64 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_bench_c64.json 2> gpurun_out/ev_bench_c64.err; echo "bench c64 rc=$?"
timeout 900 python tools/bench_configs.py --reps 50 --phases --oracle > gpurun_out/ev_configs.jsonl 2> gpurun_out/ev_configs.err; echo "configs rc=$?"
timeout 600 python tools/bench_svd.py --reps 5 --oracle > gpurun_out/ev_svd.jsonl 2> gpurun_out/ev_svd.err; echo "svd rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-chains --no-svd"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-chains --no-svd"
ncu -k regex:gemm_tma_kernel -c 1 --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/ev_traffic_gemm.csv $CMD1 > gpurun_out/ev_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
ncu -k regex:svd_jacobi_panel -c 1 --set full --import-source on --clock-control none -o gpurun_out/ev_svd_panel python tools/svd_blocks.py 181x181 > gpurun_out/ev_ncu_svd.log 2>&1; echo "ncu svd rc=$?"
python tools/prof_chain.py 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/ev_cfg3_launches.csv python tools/prof_chain.py 3 > /dev/null 2>&1; echo "ncu cfg3 rc=$?"
cut -c 1-400 gpurun_out/ev_bench_f64.json gpurun_out/ev_bench_c64.json
