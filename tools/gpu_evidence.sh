# round evidence: GPU tests, smoke, bench lines (f64, c64), config latencies, SVD, ncu launch list
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err; echo "bench rc=$?"
python bench.py --dtype c64 --no-cpu-baseline > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err; echo "bench c64 rc=$?"
timeout 900 python tools/bench_configs.py --reps 50 --phases --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 600 python tools/bench_svd.py --oracle > gpurun_out/svd.jsonl 2> gpurun_out/svd.err; echo "svd rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
cut -c 1-300 gpurun_out/bench_f64.json gpurun_out/bench_c64.json
