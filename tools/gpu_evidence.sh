# round evidence: bench lines (f64, c64), config latencies with the oracle, ncu launch list of the bench
python bench.py > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err; echo "bench rc=$?"
python bench.py --dtype c64 --no-cpu-baseline > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err; echo "bench c64 rc=$?"
timeout 900 python tools/bench_configs.py --cfgs 1,2,3,5 --reps 50 --phases --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
cat gpurun_out/bench_f64.json gpurun_out/bench_c64.json gpurun_out/configs.jsonl | cut -c 1-400
