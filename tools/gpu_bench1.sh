set -x
python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; echo "bench rc=$?"
cat gpurun_out/bench_r01a.json
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01a.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD2="python bench.py --d-leg 192 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_big -s 2 -c 1 -o gpurun_out/prof_gemm_r01a $CMD2 > gpurun_out/ncu_full_gemm.log 2>&1; echo "ncu gemm rc=$?"
$CMD2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:permute -s 6 -c 3 -o gpurun_out/prof_perm_r01a $CMD2 > gpurun_out/ncu_full_perm.log 2>&1; echo "ncu perm rc=$?"
ls -la gpurun_out
