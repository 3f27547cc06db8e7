CMD2="python bench.py --d-leg 192 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_big -s 2 -c 1 -o gpurun_out/prof_gemm_$1 $CMD2 > gpurun_out/ncu_full_gemm.log 2>&1; echo "ncu gemm rc=$?"
