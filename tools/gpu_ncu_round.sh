# ncu --set full captures of the kernels the round's numbers come from (each command first runs clean)
set -x
B="python bench.py --d-leg 192 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_mbar -s 3 -c 1 -o gpurun_out/r01_full_gemm $B > gpurun_out/ncu1.log 2>&1; echo "gemm rc=$?"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"permute_kernel" -s 9 -c 1 -o gpurun_out/r01_full_perm_rows $B > gpurun_out/ncu2.log 2>&1; echo "perm rc=$?"
C="python tools/prof_chain.py 3 1"
$C > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"gemm_skinny" -c 1 -o gpurun_out/r01_full_skinny $C > gpurun_out/ncu3.log 2>&1; echo "skinny rc=$?"
ls -la gpurun_out/*.ncu-rep
