set -x
B="python bench.py --d-leg 192 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:permute_kernel.*bool.1" -s 6 -c 1 -o gpurun_out/r01_full_perm_rows $B > gpurun_out/ncu2.log 2>&1; echo "perm rc=$?"
C="python tools/prof_chain.py 3 1"
$C > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:permute_kernel.*bool.0" -s 1 -c 1 -o gpurun_out/r01_full_perm_packed $C > gpurun_out/ncu4.log 2>&1; echo "perm0 rc=$?"
