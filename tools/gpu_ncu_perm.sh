CMD2="python bench.py --d-leg 192 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:permute -s 6 -c 4 -o gpurun_out/prof_perm_r01c $CMD2 > gpurun_out/ncu_full_perm.log 2>&1; echo "ncu perm rc=$?"
