# ncu --set full of the cfg3 chain through tk_ncon (second repetition: launches 5..9 of the tk kernels):
# the two gemm_small_kernel launches (L.theta, T3.R), the fused MPO pair and the permutes
set -x
TK_CHAIN_NCON=1 python tools/prof_chain.py 3 2 > /dev/null 2>&1 || exit 1
TK_CHAIN_NCON=1 ncu -k regex:"gemm_small_kernel|fused_pair_kernel|permute_kernel" -s 5 -c 5 --set full --import-source on \
  --clock-control none -o gpurun_out/r02_cfg3_ncon python tools/prof_chain.py 3 2 > gpurun_out/prof_ncon3.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r02_cfg3_ncon.ncu-rep --page raw --csv > gpurun_out/r02_cfg3_ncon_raw.csv 2>/dev/null
