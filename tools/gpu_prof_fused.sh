# ncu --set full of the cfg3 chain's fused MPO pair kernel and small-tile GEMMs (round-2 chain analysis)
cd /root/repo
python tools/prof_chain.py 3 > /dev/null 2>&1; echo "plain rc=$?"
timeout 600 ncu -k regex:"fused_pair|gemm_small" -c 3 --set full --import-source on --clock-control none -o gpurun_out/fused_full python tools/prof_chain.py 3 > gpurun_out/fused_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/fused_ncu.log
