cd /root/repo
python -c "import sys; sys.path.insert(0,'paper_2508_10076_b200'); import build; build.build()"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/r2u_fused -f python tools/prof_chain.py 3 1 > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gather -c 1 -o gpurun_out/r2u_gather -f env TK_CHAIN_NO_FUSE=1 python tools/prof_chain.py 3 1 > /dev/null 2>&1; echo "ncu full rc=$?"
