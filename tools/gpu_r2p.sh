python tools/prof_chain.py 3 2 > /dev/null 2>&1
ncu --kernel-name-base demangled -k "regex:gather_skinny_kernel" -c 1 --set full --import-source on -o gpurun_out/r2p_gather python tools/prof_chain.py 3 1 > gpurun_out/r2p_ncu1.log 2>&1; echo "ncu gather rc=$?"
ncu -k regex:gemm_small_kernel -c 1 --set full --import-source on -o gpurun_out/r2p_small python tools/prof_chain.py 3 1 > gpurun_out/r2p_ncu2.log 2>&1; echo "ncu small rc=$?"
