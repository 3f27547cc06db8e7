timeout 900 python -m pytest tests/test_gpu_svd.py -x -q > gpurun_out/r2e_svd_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_svd_pytest.log
TK_SVD_DEBUG=1 timeout 300 python tools/bench_svd.py --reps 1 > /dev/null 2> gpurun_out/r2e_svd.err; echo "svd dbg rc=$?"
grep "x 1[0-9][0-9]\|x 9[0-9]\|x 6[0-9]" gpurun_out/r2e_svd.err | sort | uniq | head -20
timeout 300 python tools/bench_svd.py --reps 5 > gpurun_out/r2e_svd.jsonl 2>/dev/null; echo "svd rc=$?"
cut -c1-150 gpurun_out/r2e_svd.jsonl
