set -x
timeout 900 python -m pytest tests/test_gpu_svd.py -x -q > gpurun_out/r2d_svd_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2d_svd_pytest.log
timeout 600 python tools/bench_svd.py --reps 5 --oracle > gpurun_out/r2d_svd.jsonl 2> gpurun_out/r2d_svd.err; echo "svd bench rc=$?"; cat gpurun_out/r2d_svd.jsonl; tail -3 gpurun_out/r2d_svd.err
