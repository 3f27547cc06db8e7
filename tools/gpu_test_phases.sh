python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python tools/bench_configs.py --cfgs 1,2,3,5 --phases --reps 20 > gpurun_out/phases.jsonl 2>&1; echo "rc=$?"; cat gpurun_out/phases.jsonl
