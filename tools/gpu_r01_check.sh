set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo "bench rc=$?"; cat gpurun_out/bench_h.json
timeout 600 python tools/bench_configs.py > gpurun_out/configs_h.jsonl 2> gpurun_out/configs_h.err; echo "configs rc=$?"; cat gpurun_out/configs_h.jsonl
