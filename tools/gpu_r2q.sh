python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q_pytest.log
timeout 300 python tools/bench_configs.py --cfgs 2,3 --reps 30 --phases 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d.get('phase_us_per_step'))
"
