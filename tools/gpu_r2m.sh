python -m pytest tests -m gpu -x -q > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2m_pytest.log
timeout 600 python tools/bench_configs.py --cfgs 1,2,3,5,6,7,8 --reps 30 --phases > gpurun_out/r2m_configs.jsonl 2> gpurun_out/r2m_configs.err; echo "configs rc=$?"
python -c "
import json
for l in open('gpurun_out/r2m_configs.jsonl'):
    d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d.get('phase_us_per_step'))
"
