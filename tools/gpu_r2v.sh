# gather output-permute fold + ncon relabel: parity; chains ncon vs pairwise
cd /root/repo
python -c "import sys; sys.path.insert(0,'paper_2508_10076_b200'); import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2v_pytest.log
timeout 600 python tools/bench_chains.py 2,3,5,6,7,8 > gpurun_out/r2v_chains.jsonl 2> gpurun_out/r2v_chains.err
python -c "
import json
for l in open('gpurun_out/r2v_chains.jsonl'):
    d=json.loads(l); print(d['cfg'], 'ncon', d['us_per_chain'], d['launches'], 'pairwise', d['us_per_chain_pairwise'], d['launches_pairwise'], 'roof', d['roofline_us'])
"
