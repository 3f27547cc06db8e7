# chain parity (fused pair, ncon, chains) + chain timings of the current build
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q -x > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/chk_pytest.log | cut -c1-300
timeout 600 python tools/bench_chains.py 2,3 > gpurun_out/chk_chains.jsonl 2> gpurun_out/chk_chains.err; echo "chains rc=$?"; tail -2 gpurun_out/chk_chains.err
python -c "
import json
for l in open('gpurun_out/chk_chains.jsonl'):
    d=json.loads(l); print(d['cfg'], 'ncon', d['us_per_chain'], d['launches'], 'pairwise', d['us_per_chain_pairwise'], 'roof', d['roofline_us'])
"
python tools/prof_chain.py 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/chk_cfg3_launches.csv python tools/prof_chain.py 3 > /dev/null 2>&1; echo "ncu rc=$?"
grep fused gpurun_out/chk_cfg3_launches.csv | cut -c1-40,150-
