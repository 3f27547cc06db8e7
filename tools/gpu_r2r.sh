# fused MPO pair (tk_contract2): parity + chain timings fused / unfused + ncu of the fused kernel
cd /root/repo
python -c "import sys; sys.path.insert(0,'paper_2508_10076_b200'); import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_fused.py -q > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2r_pytest.log
for f in "" "--no-fuse"; do
timeout 300 python tools/bench_configs.py --cfgs 2,3 --reps 30 $f 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$f', d['cfg'], d['us_per_chain_graph'], d['launches'], d['calls'])
"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused --csv python tools/prof_chain.py 3 2 > gpurun_out/r2r_ncu.csv 2>&1; echo "ncu rc=$?"
grep fused gpurun_out/r2r_ncu.csv | awk -F'","' '{print $(NF-2), $NF}' | head -12
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/r2r_fused -f python tools/prof_chain.py 3 1 > /dev/null 2>&1; echo "ncu full rc=$?"
