# ncon left fold + relabel: parity; per-kernel launch lists of the cfg3 chain (unfused / fused / ncon)
cd /root/repo
python -c "import sys; sys.path.insert(0,'paper_2508_10076_b200'); import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2t_pytest.log
for v in "TK_CHAIN_NO_FUSE=1" "TK_CHAIN_X=1" "TK_CHAIN_NCON=1"; do
env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_chain.py 3 2 > gpurun_out/r2t_launch_$v.csv 2>&1
echo "== $v"; python - "gpurun_out/r2t_launch_$v.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
rows = rows[len(rows)//2:]   # second rep
tot = 0
for r in rows:
    t = float(r[-1]) / 1000; tot += t
    print(f"  {t:8.2f} us  {r[4][:90]}")
print(f"  total {tot:.1f} us")
PY
done
