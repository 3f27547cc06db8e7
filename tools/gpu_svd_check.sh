# SVD parity + timing of the current build (tests/test_gpu_svd.py, tools/bench_svd.py)
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_svd.py -q -x > gpurun_out/svdchk_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/svdchk_pytest.log | cut -c1-300
timeout 300 python tools/bench_svd.py --reps 5 > gpurun_out/svdchk.jsonl 2> gpurun_out/svdchk.err; echo "bench rc=$?"; tail -3 gpurun_out/svdchk.err
TK_SVD_DEBUG=1 timeout 120 python tools/svd_blocks.py 133x133,181x181 2>&1 | sort -u | tail -6
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/svdchk.jsonl") if l.startswith("{")]
print([(r["case"][:12], r["us_svd"]) for r in rows])
PY
