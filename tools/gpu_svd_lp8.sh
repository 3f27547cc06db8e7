# SVD panel kernel: 16 vs 32 lanes per pair (parity + timing)
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_svd.py -q -x > gpurun_out/svdlp8_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/svdlp_pytest.log | cut -c1-300
for lp in 8 16; do echo "== LP $lp"; TK_LIB_PATH=_variants/libtk_knobs8.so TK_SVD_LP=$lp timeout 300 python tools/bench_svd.py --reps 5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['case'][:14], d['us_svd'])"
TK_LIB_PATH=_variants/libtk_knobs8.so TK_SVD_LP=$lp TK_SVD_DEBUG=1 timeout 120 python tools/svd_blocks.py 133x133,181x181 2>&1 | sort -u | tail -4; done
