# GEMM tile rasterisation band vs DRAM traffic and time (cfg4 D_leg 384, gemm_tma_kernel)
cd /root/repo
for band in ${BANDS:-1 2 3 4}; do
  echo "== band $band"
  TK_LIB_PATH=_variants/libtk_knobs.so TK_GEMM_BAND=$band timeout 600 ncu -k regex:gemm_tma_kernel -c 1 --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-chains --no-svd 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
  TK_LIB_PATH=_variants/libtk_knobs.so TK_GEMM_BAND=$band timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-chains --no-svd | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TFLOP/s', d['roofline']['achieved'], d['roofline']['frac'])"
done
