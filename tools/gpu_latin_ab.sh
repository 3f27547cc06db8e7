# A/B: Latin-square warp -> sub-tile mapping of the DMMA GEMM kernels (default build) against the old
# wm = warp % WARPS_M mapping (_variants/libtk_nolatin.so, built with tools/build_variant.sh nolatin
# "-DTK_WARP_LATIN=0"): parity of the default build first, then the bench line (cfg4 GEMM phase, chains)
# alternating between the two libraries.
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fused.py -m gpu -q -x > gpurun_out/latin_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/latin_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-svd"
for r in 1 2; do
  $B > gpurun_out/latin_new_$r.json 2> gpurun_out/latin_new_$r.err; echo "new rc=$?"
  TK_LIB_PATH=_variants/libtk_nolatin.so $B > gpurun_out/latin_old_$r.json 2> gpurun_out/latin_old_$r.err; echo "old rc=$?"
done
python - <<'PY'
import json
for n in ("new_1", "old_1", "new_2", "old_2"):
    d = json.loads(open(f"gpurun_out/latin_{n}.json").read().strip().splitlines()[-1])
    print(n, d["value"], d["phase_ms"]["gemm"], d["roofline"]["frac"], {k: v["us_per_chain"] for k, v in d["chains"].items()})
PY
