"""Register / spill budget of the hot kernels, read from the built library with cuobjdump (no GPU needed).

Occupancy is part of these kernels' design: the cfg4 rows-only permute must fit
40 registers (6 CTAs of 256 threads per SM: 5.41 TB/s; 48 registers / 5 CTAs: 5.24; 56 / 4: 4.62), at the
price of one spilled word; the big-tile GEMMs (TMA and cp.async) 128 (one 512-thread CTA per SM) without
spills; the
latency-path kernels at most a word or two (the general permute kernel carries every small-permute job
type under the 64-register cap of 4 CTAs per SM).
"""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2508_10076_b200",
                   "libtk_b200.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

BUDGET = {  # demangled-name prefix -> (max registers, max stack bytes)
    "void tk::permute_kernel<0, true>": (40, 8),
    "void tk::gemm_mbar_kernel<2>": (128, 0),
    "tk::gemm_small_kernel": (128, 0),
    "tk::gemm_tma_kernel": (128, 0),
    "tk::gemm_skinny_kernel": (85, 0),
    "void tk::permute_kernel<0, false>": (64, 16),
    "void tk::gather_skinny_kernel<8, 8>": (85, 0),
    "void tk::fused_pair_kernel<8>": (80, 0),
    "void tk::permute_recouple_kernel<0>": (85, 0),
}


def _resources():
    if not os.path.exists(LIB) or not os.path.exists(CUOBJDUMP):
        pytest.skip("library or cuobjdump not available")
    out = subprocess.run([CUOBJDUMP, "-res-usage", LIB], capture_output=True, text=True).stdout
    demangled = subprocess.run(["c++filt"], input=out, capture_output=True, text=True).stdout
    res, name = {}, None
    for line in demangled.splitlines():
        m = re.match(r"\s*Function (.*):\s*$", line)
        if m:
            name = m.group(1)
            continue
        r = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if r and name:
            res[name] = (int(r.group(1)), int(r.group(2)))
            name = None
    return res


def test_hot_kernels_register_budget_and_no_spills():
    res = _resources()
    for prefix, (cap, scap) in BUDGET.items():
        hits = [(n, v) for n, v in res.items() if n.startswith(prefix + "(")]
        assert hits, f"kernel {prefix} not found in {LIB}"
        for n, (reg, stack) in hits:
            assert reg <= cap, f"{n}: {reg} registers > {cap}"
            assert stack <= scap, f"{n}: {stack} bytes of stack (spills) > {scap}"
