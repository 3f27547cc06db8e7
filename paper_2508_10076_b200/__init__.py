"""B200-native symmetric-tensor contraction (arXiv 2508.10076 hot path).

The product is the C-ABI library libtk_b200.so (include/tk.h): a host C++
planner (graded spaces, fusion trees, permute/contract plans, plan cache) and
sm_100a CUDA kernels (batched subblock permute, grouped FP64 DMMA GEMM).
`paper_2508_10076_b200.tk` is its thin ctypes binding; `layout_io` places and
reads seeded subblock values through the library's own layout queries.
"""
# `tk` is not imported here so that `paper_2508_10076_b200.build` can run on a fresh checkout;
# importing `paper_2508_10076_b200.tk` raises ImportError when the in-tree library is missing
# (there is no CPU fallback).
__all__ = ["tk", "layout_io", "build"]
