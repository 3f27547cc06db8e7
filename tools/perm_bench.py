"""Permute-kernel microbenchmark on cfg4-shaped tensors (GB/s of algorithmic bytes, CUDA events).

Patterns (A: V(x)V <- V(x)V, legs 0..3):
  identity   (0,1;2,3)  -- the kernel's ceiling on this layout (pure strided copy)
  A-operand  (0,2;1,3)  -- fastest leg kept (rows path)
  B-operand  (2,0;1,3)  -- fastest leg changes (tiled path)
plus torch copy_ of the same number of bytes as the HBM reference.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_10076_b200 import tk  # noqa: E402
from workloads import configs as W  # noqa: E402


def main():
    d_leg = int(sys.argv[1]) if len(sys.argv) > 1 else 384
    V = W.cfg4_leg(d_leg)
    spec = {"cod": [V, V], "dom": [V, V]}
    A = tk.tensor_from_spec(spec)
    a = torch.randn(A.nelems, dtype=torch.float64, device="cuda")
    out = {"d_leg": d_leg, "nelems": A.nelems}
    for name, (p, q) in {"identity": ([0, 1], [2, 3]), "A_operand": ([0, 2], [1, 3]),
                         "B_operand": ([2, 0], [1, 3]), "C_output": ([0, 2], [1, 3])}.items():
        from oracle import contract as OC  # spaces only (selection rule) for building the output tensor
        cod, dom = OC.permuted_spaces(spec["cod"], spec["dom"], p, q)
        C = tk.tensor_from_spec({"cod": cod, "dom": dom})
        c = torch.empty(C.nelems, dtype=torch.float64, device="cuda")
        for _ in range(3):
            tk.tk_permute(A, a, p, q, C, c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            tk.tk_permute(A, a, p, q, C, c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        out[name] = {"ms": round(ms, 3), "GB_s": round(2 * 8 * A.nelems / ms / 1e6, 1)}
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out["torch_copy"] = {"ms": round(ms, 3), "GB_s": round(2 * 8 * A.nelems / ms / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
