"""Runs one blockwise SVD of a config's two-site tensor a few times (target for ncu captures)."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_10076_b200 import tk, layout_io  # noqa: E402
from workloads import configs as W  # noqa: E402

cfg = W.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]()
spec, idx = cfg["tensors"]["theta"]
A = tk.tensor_from_spec(spec)
a = torch.from_numpy(layout_io.fill(A, cfg["cfg"], idx)).cuda()
nb = tk.tk_svd_workspace(A, [0, 1], [2, 3])
ws = torch.empty(nb // 8 + 64, dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    tk.tk_svd(A, a, [0, 1], [2, 3], ws, ws.numel() * 8)
torch.cuda.synchronize()
