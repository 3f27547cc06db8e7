"""Single-block SVD timing (tile kernel / cluster kernel) for the Jacobi-round analysis: one U(1) sector
of rows x cols, tk_svd timed with CUDA events (median of reps)."""
import json
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_10076_b200 import tk  # noqa: E402
from workloads import configs as W  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                                                       ["16x16", "32x32", "64x64", "133x133", "181x181"])]
for rows, cols in shapes:
    A = tk.tensor_from_spec({"cod": [W.space("U1", [((0,), rows)])], "dom": [W.space("U1", [((0,), cols)])]},
                            tk.TK_F64)
    a = torch.from_numpy(np.random.default_rng(1).standard_normal(A.nelems)).cuda()
    nb = tk.tk_svd_workspace(A, [0], [1])
    ws = torch.empty(nb // 8 + 64, dtype=torch.float64, device="cuda")
    ts = []
    for r in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tk.tk_svd(A, a, [0], [1], ws, ws.numel() * 8)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"shape": f"{rows}x{cols}", "us": round(float(np.median(ts)), 1)}), flush=True)
