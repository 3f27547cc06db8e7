"""Run one BASELINE config's chain a few times (for ncu captures): python tools/prof_chain.py CFG [REPS].
TK_CHAIN_NO_FUSE=1: every step through tk_contract; TK_CHAIN_NCON=1: the network through tk_ncon."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_configs import build, run_chain  # noqa: E402
from workloads import configs as W  # noqa: E402
from paper_2508_10076_b200 import tk  # noqa: E402

if __name__ == "__main__":
    k = int(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    makers = {1: W.cfg1, 2: W.cfg2, 3: W.cfg3, 4: lambda: W.cfg4(d_leg=128), 5: W.cfg5, 6: W.cfg6, 7: W.cfg7, 8: W.cfg8}
    cfg = makers[k]()
    T, steps = build(cfg, torch.device("cuda", 0), fuse=os.environ.get("TK_CHAIN_NO_FUSE") is None)
    if os.environ.get("TK_CHAIN_NCON"):
        names, labels, order, ncod, out = W.chain_as_ncon(cfg)
        tens = [T[n][0] for n in names]
        n = tk.tk_ncon_workspace(tens, labels, order, ncod)
        ws = torch.empty(n // 8 + 32, dtype=torch.float64, device="cuda")
        for _ in range(reps):
            tk.tk_ncon(tens, [T[x][1] for x in names], labels, order, ncod, T[out][0], T[out][1], ws=ws,
                       ws_bytes=ws.numel() * 8)
    else:
        for _ in range(reps):
            run_chain(T, steps)
    torch.cuda.synchronize()
    print("ok")
