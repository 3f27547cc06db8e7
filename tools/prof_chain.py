"""Run one BASELINE config's chain a few times (for ncu captures): python tools/prof_chain.py CFG [REPS]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_configs import build, run_chain  # noqa: E402
from workloads import configs as W  # noqa: E402

if __name__ == "__main__":
    k = int(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    makers = {1: W.cfg1, 2: W.cfg2, 3: W.cfg3, 4: lambda: W.cfg4(d_leg=128), 5: W.cfg5, 6: W.cfg6, 7: W.cfg7, 8: W.cfg8}
    T, steps = build(makers[k](), torch.device("cuda", 0), fuse=os.environ.get("TK_CHAIN_NO_FUSE") is None)
    for _ in range(reps):
        run_chain(T, steps)
    torch.cuda.synchronize()
    print("ok")
