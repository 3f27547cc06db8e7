"""Blockwise truncated SVD of the two-site tensors (Alg. 12's final step) on one B200.

For cfg2 (U(1), chi 512), cfg3 (fermionic U(1)xU(1), chi 2048) and cfg6's SU(2) A-tensor: the time of
tk_svd (permute + Jacobi sweeps), tk_svd_truncate (spectrum D2H + global rule, host) and tk_svd_extract,
CUDA events / wall clock, median of reps; the oracle's time (numpy LAPACK per block + its own permute)
on the host cores beside it. One JSON line per case.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_10076_b200 import tk, layout_io  # noqa: E402
from workloads import configs as W  # noqa: E402


def cases():
    c2, c3, c6, c7, c8 = W.cfg2(), W.cfg3(), W.cfg6(), W.cfg7(), W.cfg8()
    return [("cfg2 theta (alpha,s1 | s2,beta), max_dim 512", c2, "theta", [0, 1], [2, 3], 512, False),
            ("cfg3 theta (alpha,s1 | s2,beta), max_dim 2048", c3, "theta", [0, 1], [2, 3], 2048, False),
            ("cfg3 theta ComplexF64, max_dim 2048", c3, "theta", [0, 1], [2, 3], 2048, True),
            ("cfg6 A (alpha,s | beta), max_dim 1172", c6, "A", [0, 1], [2], 1172, False),
            ("cfg7 theta (alpha,s1 | s2,beta), max_dim 2058", c7, "theta", [0, 1], [2, 3], 2058, False),
            ("cfg8 theta (alpha,s1 | s2,beta), max_dim 2008", c8, "theta", [0, 1], [2, 3], 2008, False)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--oracle", action="store_true")
    args = ap.parse_args()
    for name, cfg, tname, p, q, md, cplx in cases():
        spec, idx = cfg["tensors"][tname]
        A = tk.tensor_from_spec(spec, tk.TK_C64 if cplx else tk.TK_F64)
        a = torch.from_numpy(layout_io.fill(A, cfg["cfg"], idx, cplx)).cuda()
        tdt = torch.complex128 if cplx else torch.float64
        nb = tk.tk_svd_workspace(A, p, q)
        ws = torch.empty(nb // 8 + 64, dtype=torch.float64, device="cuda")
        spec_ = None
        t_svd, t_tr, t_ex = [], [], []
        for r in range(args.reps + 2):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record()
            tk.tk_svd(A, a, p, q, ws, ws.numel() * 8)
            e1.record()
            e1.synchronize()  # the host clock times the truncation alone, not the wait for tk_svd
            h0 = time.perf_counter()
            Wsp, U, S, Vh, err, nrm = tk.tk_svd_truncate(A, p, q, ws, md, 0.0)
            h1 = time.perf_counter()
            bufs = [torch.empty(T.nelems, dtype=tdt, device="cuda") for T in (U, S, Vh)]
            x0 = torch.cuda.Event(enable_timing=True)
            x0.record()
            tk.tk_svd_extract(A, p, q, ws, U, bufs[0], S, bufs[1], Vh, bufs[2])
            e2.record()
            torch.cuda.synchronize()
            if r >= 2:
                t_svd.append(e0.elapsed_time(e1) * 1e3)
                t_tr.append((h1 - h0) * 1e6)
                t_ex.append(x0.elapsed_time(e2) * 1e3)
            spec_ = (len(tk.tk_svd_spectrum(A, p, q, ws)), err, nrm, U.nelems)
        blocks = A  # noqa
        out = {"case": name, "kind": cfg["kind"], "elements": A.nelems, "blocks": spec_[0],
               "us_svd": round(float(np.median(t_svd)), 1), "us_truncate_host": round(float(np.median(t_tr)), 1),
               "us_extract": round(float(np.median(t_ex)), 1), "trunc_err": spec_[1], "norm": spec_[2]}
        if args.oracle:
            from oracle import svd as OS, layout as OL
            from tests import harness as H
            lt = OL.homspace_layout(cfg["kind"], spec["cod"], spec["dom"])
            x = H.oracle_flat(lt, cfg["cfg"], idx, cplx)
            t0 = time.perf_counter()
            lp, xp, _ = OS.permuted(cfg["kind"], spec["cod"], spec["dom"], x, p, q)
            svds = OS.block_svd(lp, xp)
            OS.truncation(cfg["kind"], [(c, s) for c, u, s, vh in svds], md, 0.0)
            out["oracle_s"] = round(time.perf_counter() - t0, 3)
            out["oracle_cores"] = len(os.sched_getaffinity(0))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
