"""Latency / throughput of every BASELINE config through tk_contract on one B200.

For each config the whole contraction chain (cfg2/3: L*theta -> *W -> *W -> *R) runs on
resident device buffers; reported: microseconds per chain (CUDA events, median of N
replays), useful block GFLOP/s, kernel launches per chain, and the same chain replayed
as one CUDA graph (plans are warmed first; capture needs cached plans). One JSON line
per config. --oracle adds the CPU oracle's wall time for the same chain (tier 1 dense
for cfg1/2/5, tier 2 charge-tuple for cfg3) on the host cores.
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


def build(cfg, dev, fuse=False):
    """Buffers and calls of a chain; fuse=True sends every consecutive pair that tk_contract2 runs as one
    kernel (the abelian MPO steps) through it: the step then carries pair = (nb2, lb2, nc2, lc2)."""
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        t = tk.tensor_from_spec(spec)
        T[name] = (t, torch.from_numpy(layout_io.fill(t, cfg["cfg"], idx)).to(dev))
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        C = tk.tk_contract_output(T[na][0], la, T[nb][0], lb, lc, ncod)
        T[nc] = (C, torch.zeros(C.nelems, dtype=torch.float64, device=dev))
    steps, cs, i = [], cfg["steps"], 0
    while i < len(cs):
        na, la, nb, lb, nc, lc, ncod = cs[i]
        if fuse and i + 1 < len(cs) and cs[i + 1][0] == nc:
            _, la2, nb2, lb2, nc2, lc2, _ = cs[i + 1]
            n, fu = tk.tk_contract2_workspace(T[na][0], la, T[nb][0], lb, T[nc][0], lc, T[nb2][0], lb2, T[nc2][0],
                                              lc2, want_fused=True)
            if fu:
                ws = torch.empty(max(n // 8 + 64, 1), dtype=torch.float64, device=dev)
                steps.append((na, la, nb, lb, nc, lc, ws, (nb2, lb2, nc2, lc2)))
                i += 2
                continue
        ws_n = tk.tk_contract_workspace(T[na][0], la, T[nb][0], lb, T[nc][0], lc)
        ws = torch.empty(max(ws_n // 8 + 64, 1), dtype=torch.float64, device=dev)
        steps.append((na, la, nb, lb, nc, lc, ws, None))
        i += 1
    return T, steps


def _call(T, step):
    na, la, nb, lb, nc, lc, ws, pair = step
    A, a = T[na]
    B, b = T[nb]
    C, c = T[nc]
    if pair is None:
        tk.tk_contract(A, a, la, B, b, lb, C, c, lc, ws=ws, ws_bytes=ws.numel() * 8)
    else:
        nb2, lb2, nc2, lc2 = pair
        tk.tk_contract2(A, a, la, B, b, lb, C, lc, T[nb2][0], T[nb2][1], lb2, T[nc2][0], T[nc2][1], lc2, ws=ws,
                        ws_bytes=ws.numel() * 8)


def run_chain(T, steps):
    launches = 0
    for st in steps:
        _call(T, st)
        launches += tk.tk_last_launch_count()
    return launches


def chain_flops(T, steps):
    tk.tk_profile_enable(True)
    fl = 0.0
    for (na, la, nb, lb, nc, lc, ws, pair) in steps:
        if pair is not None:  # a fused pair: the two steps' block flops from their plans
            nb2, lb2, nc2, lc2 = pair
            fl += tk.tk_contract_roofline(T[na][0], la, T[nb][0], lb, T[nc][0], lc, 1e12, 1e12)["flops"]
            fl += tk.tk_contract_roofline(T[nc][0], lc, T[nb2][0], lb2, T[nc2][0], lc2, 1e12, 1e12)["flops"]
            continue
        A, a = T[na]
        B, b = T[nb]
        C, c = T[nc]
        tk.tk_contract(A, a, la, B, b, lb, C, c, lc, ws=ws, ws_bytes=ws.numel() * 8)
        torch.cuda.synchronize()
        fl += tk.tk_phase_times()[2]
    tk.tk_profile_enable(False)
    return fl


def phase_breakdown(T, steps, reps=20):
    """Median per-step [permute A, permute B, GEMM, permute C] microseconds (CUDA events per phase)."""
    tk.tk_profile_enable(True)
    res = []
    for (na, la, nb, lb, nc, lc, ws, pair) in steps:
        A, a = T[na]
        B, b = T[nb]
        C, c = T[nc]
        if pair is not None:
            continue
        ms = []
        for _ in range(reps):
            tk.tk_contract(A, a, la, B, b, lb, C, c, lc, ws=ws, ws_bytes=ws.numel() * 8)
            torch.cuda.synchronize()
            ms.append(tk.tk_phase_times()[0])
        res.append([round(float(x) * 1e3, 1) for x in np.median(np.array(ms), axis=0)])
    tk.tk_profile_enable(False)
    return res


def time_events(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def oracle_time(cfg):
    from tests import harness as H
    t0 = time.perf_counter()
    if cfg["cfg"] in (7, 8):
        return None, "none at full size (dense oracle needs 5.4 GB intermediates)"
    if cfg["cfg"] == 3:
        H.oracle_chain_blocks(cfg)
        tier = "tier 2 (charge-tuple einsum)"
    else:
        H.oracle_chain_dense(cfg)
        tier = "tier 1 (dense embedding + einsum)"
    return time.perf_counter() - t0, tier


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="1,2,3,5,6,7,8")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--phases", action="store_true", help="per-step [permA, permB, gemm, permC] us")
    ap.add_argument("--no-fuse", action="store_true", help="every step through tk_contract (no tk_contract2)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    makers = {1: W.cfg1, 2: W.cfg2, 3: W.cfg3, 4: lambda: W.cfg4(d_leg=128), 5: W.cfg5, 6: W.cfg6, 7: W.cfg7, 8: W.cfg8}
    for k in [int(x) for x in args.cfgs.split(",")]:
        cfg = makers[k]()
        T, steps = build(cfg, dev, fuse=not args.no_fuse)
        fl = chain_flops(T, steps)
        for _ in range(5):
            launches = run_chain(T, steps)
        torch.cuda.synchronize()
        us = time_events(lambda: run_chain(T, steps), args.reps)
        # whole chain as one CUDA graph
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run_chain(T, steps)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            run_chain(T, steps)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        us_g = time_events(g.replay, args.reps)
        out = {"cfg": k, "kind": cfg["kind"], "steps": len(cfg["steps"]), "calls": len(steps), "block_flops": fl, "launches": launches,
               "us_per_chain": round(us, 2), "GFLOP_s": round(fl / (us * 1e-6) / 1e9, 2),
               "us_per_chain_graph": round(us_g, 2), "GFLOP_s_graph": round(fl / (us_g * 1e-6) / 1e9, 2)}
        if args.phases:
            out["phase_us_per_step"] = phase_breakdown(T, steps)
        if args.oracle:
            t, tier = oracle_time(cfg)
            out["oracle_s"] = round(t, 3) if t is not None else None
            out["oracle_tier"] = tier
            out["oracle_cores"] = len(os.sched_getaffinity(0))
            out["speedup_vs_oracle_graph"] = round(t / (us_g * 1e-6), 1) if t is not None else None
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
