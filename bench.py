"""Benchmark of the symmetric-tensor contraction hot path on B200 (BASELINE.json metric).

metric: useful block GFLOP/s of tk_contract (Float64) -- SUM over coupled sectors of 2 M_c K_c N_c
        (block-sparse flops only, never the dense equivalent) / time -- plus permute GB/s,
        each as a fraction of roofline.
workload (N=1): config 4, "U(1) PEPS/CTMRG-style large contraction, Float64", the largest
        U(1) config, at leg dim 384 (reading C20: the literal 4096 needs 115 TB per operand).
        A step = one tk_contract C(x1,y2;x3,y4) = sum A(x1,x2;x3,x4) B(x4,y2;x2,y4):
        permute A, permute B, grouped DMMA GEMM, permute C (all launches inside the timed region).
Inputs are resident in HBM and far larger than L2 (8.9 GB per operand), so no flush is needed.

Multi-GPU: the path does not shard in this build ("replicas only"): every rank runs
the same workload on its own GPU; value = all ranks' flops / max-over-ranks time.

--impl reference: the CPU oracle (tier-2 charge-tuple einsum) timed on the host cores on a
bounded sample of the same workload (a fixed set of output subblocks per step).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CHAIN_CFGS = (2, 3, 5, 6, 7, 8)   # the DMRG-shaped chains (Alg. 11 / 12 contractions), timed beside cfg4
GEMM_KERNEL = ("gemm_tma_kernel (persistent, TMA-fed grouped DMMA GEMM over the coupled sectors; big tiles) "
               "+ gemm_small_kernel (edge classes)")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def workload(args):
    from workloads import configs as W
    cfg = W.cfg4(d_leg=args.d_leg, complex_=args.dtype == "c64")
    return cfg


def dtype_name(args):
    return "ComplexF64" if args.dtype == "c64" else "Float64"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU oracle
def oracle_inputs(cfg):
    """Input blocks for the oracle, generated on first use and then cached (so that timed
    oracle steps measure the contraction, not the input generator)."""
    from oracle import layout as OL, blocksparse as BS
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][0]
    A, B = cfg["tensors"][na][0], cfg["tensors"][nb][0]
    kind = cfg["kind"]
    cx = cfg.get("dtype") == "c64"
    return (BS.LazyBlocks(OL.homspace_layout(kind, A["cod"], A["dom"]), cfg["cfg"], cfg["tensors"][na][1], cx),
            BS.LazyBlocks(OL.homspace_layout(kind, B["cod"], B["dom"]), cfg["cfg"], cfg["tensors"][nb][1], cx))


def oracle_sample(cfg, budget_s, keys=None, seed=0, inputs=None):
    """Tier-2 oracle on output subblocks of C. Returns (flops, seconds, keys used)."""
    from oracle import layout as OL, contract as OC, blocksparse as BS
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][0]
    A, B = cfg["tensors"][na][0], cfg["tensors"][nb][0]
    kind = cfg["kind"]
    Ab, Bb = inputs if inputs is not None else oracle_inputs(cfg)
    cod, dom = OC.output_spaces(A["cod"], A["dom"], B["cod"], B["dom"], la, lb, lc, ncod)
    lt = OL.homspace_layout(kind, cod, dom)
    all_keys = [tuple(s.key[0]) + tuple(s.key[3]) for s in lt.subblocks]
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(all_keys))
    stats = {"flops": 0.0}
    used = []
    t0 = time.perf_counter()
    if keys is not None:
        BS.contract_blocks(kind, Ab, A["cod"], A["dom"], la, Bb, B["cod"], B["dom"], lb, lc, ncod,
                           out_keys=keys, stats=stats)
        used = keys
    else:
        # grow the batch of output subblocks until one batch alone takes about budget_s
        n = 4
        while True:
            batch = [all_keys[i] for i in order[:n]]
            stats = {"flops": 0.0}
            t0 = time.perf_counter()
            BS.contract_blocks(kind, Ab, A["cod"], A["dom"], la, Bb, B["cod"], B["dom"], lb, lc, ncod,
                               out_keys=batch, stats=stats)
            dt = time.perf_counter() - t0
            used = batch
            if dt >= budget_s or n >= len(all_keys):
                break
            n = min(len(all_keys), max(n + 1, int(n * min(8.0, 1.2 * budget_s / max(dt, 1e-3)))))
    # useful flops: 2MKN per real block product, 8MKN per complex one (reading C21)
    return stats["flops"] * (4.0 if cfg.get("dtype") == "c64" else 1.0), time.perf_counter() - t0, used


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workload(args)
    cores = len(os.sched_getaffinity(0))
    # calibrate one step's sample (~8 s of oracle work), then time W + K identical steps
    inputs = oracle_inputs(cfg)
    _, _, keys = oracle_sample(cfg, budget_s=args.ref_step_s, inputs=inputs)
    for _ in range(args.warmup):
        oracle_sample(cfg, 0, keys=keys, inputs=inputs)
    fl, tot = 0.0, 0.0
    for _ in range(args.steps):
        f, t, _ = oracle_sample(cfg, 0, keys=keys, inputs=inputs)
        fl += f
        tot += t
    value = fl / tot / 1e9
    sample = (f"{len(keys)} of the C output subblocks of cfg4 ({dtype_name(args)}, D_leg={args.d_leg}) per step, "
              f"tier-2 charge-tuple einsum (oracle/blocksparse.py)")
    line = {
        "impl": "reference", "metric": f"useful block GFLOP/s of tk_contract ({dtype_name(args)})",
        "value": round(value, 4),
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / args.steps, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded N(0,1), workloads/gen.py)",
        "config": {"workload": f"cfg4 U(1) PEPS rank-4 x rank-4 contraction, {dtype_name(args)}, D_leg={args.d_leg} "
                               f"(reading C20)", "d_leg": args.d_leg},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- multi-rank plumbing
def max_over_ranks(x, world, device=None):
    """Max of a per-rank device time over all ranks (the contract's max-over-ranks timing)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gflops(flops_per_step, steps, world, total_ms):
    """Replicas only: every rank runs the same workload; value = all ranks' flops /
    the slowest rank's time (weak scaling)."""
    return world * flops_per_step * steps / (total_ms * 1e-3) / 1e9


# --------------------------------------------------------------------------- in-run peaks
def measure_fp64_peak(stream, dev):
    """FP64 roofline denominator measured in THIS process (MEASURED_PEAKS.json has no FP64 entry):
    the library's DMMA probe (tk_dmma_probe: 148 x 4 CTAs of 8 warps, back-to-back independent
    mma.sync m8n8k4 f64) and cuBLAS DGEMM 8192^3 through torch.matmul, best of 5 each (CUDA events)."""
    import torch
    from paper_2508_10076_b200 import tk
    blocks, iters = 148 * 4, 65536

    def probe(reps=1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fl = sum(tk.tk_dmma_probe(blocks, iters, stream=stream) for _ in range(reps))
        e1.record(stream)
        e1.synchronize()
        return fl / (e0.elapsed_time(e1) * 1e-3) / 1e12
    probe()
    dmma = max(probe() for _ in range(5))          # burst: ~35 ms launches
    dmma_sus = probe(reps=40)                      # sustained: ~1.4 s back to back
    n = 8192
    x = torch.randn(n, n, dtype=torch.float64, device=dev)
    y = torch.randn(n, n, dtype=torch.float64, device=dev)
    with torch.cuda.stream(stream):
        torch.matmul(x, y)
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.matmul(x, y)
            e1.record(stream)
            e1.synchronize()
            best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del x, y
    return {"dmma_probe_tflops": round(dmma, 3), "dmma_probe_sustained_tflops": round(dmma_sus, 3),
            "cublas_dgemm_8192_tflops": round(best, 3)}


def time_chains(dev, stream0, peak_flops, hbm_bytes_s, reps=30):
    """Every DMRG-shaped chain (cfg2/3/5/6/7/8 at their full sizes) replayed as ONE CUDA graph; L2 is
    flushed (a 256 MB write) before every timed replay; median of `reps` CUDA-event timings. Two ways:
    the network through tk_ncon (`us_per_chain`: the library orders the intermediates -- a gathered MPO
    step stores straight into the next GEMM's operand order -- and runs the abelian MPO pair through
    tk_contract2) and the config's explicit pairwise steps (`us_per_chain_pairwise`: one tk_contract per
    step, intermediates in the config's orders). Roofline per SURVEY §8(d) over the config's pairwise steps: sum of
    tk_contract_roofline (GEMM blocks max(flops/P, bytes/BW) + permute bytes/BW) at the in-run DMMA peak
    and MEASURED_PEAKS' HBM bandwidth. `us_per_call_eager`: the tk_ncon call issued without a graph, back to back
    (host wall clock per call, plans cached, no L2 flush): the API's host cost shows where it exceeds the graph time."""
    import torch
    from paper_2508_10076_b200 import tk, layout_io
    from workloads import configs as W
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(dev)          # graphs are captured (and replayed) on a side stream
    stream.wait_stream(stream0)
    out = {}
    for k in CHAIN_CFGS:
        cfg = W.CONFIGS[k]()
        T = {}
        for name, (spec, idx) in cfg["tensors"].items():
            t = tk.tensor_from_spec(spec)
            T[name] = (t, torch.from_numpy(layout_io.fill(t, cfg["cfg"], idx)).to(dev))
        steps, roof = [], {"flops": 0.0, "gemm_bytes": 0.0, "permute_bytes": 0.0, "seconds": 0.0}
        for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
            A, B = T[na][0], T[nb][0]
            C = tk.tk_contract_output(A, la, B, lb, lc, ncod)
            T[nc] = (C, torch.zeros(C.nelems, dtype=torch.float64, device=dev))
            r = tk.tk_contract_roofline(A, la, B, lb, C, lc, peak_flops, hbm_bytes_s)
            for key in roof:
                roof[key] += r[key]
        # the config's explicit pairwise chain: one tk_contract per step, intermediates in the config's
        # leg orders (the baseline the network path below is compared with)
        for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
            nws = tk.tk_contract_workspace(T[na][0], la, T[nb][0], lb, T[nc][0], lc)
            ws = torch.empty(max(nws // 8 + 64, 1), dtype=torch.float64, device=dev)
            steps.append((na, la, nb, lb, nc, lc, ws))

        def chain():
            n = 0
            for (na, la, nb, lb, nc, lc, ws) in steps:
                tk.tk_contract(T[na][0], T[na][1], la, T[nb][0], T[nb][1], lb, T[nc][0], T[nc][1], lc, ws=ws,
                               ws_bytes=ws.numel() * 8, stream=stream)
                n += tk.tk_last_launch_count()
            return n
        # the same network through tk_ncon (the library plans the intermediates' leg orders and runs the
        # fusable pairs through tk_contract2; same pairwise order, same arithmetic)
        names, nlabels, norder, ncod_out, out_name = W.chain_as_ncon(cfg)
        nT = [T[nm][0] for nm in names]
        nws_n = tk.tk_ncon_workspace(nT, nlabels, norder, ncod_out)
        nws = torch.empty(max(nws_n // 8 + 64, 1), dtype=torch.float64, device=dev)
        Cn = T[out_name][0]

        def network():
            tk.tk_ncon(nT, [T[nm][1] for nm in names], nlabels, norder, ncod_out, Cn, T[out_name][1], ws=nws,
                       ws_bytes=nws.numel() * 8, stream=stream)
            return tk.tk_last_launch_count()

        def timed(fn):
            with torch.cuda.stream(stream):
                n = fn()
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    fn()
                for _ in range(3):
                    g.replay()
                ts = []
                for _ in range(reps):
                    flush.fill_(1.0)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
            del g
            return float(np.median(ts)), n
        us_pw, launches_pw = timed(chain)
        us, launches = timed(network)
        # the same tk_ncon call without a graph: host wall clock per call, back to back (plans cached: what
        # a caller's loop pays per chain when it does not capture a graph), stream drained at the end
        with torch.cuda.stream(stream):
            network()
            torch.cuda.synchronize(dev)
            h0 = time.perf_counter()
            for _ in range(reps):
                network()
            torch.cuda.synchronize(dev)
            us_eager = (time.perf_counter() - h0) / reps * 1e6
        out[f"cfg{k}"] = {"kind": cfg["kind"], "us_per_chain": round(us, 2), "launches": launches,
                          "api": "tk_ncon", "steps": len(cfg["steps"]),
                          "us_per_chain_pairwise": round(us_pw, 2), "launches_pairwise": launches_pw,
                          "us_per_call_eager": round(us_eager, 2),
                          "block_flops": roof["flops"],
                          "GFLOP_s": round(roof["flops"] / (us * 1e-6) / 1e9, 2),
                          "roofline_us": round(roof["seconds"] * 1e6, 2),
                          "roofline_frac": round(roof["seconds"] * 1e6 / us, 3),
                          "permute_bytes": roof["permute_bytes"], "gemm_min_bytes": roof["gemm_bytes"]}
        del T, steps, nws
        torch.cuda.empty_cache()
    return out


def time_svd(dev, stream, reps=7, oracle=True):
    """The two-site truncated SVD that closes Alg. 12: theta (alpha, s1 ; s2, beta) of cfg2 and
    cfg3 at full size, split as (alpha, s1) | (s2, beta). `us_svd` is tk_svd (permute into the workspace +
    the blockwise Jacobi SVD), `us_extract` tk_svd_extract (U, S, Vh of the kept values), CUDA events on
    the launching stream, median of `reps`; the global truncation (tk_svd_truncate: spectrum D2H + rule + new
    host objects) is timed by the wall clock after tk_svd has completed. The oracle (numpy LAPACK per block + its own permute, oracle/svd.py) runs on the host
    cores beside it (rank 0 only, ~1 s)."""
    import torch
    from paper_2508_10076_b200 import tk, layout_io
    from workloads import configs as W
    out = {}
    for name, cfg, md in (("cfg2", W.cfg2(), 512), ("cfg3", W.cfg3(), 2048)):
        spec, idx = cfg["tensors"]["theta"]
        A = tk.tensor_from_spec(spec)
        a = torch.from_numpy(layout_io.fill(A, cfg["cfg"], idx)).to(dev)
        p, q = [0, 1], [2, 3]
        nb = tk.tk_svd_workspace(A, p, q)
        ws = torch.empty(nb // 8 + 64, dtype=torch.float64, device=dev)
        ts, tt, tx = [], [], []
        for r in range(reps + 2):
            e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            torch.cuda.synchronize(dev)
            e0.record(stream)
            tk.tk_svd(A, a, p, q, ws, ws.numel() * 8, stream=stream)
            e1.record(stream)
            e1.synchronize()  # so the host clock below times the truncation alone, not the wait for tk_svd
            h0 = time.perf_counter()
            Wsp, U, S, Vh, err, nrm = tk.tk_svd_truncate(A, p, q, ws, md, 0.0, stream=stream)
            h1 = time.perf_counter()
            bufs = [torch.empty(T.nelems, dtype=torch.float64, device=dev) for T in (U, S, Vh)]
            e2.record(stream)
            tk.tk_svd_extract(A, p, q, ws, U, bufs[0], S, bufs[1], Vh, bufs[2], stream=stream)
            e3.record(stream)
            torch.cuda.synchronize(dev)
            if r >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
                tt.append((h1 - h0) * 1e6)
                tx.append(e2.elapsed_time(e3) * 1e3)
        spec_ = tk.tk_svd_spectrum(A, p, q, ws, stream=stream)
        d = {"blocks": len(spec_), "largest_block_k": max(len(x) for x in spec_), "elements": A.nelems, "max_dim": md,
             "us_svd": round(float(np.median(ts)), 1), "us_truncate_host": round(float(np.median(tt)), 1),
             "us_extract": round(float(np.median(tx)), 1), "trunc_err": err, "norm": nrm}
        if oracle:
            from oracle import svd as OS, layout as OL
            from tests import harness as H
            lt = OL.homspace_layout(cfg["kind"], spec["cod"], spec["dom"])
            x = H.oracle_flat(lt, cfg["cfg"], idx)
            t0 = time.perf_counter()
            lp, xp, _ = OS.permuted(cfg["kind"], spec["cod"], spec["dom"], x, p, q)
            svds = OS.block_svd(lp, xp)
            OS.truncation(cfg["kind"], [(c, s_) for c, u, s_, vh in svds], md, 0.0)
            d["oracle_s"] = round(time.perf_counter() - t0, 3)
            d["oracle_cores"] = len(os.sched_getaffinity(0))
            d["oracle_kind"] = "numpy LAPACK gesdd per block (oracle/svd.py), host cores"
        out[name] = d
        del ws, a
    return out


# --------------------------------------------------------------------------- GPU
def run_gpu(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    from paper_2508_10076_b200 import tk, layout_io

    cfg = workload(args)
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][0]
    cplx = args.dtype == "c64"
    tdt, esz = (torch.complex128, 16) if cplx else (torch.float64, 8)
    A = tk.tensor_from_spec(cfg["tensors"][na][0], tk.TK_C64 if cplx else tk.TK_F64)
    B = tk.tensor_from_spec(cfg["tensors"][nb][0], tk.TK_C64 if cplx else tk.TK_F64)
    C = tk.tk_contract_output(A, la, B, lb, lc, ncod)
    t0 = time.time()
    a_h = torch.from_numpy(layout_io.fill(A, cfg["cfg"], cfg["tensors"][na][1], cplx))
    b_h = torch.from_numpy(layout_io.fill(B, cfg["cfg"], cfg["tensors"][nb][1], cplx))
    t_fill = time.time() - t0
    a = a_h.to(dev)
    b = b_h.to(dev)
    c = torch.empty(C.nelems, dtype=tdt, device=dev)
    t0 = time.perf_counter()
    ws_n = tk.tk_contract_workspace(A, la, B, lb, C, lc)   # builds + caches the plan (cold)
    t_plan_cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    tk.tk_contract_workspace(A, la, B, lb, C, lc)
    t_plan_cached = time.perf_counter() - t0
    ws = torch.empty(ws_n // 8 + 64, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        tk.tk_contract(A, a, la, B, b, lb, C, c, lc, ws=ws, ws_bytes=ws.numel() * 8, stream=stream)

    fp64 = measure_fp64_peak(stream, dev)           # roofline denominator, measured in this run
    peak_tf = fp64["dmma_probe_sustained_tflops"]
    tk.tk_profile_enable(True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    phase = np.zeros(4)
    launches = 0
    flops = 0.0
    pbytes = np.zeros(4)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
        launches += tk.tk_last_launch_count()
        stream.synchronize()   # per-phase events are read back each step (one host sync per ~0.7 s step)
        ms4, by4, fl = tk.tk_phase_times()
        phase += np.array(ms4)
        pbytes = np.array(by4)
        flops = fl
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    total_ms = max_over_ranks(total_ms, world, dev)
    ms_step = total_ms / args.steps
    value = whole_job_gflops(flops, args.steps, world, total_ms)

    # ---- end to end through the public call with host buffers (pinned), copies inside the timed region.
    # Every step copies its inputs host -> device and its result device -> host. Steps are pipelined the
    # way a stream of contractions runs in practice: inputs and outputs are double-buffered on the
    # device, H2D of step k+1 and D2H of step k-1 run on their own streams (separate copy engines)
    # while step k computes; the timed region spans the first H2D to the last D2H.
    e2e = None
    if args.e2e_steps > 0:
        a_p = a_h.pin_memory()
        b_p = b_h.pin_memory()
        c_p = [torch.empty(C.nelems, dtype=tdt).pin_memory() for _ in range(2)]
        a_d, b_d, c_d = [a, torch.empty_like(a)], [b, torch.empty_like(b)], [c, torch.empty_like(c)]
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        S = args.e2e_steps
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        in_ready, done, out_copied = [ev() for _ in range(S)], [ev() for _ in range(S)], [ev() for _ in range(S)]
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        x0.record(h2d)
        for k in range(S):
            i = k % 2
            if k >= 2:
                h2d.wait_event(done[k - 2])           # input buffer i is free again
            with torch.cuda.stream(h2d):
                a_d[i].copy_(a_p, non_blocking=True)
                b_d[i].copy_(b_p, non_blocking=True)
                in_ready[k].record(h2d)
            stream.wait_event(in_ready[k])
            if k >= 2:
                stream.wait_event(out_copied[k - 2])  # output buffer i has been read back
            tk.tk_contract(A, a_d[i], la, B, b_d[i], lb, C, c_d[i], lc, ws=ws, ws_bytes=ws.numel() * 8, stream=stream)
            done[k].record(stream)
            d2h.wait_event(done[k])
            with torch.cuda.stream(d2h):
                c_p[i].copy_(c_d[i], non_blocking=True)
                out_copied[k].record(d2h)
        x1.record(d2h)
        torch.cuda.synchronize(dev)
        e2e_ms = x0.elapsed_time(x1)
        e2e_ms = max_over_ranks(e2e_ms, world, dev)
        e2e = {"value": round(whole_job_gflops(flops, S, world, e2e_ms), 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int((A.nelems + B.nelems) * esz), "d2h_bytes_per_step": int(C.nelems * esz),
               "ms_per_step": round(e2e_ms / S, 2),
               "pipelining": "double-buffered device inputs/outputs; H2D(k+1) and D2H(k-1) overlap compute(k)"}
        del a_d, b_d, c_d

    peaks = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    ph = phase / args.steps
    gemm_tf = flops / (ph[2] * 1e-3) / 1e12
    gemm_alg_bytes = tk.tk_contract_roofline(A, la, B, lb, C, lc, 1e12, 1e12)["gemm_bytes"]
    perm = {}
    for i, nm in ((0, "permute_A"), (1, "permute_B"), (3, "permute_C")):
        if pbytes[i] > 0:
            gbs = pbytes[i] / (ph[i] * 1e-3) / 1e9
            perm[nm] = {"ms": round(float(ph[i]), 3), "GB_s": round(gbs, 1), "frac_of_measured_hbm": round(gbs / hbm, 3),
                        "frac_of_8TBs": round(gbs / 8000.0, 3), "bytes": int(pbytes[i])}
    perm_bytes = float(pbytes[0] + pbytes[1] + pbytes[3])
    perm_ms = float(ph[0] + ph[1] + ph[3])
    # DRAM bytes per GEMM launch from the ncu --set full capture of this build (profiles/, named per round);
    # ncu cannot run inside the timed process, so the capture's file and build are named beside the number
    traffic, traffic_src = None, None
    tfile = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            traffic = tj.get("gemm_dram_bytes_per_launch")
            traffic_src = f"profiles/r02_ncu_traffic.json ({tj.get('build', '?')})"
        except Exception:
            traffic = None
    chains = None
    if not args.no_chains and not cplx:
        chains = time_chains(dev, stream, peak_tf * 1e12, hbm * 1e9)
    svd = None
    if not args.no_svd and not cplx:
        svd = time_svd(dev, stream, oracle=(rank == 0 and world == 1 and not args.no_cpu_baseline))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not cplx:
        inputs = oracle_inputs(cfg)
        _, _, keys = oracle_sample(cfg, budget_s=args.cpu_budget_s / 2, inputs=inputs)   # calibrate + generate
        fl_s, t_s, _ = oracle_sample(cfg, 0, keys=keys, inputs=inputs)
        cpu = {"value": round(fl_s / t_s / 1e9, 4), "unit": "GFLOP/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "oracle",
               "sample": f"{len(keys)} random C output subblocks of this workload via the tier-2 charge-tuple "
                         f"einsum (oracle/blocksparse.py), {fl_s:.3e} useful flops in {t_s:.1f} s"}

    line = {
        "metric": f"useful block GFLOP/s of tk_contract ({dtype_name(args)})",
        "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded N(0,1) per subblock, workloads/gen.py)",
        "config": {"workload": f"cfg4 U(1) PEPS rank-4 x rank-4 contraction, {dtype_name(args)}, D_leg={args.d_leg} "
                               f"(reading C20)", "d_leg": args.d_leg, "parallelism": "replicas only",
                   "useful_flops_per_step": flops,
                   "l2": f"inputs ({A.nelems * esz / 1e9:.1f} GB/operand) >> 126 MB L2, no flush needed"},
        "roofline": {"bound": "tensor", "kernel": GEMM_KERNEL,
                     "achieved": round(gemm_tf, 3), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(gemm_tf / peak_tf, 4),
                     "peak_source": "this run: sustained tk_dmma_probe (FP64 DMMA, no memory traffic; "
                                    "MEASURED_PEAKS.json has no FP64 entry)", "fp64_peaks_this_run": fp64,
                     "frac_of_cublas_dgemm": round(gemm_tf / fp64["cublas_dgemm_8192_tflops"], 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": gemm_alg_bytes},
        "roofline_permute": {"bound": "hbm", "kernel": "permute_kernel (operand permutes A~, B~ and output C)",
                             "achieved": round(perm_bytes / (perm_ms * 1e-3) / 1e9, 1) if perm_ms > 0 else None,
                             "peak": hbm, "unit": "GB/s",
                             "frac": round(perm_bytes / (perm_ms * 1e-3) / 1e9 / hbm, 4) if perm_ms > 0 else None,
                             "frac_of_8TBs": round(perm_bytes / (perm_ms * 1e-3) / 1e9 / 8000.0, 4) if perm_ms > 0 else None,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs (torch copy, driver-written)",
                             "algorithmic_bytes": perm_bytes, "phases": perm},
        "chains": chains,
        "svd": svd,
        "phase_ms": {"permute_A": round(float(ph[0]), 3), "permute_B": round(float(ph[1]), 3),
                     "gemm": round(float(ph[2]), 3), "permute_C": round(float(ph[3]), 3)},
        "planner_ms": {"cold": round(t_plan_cold * 1e3, 2), "cached": round(t_plan_cached * 1e3, 4)},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "input_fill_s": round(t_fill, 2),
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "c64"],
                    help="f64: the BASELINE metric (D_leg 384); c64: cfg4's ComplexF64 variant (D_leg 320)")
    ap.add_argument("--d-leg", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="end-to-end steps (host buffers, copies inside the timed region); default: --steps")
    ap.add_argument("--cpu-budget-s", type=float, default=24.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-chains", action="store_true", help="skip the cfg2/3/5/6/7/8 chain timings")
    ap.add_argument("--no-svd", action="store_true", help="skip the two-site SVD timings (cfg2/cfg3 theta)")
    args = ap.parse_args()
    if args.e2e_steps is None:
        args.e2e_steps = args.steps
    if args.d_leg is None:
        args.d_leg = 320 if args.dtype == "c64" else 384
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
