"""Shared test harness: run a config through the CUDA path and through the oracle.

CUDA side: library tensors, inputs placed by the library's layout (layout_io),
tk_contract on the current stream, result copied back as a flat buffer.
Oracle side: the oracle's own layout, the same keyed seeded values, dense
embedding + einsum (tier 1) or charge-tuple einsum (tier 2).
"""
import math

import numpy as np

from oracle import layout as OL, dense as OD, contract as OC, blocksparse as BS
from workloads import gen


# ------------------------------------------------------------------ oracle side
def oracle_flat(layout, cfg, tidx, complex_=False):
    flat = np.zeros(layout.nelems, dtype=np.complex128 if complex_ else np.float64)
    for sb in layout.subblocks:
        n = math.prod(sb.extents)
        v = gen.subblock_values(cfg, tidx, sb.key, n, complex_)
        OD.subblock_array(layout, flat, sb)[...] = v.reshape(sb.extents, order="F")
    return flat


def oracle_chain_dense(cfg, complex_=False, conj=None):
    """Tier 1: dense results of every step of a config. Returns {name: (layout, dense)}.

    complex_: ComplexF64 inputs; conj: {step index: (conjA, conjB)} -- elementwise complex
    conjugation of that step's operands (tk_contract's conjA / conjB)."""
    kind = cfg["kind"]
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        lt = OL.homspace_layout(kind, spec["cod"], spec["dom"])
        T[name] = (spec["cod"], spec["dom"], lt, OD.to_dense(lt, oracle_flat(lt, cfg["cfg"], idx, complex_)))
    out = {}
    for si, (na, la, nb, lb, nc, lc, ncod) in enumerate(cfg["steps"]):
        Ac, Ad, _, A = T[na]
        Bc, Bd, _, B = T[nb]
        ca, cb = (conj or {}).get(si, (False, False))
        A = np.conj(A) if ca else A
        B = np.conj(B) if cb else B
        D = OC.contract(kind, A, Ac + Ad, len(Ac), la, B, Bc + Bd, len(Bc), lb, lc, ncod)
        cod, dom = OC.output_spaces(Ac, Ad, Bc, Bd, la, lb, lc, ncod)
        lt = OL.homspace_layout(kind, cod, dom)
        T[nc] = (cod, dom, lt, D)
        out[nc] = (lt, D)
    return out


LazyBlocks = BS.LazyBlocks


def oracle_chain_blocks(cfg, out_keys_last=None, complex_=False):
    """Tier 2 (abelian): charge-tuple einsum through the chain. Returns {name: (layout, blocks)}."""
    kind = cfg["kind"]
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        lt = OL.homspace_layout(kind, spec["cod"], spec["dom"])
        T[name] = (spec["cod"], spec["dom"], LazyBlocks(lt, cfg["cfg"], idx, complex_))
    out = {}
    steps = cfg["steps"]
    for si, (na, la, nb, lb, nc, lc, ncod) in enumerate(steps):
        Ac, Ad, Ab = T[na]
        Bc, Bd, Bb = T[nb]
        keys = out_keys_last if si == len(steps) - 1 else None
        blocks, (cod, dom) = BS.contract_blocks(kind, Ab, Ac, Ad, la, Bb, Bc, Bd, lb, lc, ncod, out_keys=keys)
        T[nc] = (cod, dom, blocks)
        out[nc] = (OL.homspace_layout(kind, cod, dom), blocks)
    return out


def flat_blocks(layout, flat):
    return BS.to_blocks(layout, flat)


# ------------------------------------------------------------------ CUDA side
def gpu_chain(cfg, alpha=1.0, beta=0.0, c_init=None, keep=True, complex_=False, conj=None):
    """Run every step of cfg through tk_contract. Returns {name: (tk.Tensor, host flat)}."""
    import torch
    from paper_2508_10076_b200 import tk, layout_io
    dev = torch.device("cuda")
    dt = torch.complex128 if complex_ else torch.float64
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        t = tk.tensor_from_spec(spec, tk.TK_C64 if complex_ else tk.TK_F64)
        flat = layout_io.fill(t, cfg["cfg"], idx, complex_)
        T[name] = (t, torch.from_numpy(flat).to(dev))
    out = {}
    for si, (na, la, nb, lb, nc, lc, ncod) in enumerate(cfg["steps"]):
        ca, cb = (conj or {}).get(si, (False, False))
        A, a = T[na]
        B, b = T[nb]
        C = tk.tk_contract_output(A, la, B, lb, lc, ncod)
        if c_init is not None:
            c = torch.from_numpy(c_init(C)).to(dev)
        else:
            c = torch.full((C.nelems,), float("nan"), dtype=dt, device=dev)
        ws_n = tk.tk_contract_workspace(A, la, B, lb, C, lc)
        ws = torch.empty(max(ws_n // 8 + 32, 1), dtype=torch.float64, device=dev)
        tk.tk_contract(A, a, la, B, b, lb, C, c, lc, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8,
                       conjA=ca, conjB=cb)
        torch.cuda.synchronize()
        T[nc] = (C, c)
        out[nc] = (C, c.cpu().numpy() if keep else None)
    return out


def gpu_chain_fused(cfg, alpha=1.0, beta=0.0, c_init=None):
    """Like gpu_chain, but every consecutive pair (step i's output is step i+1's A operand) that
    tk_contract2 runs as ONE kernel goes through tk_contract2 (its intermediate is then absent from the
    result). Returns ({name: (tk.Tensor, host flat)}, [fused step indices]). alpha / beta / c_init apply
    to the last call that writes each output, as in gpu_chain."""
    import torch
    from paper_2508_10076_b200 import tk, layout_io
    dev = torch.device("cuda")
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        t = tk.tensor_from_spec(spec)
        T[name] = (t, torch.from_numpy(layout_io.fill(t, cfg["cfg"], idx)).to(dev))
    steps = cfg["steps"]
    desc = {}
    for (na, la, nb, lb, nc, lc, ncod) in steps:
        A = desc.get(na, T[na][0] if na in T else None)
        desc[nc] = tk.tk_contract_output(A, la, desc.get(nb, T[nb][0] if nb in T else None), lb, lc, ncod)
    out, fused = {}, []

    def new_out(C):
        if c_init is not None:
            return torch.from_numpy(c_init(C)).to(dev)
        return torch.full((C.nelems,), float("nan"), dtype=torch.float64, device=dev)

    i = 0
    while i < len(steps):
        na, la, nb, lb, nc, lc, ncod = steps[i]
        if i + 1 < len(steps) and steps[i + 1][0] == nc:
            _, la2, nb2, lb2, nc2, lc2, _ = steps[i + 1]
            Tm, C = desc[nc], desc[nc2]
            n, fu = tk.tk_contract2_workspace(T[na][0], la, T[nb][0], lb, Tm, lc, T[nb2][0], lb2, C, lc2,
                                              want_fused=True)
            if fu:
                c = new_out(C)
                ws = torch.empty(max(n // 8 + 32, 1), dtype=torch.float64, device=dev)
                tk.tk_contract2(T[na][0], T[na][1], la, T[nb][0], T[nb][1], lb, Tm, lc, T[nb2][0], T[nb2][1], lb2,
                                C, c, lc2, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8)
                torch.cuda.synchronize()
                T[nc2] = (C, c)
                out[nc2] = (C, c.cpu().numpy())
                fused.append(i)
                i += 2
                continue
        A, a = T[na]
        B, b = T[nb]
        C = desc[nc]
        c = new_out(C)
        n = tk.tk_contract_workspace(A, la, B, lb, C, lc)
        ws = torch.empty(max(n // 8 + 32, 1), dtype=torch.float64, device=dev)
        tk.tk_contract(A, a, la, B, b, lb, C, c, lc, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8)
        torch.cuda.synchronize()
        T[nc] = (C, c)
        out[nc] = (C, c.cpu().numpy())
        i += 1
    return out, fused
