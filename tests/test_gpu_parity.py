"""Parity of the CUDA path (through the C ABI) against the oracle -- needs a B200.

Tolerance: relative Frobenius error <= 1e-12 in Float64 (BASELINE north_star);
layouts are compared exactly elsewhere (test_library_host.py). Every output buffer
starts as NaN so that an element the kernels fail to write cannot pass.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import layout as OL, dense as OD, contract as OC, blocksparse as BS  # noqa: E402
from workloads import configs as W  # noqa: E402
from tests import harness as H  # noqa: E402

TOL = 1e-12


def rel_err_dense(layout, flat, D):
    return OC.rel_frobenius(OD.to_dense(layout, flat), D)


def rel_err_blocks(layout, flat, blocks, keys=None):
    got = BS.to_blocks(layout, flat)
    num = den = 0.0
    for k, g in got.items():
        if keys is not None and k not in keys:
            continue
        r = blocks.get(k)
        if r is None:
            r = np.zeros_like(g)
        num += float(np.sum(np.abs(g - r) ** 2))
        den += float(np.sum(np.abs(r) ** 2))
    return math.sqrt(num / den) if den > 0 else math.sqrt(num)


@pytest.mark.parametrize("cfgfun", [W.cfg1, W.cfg2, lambda: W.cfg3(chi=96), lambda: W.cfg4(d_leg=32),
                                    lambda: W.cfg5(), lambda: W.cfg5(mults=(3, 5, 4, 2, 2, 1, 1)),
                                    lambda: W.cfg6(), lambda: W.cfg6(mults=(3, 4, 3, 2, 2, 1, 1)),
                                    lambda: W.cfg7(n_mult=50), lambda: W.cfg7(n_mult=24),
                                    lambda: W.cfg8(n_mult=30), lambda: W.cfg8(n_mult=12)],
                         ids=["cfg1", "cfg2", "cfg3_chi96", "cfg4_d32", "cfg5", "cfg5_small", "cfg6", "cfg6_small",
                              "cfg7_m50", "cfg7_m24", "cfg8_m30", "cfg8_m12"])
def test_chain_dense_oracle(cfgfun):
    cfg = cfgfun()
    ref = H.oracle_chain_dense(cfg)
    got = H.gpu_chain(cfg)
    for name, (lt, D) in ref.items():
        C, flat = got[name]
        assert C.nelems == lt.nelems
        assert not np.isnan(flat).any(), f"{name}: unwritten output elements"
        err = rel_err_dense(lt, flat, D)
        assert err <= TOL, f"{name}: rel Frobenius {err:.3e}"


@pytest.mark.parametrize("cfgfun", [lambda: W.cfg3(), lambda: W.cfg4(d_leg=128)], ids=["cfg3_full", "cfg4_d128"])
def test_chain_tier2_oracle(cfgfun):
    cfg = cfgfun()
    ref = H.oracle_chain_blocks(cfg)
    got = H.gpu_chain(cfg)
    for name, (lt, blocks) in ref.items():
        C, flat = got[name]
        assert not np.isnan(flat).any()
        err = rel_err_blocks(lt, flat, blocks)
        assert err <= TOL, f"{name}: rel Frobenius {err:.3e}"


def test_alpha_beta_accumulate():
    cfg = W.cfg2(chi=128)
    cfg["steps"] = cfg["steps"][:1]
    ref = H.oracle_chain_dense(cfg)
    rng = np.random.default_rng(3)
    init = {}

    def c_init(C):
        x = rng.standard_normal(C.nelems)
        init["x"] = x
        return x

    got = H.gpu_chain(cfg, alpha=-0.75, beta=0.5, c_init=c_init)
    lt, D = ref["T1"]
    C, flat = got["T1"]
    want = -0.75 * D + 0.5 * OD.to_dense(lt, init["x"])
    assert rel_err_dense(lt, flat, want) <= TOL


# ------------------------------------------------------------------ ComplexF64 (cfg4 names it)
@pytest.mark.parametrize("cfgfun", [W.cfg1, W.cfg2, lambda: W.cfg3(chi=64), lambda: W.cfg4(d_leg=24),
                                    lambda: W.cfg5(mults=(3, 5, 4, 2, 2, 1, 1)),
                                    lambda: W.cfg6(mults=(3, 4, 3, 2, 2, 1, 1)), lambda: W.cfg7(n_mult=24),
                                    lambda: W.cfg8(n_mult=12)],
                         ids=["cfg1", "cfg2", "cfg3_chi64", "cfg4_d24", "cfg5_small", "cfg6_small", "cfg7_m24",
                              "cfg8_m12"])
def test_chain_complex_dense_oracle(cfgfun):
    """ComplexF64 through the real-representation GEMM (reading C21) against the dense oracle."""
    cfg = cfgfun()
    ref = H.oracle_chain_dense(cfg, complex_=True)
    got = H.gpu_chain(cfg, complex_=True)
    for name, (lt, D) in ref.items():
        C, flat = got[name]
        assert flat.dtype == np.complex128 and not np.isnan(flat).any(), name
        err = rel_err_dense(lt, flat, D)
        assert err <= TOL, f"{name}: rel Frobenius {err:.3e}"


@pytest.mark.parametrize("ca,cb", [(True, False), (False, True), (True, True)])
def test_complex_conj_flags(ca, cb):
    cfg = W.cfg3(chi=48)
    cfg["steps"] = cfg["steps"][:2]
    conj = {0: (ca, cb), 1: (cb, ca)}
    ref = H.oracle_chain_dense(cfg, complex_=True, conj=conj)
    got = H.gpu_chain(cfg, complex_=True, conj=conj)
    for name, (lt, D) in ref.items():
        err = rel_err_dense(lt, got[name][1], D)
        assert err <= TOL, f"{name}: rel Frobenius {err:.3e}"


def test_complex_alpha_beta():
    cfg = W.cfg4(d_leg=16)
    ref = H.oracle_chain_dense(cfg, complex_=True)
    rng = np.random.default_rng(5)
    init = {}

    def c_init(C):
        x = rng.standard_normal(C.nelems) + 1j * rng.standard_normal(C.nelems)
        init["x"] = x
        return x

    got = H.gpu_chain(cfg, alpha=0.5, beta=-1.25, c_init=c_init, complex_=True)
    lt, D = ref["C"]
    want = 0.5 * D - 1.25 * OD.to_dense(lt, init["x"])
    assert rel_err_dense(lt, got["C"][1], want) <= TOL


def _spaces(cfg):
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][0]
    A, B = cfg["tensors"][na][0], cfg["tensors"][nb][0]
    return OC.output_spaces(A["cod"], A["dom"], B["cod"], B["dom"], la, lb, lc, ncod)


# ------------------------------------------------------------------ tk_permute
def _perm_case(kind, secs, cod_d, dom_d, p, q, alpha=1.0, beta=0.0, seed=0):
    from paper_2508_10076_b200 import tk
    V = W.space(kind, secs)
    cod = [W.dual(V) if d else V for d in cod_d]
    dom = [W.dual(V) if d else V for d in dom_d]
    lt = OL.homspace_layout(kind, cod, dom)
    x = np.random.default_rng(seed).standard_normal(lt.nelems)
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    ls = OL.homspace_layout(kind, c2, d2)
    par = [OD.parity_vector(s) for s in cod + dom]
    ref = OC.permute_dense(OD.to_dense(lt, x), par, len(cod), p, q)
    A = tk.tensor_from_spec({"cod": cod, "dom": dom})
    C = tk.tensor_from_spec({"cod": c2, "dom": d2})
    a = torch.from_numpy(x).cuda()
    y0 = np.random.default_rng(seed + 1).standard_normal(ls.nelems)
    c = torch.from_numpy(y0 if beta != 0 else np.full(ls.nelems, np.nan)).cuda()
    tk.tk_permute(A, a, p, q, C, c, alpha=alpha, beta=beta)
    torch.cuda.synchronize()
    got = c.cpu().numpy()
    want = alpha * ref + (beta * OD.to_dense(ls, y0) if beta != 0 else 0)
    return OC.rel_frobenius(OD.to_dense(ls, got), want)


@pytest.mark.parametrize("kind,secs", [
    ("U1", [((-2,), 3), ((-1,), 17), ((0,), 40), ((1,), 33), ((3,), 5)]),
    ("fU1xU1", [((0, 0), 9), ((1, 1), 21), ((1, -1), 4), ((2, 0), 35), ((-1, 1), 2)]),
    ("SU2", [((0,), 5), ((1,), 3), ((2,), 4), ((3,), 2)]),
    ("Z2", [((0,), 37), ((1,), 29)]),
    ("fU1xSU2", [((0, 0), 5), ((1, 1), 3), ((-1, 1), 4), ((2, 0), 2), ((1, 3), 2)]),
    ("fSU2xSU2", [((0, 0), 4), ((1, 1), 3), ((0, 2), 2), ((2, 0), 2), ((1, 0), 2), ((0, 1), 3)]),
])
def test_permute_random(kind, secs):
    rng = np.random.default_rng(11)
    for trial in range(8):
        N = int(rng.integers(2, 5))
        n1 = int(rng.integers(0, N + 1))
        duals = [bool(x) for x in rng.integers(0, 2, N)]
        perm = list(rng.permutation(N))
        k = int(rng.integers(0, N + 1))
        if kind in ("SU2", "fU1xSU2", "fSU2xSU2") and N > 3:
            continue
        err = _perm_case(kind, secs, duals[:n1], duals[n1:], perm[:k], perm[k:],
                         alpha=float(rng.choice([1.0, -2.0])), beta=float(rng.choice([0.0, 0.5])), seed=trial)
        assert err <= TOL, (trial, N, n1, perm, k, err)


def test_permute_large_tiled_paths():
    # big extents exercise the 32x32 smem-tiled transpose (src-fastest != dst-fastest) and the rows path
    secs = [((-1,), 70), ((0,), 90), ((1,), 65)]
    assert _perm_case("U1", secs, [0, 0], [0, 0], [2, 0], [1, 3]) <= TOL   # B-operand pattern of cfg4
    assert _perm_case("U1", secs, [0, 0], [0, 0], [0, 2], [1, 3]) <= TOL   # A-operand pattern of cfg4
    assert _perm_case("U1", secs, [0, 1], [1], [2, 1, 0], []) <= TOL


# ------------------------------------------------------------------ tk_contract_tuples (explicit Alg. 4)
def _tuples_case(kind, A_sp, B_sp, tup, alpha=1.0, beta=0.0, seed=0, cplx=False, conjA=False):
    from paper_2508_10076_b200 import tk
    pA, qA, pB, qB, pAB, qAB = tup
    la = OL.homspace_layout(kind, A_sp["cod"], A_sp["dom"])
    lb = OL.homspace_layout(kind, B_sp["cod"], B_sp["dom"])
    rng = np.random.default_rng(seed)
    def draw(n):
        x = rng.standard_normal(n)
        return x + 1j * rng.standard_normal(n) if cplx else x
    xa, xb = draw(la.nelems), draw(lb.nelems)
    dt = tk.TK_C64 if cplx else tk.TK_F64
    A, B = tk.tensor_from_spec(A_sp, dt), tk.tensor_from_spec(B_sp, dt)
    C = tk.tk_contract_tuples_output(A, pA, qA, B, pB, qB, pAB, qAB)
    Asp, Bsp = A_sp["cod"] + A_sp["dom"], B_sp["cod"] + B_sp["dom"]
    at_cod, _ = OC.permuted_spaces(A_sp["cod"], A_sp["dom"], pA, qA)   # selection rule
    _, bt_dom = OC.permuted_spaces(B_sp["cod"], B_sp["dom"], pB, qB)
    cod, dom = OC.permuted_spaces(at_cod, bt_dom, pAB, qAB)
    lc = OL.homspace_layout(kind, cod, dom)
    assert C.nelems == lc.nelems
    y0 = draw(lc.nelems)
    tdt = torch.complex128 if cplx else torch.float64
    a, b = torch.from_numpy(xa).to(tdt).cuda(), torch.from_numpy(xb).to(tdt).cuda()
    c = torch.from_numpy(y0.copy()).to(tdt).cuda() if beta != 0 else torch.full((lc.nelems,), float("nan"), dtype=tdt,
                                                                                 device="cuda")
    nws = tk.tk_contract_tuples_workspace(A, pA, qA, B, pB, qB, C, pAB, qAB)
    ws = torch.empty(max(nws // 8 + 32, 1), dtype=torch.float64, device="cuda")
    tk.tk_contract_tuples(A, a, pA, qA, B, b, pB, qB, C, c, pAB, qAB, alpha=alpha, beta=beta, ws=ws,
                          ws_bytes=ws.numel() * 8, conjA=conjA)
    torch.cuda.synchronize()
    DA = OD.to_dense(la, xa)
    if conjA:
        DA = np.conj(DA)
    D = OC.contract_alg4_tuples(DA, Asp, len(A_sp["cod"]), OD.to_dense(lb, xb), Bsp, len(B_sp["cod"]),
                                pA, qA, pB, qB, pAB, qAB)
    want = alpha * D + (beta * OD.to_dense(lc, y0) if beta != 0 else 0.0)
    return OC.rel_frobenius(OD.to_dense(lc, c.cpu().numpy()), want), (A, a, B, b, C, c, ws)


_FV = [((0, 0), 3), ((1, 1), 4), ((1, -1), 2), ((2, 0), 3), ((-1, 1), 2)]
# A: V V V <- V (legs 0..3), B: V <- V V* (legs 0..2); ket/bra pairs A2-B1 and A3-B0, open A0, A1, B2
_TUPLES = [([0, 1], [2, 3], [1, 0], [2], [2, 0], [1]),      # base (= reading C2 for A[1,2,3,4] B[4,3,5] -> C[5,1;2])
           ([1, 0], [2, 3], [1, 0], [2], [2, 1], [0]),      # pA reversed (pAB compensates)
           ([0, 1], [3, 2], [0, 1], [2], [2, 0], [1]),      # contracted legs in the other order
           ([0, 1], [2, 3], [1, 0], [2], [0, 2], [1]),      # output permute crossing A1 and B2 (odd-odd signs)
           ([1, 0], [3, 2], [0, 1], [2], [1, 2], [0]),      # the same output, both reorders
           ]


@pytest.mark.parametrize("kind", ["fU1xU1", "U1xU1"])
def test_contract_tuples_vs_oracle(kind):
    V = W.space(kind, _FV)
    A_sp = {"cod": [V, V, V], "dom": [V]}
    B_sp = {"cod": [V], "dom": [V, W.dual(V)]}
    outs = []
    for i, tup in enumerate(_TUPLES):
        err, (_, _, _, _, C, c, _) = _tuples_case(kind, A_sp, B_sp, tup, seed=3)
        assert err <= TOL, (i, err)
        outs.append(c.cpu().numpy())
    # reading C13: reordering pA (with pAB) or the contracted pairs leaves C unchanged (same layout here)
    for o in outs[1:3]:
        assert np.allclose(o, outs[0], rtol=1e-13, atol=1e-13)
    assert np.allclose(outs[4], outs[3], rtol=1e-13, atol=1e-13)


def test_contract_tuples_matches_labels_path():
    """Tuples equal to reading C2's (labels A[1,2,3,4], B[4,3,5] -> C[5,1;2]) give tk_contract's result."""
    from paper_2508_10076_b200 import tk
    V = W.space("fU1xU1", _FV)
    A_sp = {"cod": [V, V, V], "dom": [V]}
    B_sp = {"cod": [V], "dom": [V, W.dual(V)]}
    err, (A, a, B, b, C, c, ws) = _tuples_case("fU1xU1", A_sp, B_sp, _TUPLES[0], seed=4)
    assert err <= TOL
    c2 = torch.full_like(c, float("nan"))
    labA, labB, labC = [1, 2, 3, 4], [4, 3, 5], [5, 1, 2]
    C2 = tk.tk_contract_output(A, labA, B, labB, labC, 2)
    assert C2.nelems == C.nelems
    nws = tk.tk_contract_workspace(A, labA, B, labB, C2, labC)
    ws2 = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
    tk.tk_contract(A, a, labA, B, b, labB, C2, c2, labC, ws=ws2, ws_bytes=ws2.numel() * 8)
    torch.cuda.synchronize()
    assert torch.equal(c, c2)


def test_contract_tuples_su2_complex():
    V = W.space("SU2", [((0,), 3), ((1,), 2), ((2,), 2)])
    A_sp = {"cod": [V, V], "dom": [V]}
    B_sp = {"cod": [V], "dom": [V, V]}
    # contract A1-B1 (V cod / V dom) and A2-B0 (V dom / V cod), contracted legs in B's order
    tup = ([0], [2, 1], [0, 1], [2], [1], [0])
    err, _ = _tuples_case("SU2", A_sp, B_sp, tup, seed=5, alpha=-0.5)
    assert err <= TOL
    err, _ = _tuples_case("SU2", A_sp, B_sp, tup, seed=6, cplx=True, conjA=True, beta=0.25)
    assert err <= TOL
    Vf = W.space("fU1xU1", _FV)
    err, _ = _tuples_case("fU1xU1", {"cod": [Vf, Vf, Vf], "dom": [Vf]}, {"cod": [Vf], "dom": [Vf, W.dual(Vf)]},
                          _TUPLES[1], seed=7, cplx=True, conjA=True)
    assert err <= TOL
