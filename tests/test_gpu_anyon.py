"""Planar operations on anyonic tensors (Fib, Ising) through the C ABI -- needs a B200.

tk_permute for every cyclic transpose of rank-3/4 tensors with degeneracies > 1 against the planar
oracle (oracle/planar.py, pinned in tests/test_oracle_planar.py), and a planar contraction
(Alg. 4 with planar permutes: bends and a rotation of the output) against the oracle's
contract_planar. Relative Frobenius error on the reduced data (anyons have no dense embedding).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import planar as OP, layout as OL  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12
SECS = {"Fib": [((0,), 3), ((1,), 5)], "Ising": [((0,), 4), ((1,), 3), ((2,), 2)]}


def _cyclic(n1, N, r, n1p):
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    T = [S[(i + r) % N] for i in range(N)]
    return T[:n1p], list(reversed(T[n1p:]))


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("kind", ["Fib", "Ising"])
def test_planar_permute(kind):
    from paper_2508_10076_b200 import tk
    V = W.space(kind, SECS[kind])
    Vd = W.dual(V)
    rng = np.random.default_rng(4)
    for cod, dom in (([V, Vd], [V]), ([V, V], [Vd, V]), ([V], [V, Vd, V])):
        lt = OL.homspace_layout(kind, cod, dom)
        x = rng.standard_normal(lt.nelems)
        n1, N = len(cod), len(cod) + len(dom)
        for r in range(N):
            for n1p in range(N + 1):
                p, q = _cyclic(n1, N, r, n1p)
                ref, ls = OP.apply_planar(kind, cod, dom, x, p, q)
                A = tk.tensor_from_spec({"cod": cod, "dom": dom})
                C = tk.tensor_from_spec({"cod": ls.cod, "dom": ls.dom})
                a = torch.from_numpy(x).cuda()
                c = torch.full((ls.nelems,), float("nan"), dtype=torch.float64, device="cuda")
                tk.tk_permute(A, a, p, q, C, c)
                torch.cuda.synchronize()
                got = c.cpu().numpy()
                assert not np.isnan(got).any()
                assert _rel(got, ref) <= TOL, (cod, dom, p, q)


@pytest.mark.parametrize("kind", ["Fib", "Ising"])
@pytest.mark.parametrize("labC,ncod", [([1, 2, 4], 2), ([2, 4, 1], 2), ([4, 2, 1], 1)])
def test_planar_contraction(kind, labC, ncod):
    """C[labC] = A(a, b; c) B(c; d): identity operand permutes, a planar output rotation."""
    from paper_2508_10076_b200 import tk
    V = W.space(kind, SECS[kind])
    A_sp = {"cod": [V, V], "dom": [V]}
    B_sp = {"cod": [V], "dom": [V]}
    labA, labB = [1, 2, 3], [3, 4]
    la = OL.homspace_layout(kind, A_sp["cod"], A_sp["dom"])
    lb = OL.homspace_layout(kind, B_sp["cod"], B_sp["dom"])
    rng = np.random.default_rng(9)
    xa, xb = rng.standard_normal(la.nelems), rng.standard_normal(lb.nelems)
    ref, lc = OP.contract_planar(kind, A_sp, xa, labA, B_sp, xb, labB, labC, ncod)
    A, B = tk.tensor_from_spec(A_sp), tk.tensor_from_spec(B_sp)
    C = tk.tk_contract_output(A, labA, B, labB, labC, ncod)
    assert C.nelems == lc.nelems
    a, b = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    c = torch.full((C.nelems,), float("nan"), dtype=torch.float64, device="cuda")
    nws = tk.tk_contract_workspace(A, labA, B, labB, C, labC)
    ws = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
    tk.tk_contract(A, a, labA, B, b, labB, C, c, labC, ws=ws, ws_bytes=ws.numel() * 8)
    torch.cuda.synchronize()
    got = c.cpu().numpy()
    assert not np.isnan(got).any()
    assert _rel(got, ref) <= TOL
