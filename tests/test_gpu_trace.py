"""Partial traces through the C ABI (tk_trace) against the oracle -- needs a B200.

Bosonic kinds against the plain dense trace (oracle.contract.partial_trace_dense), anyons against the
tree-level planar oracle (oracle.planar.trace_planar); degeneracies > 1 so the diagonal sums run over
real extents; alpha / beta accumulate. 1e-12 relative Frobenius.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import layout as OL, dense as OD, contract as OC, planar as OP  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12


def _run(kind, cod, dom, x, pt, qt, p, q, alpha=1.0, beta=0.0, c0=None):
    from paper_2508_10076_b200 import tk
    cplx = np.iscomplexobj(x)
    dt, tdt = (tk.TK_C64, torch.complex128) if cplx else (tk.TK_F64, torch.float64)
    A = tk.tensor_from_spec({"cod": cod, "dom": dom}, dt)
    C = tk.tk_trace_output(A, pt, qt, p, q)
    nws = tk.tk_trace_workspace(A, pt, qt, p, q, C)
    ws = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
    a = torch.from_numpy(x).cuda()
    c = torch.from_numpy(c0.copy()).cuda() if c0 is not None else torch.full((C.nelems,), float("nan"),
                                                                            dtype=tdt, device="cuda")
    tk.tk_trace(A, a, pt, qt, p, q, C, c, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8)
    torch.cuda.synchronize()
    return c.cpu().numpy()


@pytest.mark.parametrize("kind,secs", [("U1", [((-1,), 3), ((0,), 5), ((2,), 2)]), ("Z2", [((0,), 4), ((1,), 3)]),
                                       ("SU2", [((0,), 2), ((1,), 3), ((2,), 2)]),
                                       ("U1xU1", [((0, 0), 2), ((1, 1), 3), ((-1, -1), 2)])])
def test_trace_dense(kind, secs):
    V = W.space(kind, secs)
    Vd = W.dual(V)
    rng = np.random.default_rng(2)
    for cod, dom, pt, qt, p, q in (([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [0], [3], [1], [2]),
                                   ([V, Vd, V], [V, V], [2], [4], [1, 0], [3]),
                                   ([V, V], [V, V], [0, 1], [2, 3], [], []),
                                   ([V, Vd, V], [V], [0], [1], [2], [3])):
        lt = OL.homspace_layout(kind, cod, dom)
        x = rng.standard_normal(lt.nelems)
        R, c2, d2 = OC.partial_trace_dense(OD.to_dense(lt, x), cod, dom, pt, qt, p, q)
        lc = OL.homspace_layout(kind, c2, d2)
        y0 = rng.standard_normal(lc.nelems)
        got = _run(kind, cod, dom, x, pt, qt, p, q, alpha=0.5, beta=-2.0, c0=y0)
        want = 0.5 * R - 2.0 * OD.to_dense(lc, y0)
        assert OC.rel_frobenius(OD.to_dense(lc, got), want) <= TOL, (pt, qt, p, q)


@pytest.mark.parametrize("kind,secs", [("Fib", [((0,), 3), ((1,), 4)]), ("Ising", [((0,), 3), ((1,), 2), ((2,), 2)])])
def test_trace_anyon(kind, secs):
    V = W.space(kind, secs)
    rng = np.random.default_rng(3)
    for cod, dom, pt, qt, p, q in (([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [2], [0], [1, 3], []),
                                   ([V, V], [V, V], [0, 1], [2, 3], [], [])):
        lt = OL.homspace_layout(kind, cod, dom)
        x = rng.standard_normal(lt.nelems)
        ref, lc = OP.trace_planar(kind, cod, dom, x, pt, qt, p, q)
        got = _run(kind, cod, dom, x, pt, qt, p, q)
        assert not np.isnan(got).any()
        assert np.linalg.norm(got - ref) <= TOL * max(np.linalg.norm(ref), 1e-300)


@pytest.mark.parametrize("kind,secs", [("U1", [((-1,), 3), ((0,), 5), ((2,), 2)]),
                                       ("SU2", [((0,), 2), ((1,), 3), ((2,), 2)])])
def test_trace_complex(kind, secs):
    """ComplexF64 traces (interleaved; the trace coefficients are real)."""
    V = W.space(kind, secs)
    rng = np.random.default_rng(4)
    for cod, dom, pt, qt, p, q in (([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [0, 1], [2, 3], [], [])):
        lt = OL.homspace_layout(kind, cod, dom)
        x = rng.standard_normal(lt.nelems) + 1j * rng.standard_normal(lt.nelems)
        R, c2, d2 = OC.partial_trace_dense(OD.to_dense(lt, x), cod, dom, pt, qt, p, q)
        lc = OL.homspace_layout(kind, c2, d2)
        y0 = rng.standard_normal(lc.nelems) + 1j * rng.standard_normal(lc.nelems)
        got = _run(kind, cod, dom, x, pt, qt, p, q, alpha=0.5, beta=-2.0, c0=y0)
        want = 0.5 * R - 2.0 * OD.to_dense(lc, y0)
        assert OC.rel_frobenius(OD.to_dense(lc, got), want) <= TOL, (pt, qt, p, q)
