"""Blockwise truncated SVD through the C ABI (tk_svd / tk_svd_truncate / tk_svd_extract) against the
oracle (oracle/svd.py) -- needs a B200. SURVEY NEXT-1.

Compared: every block's singular values (relative to the largest, 1e-12), the kept counts and the
truncation error of the global rule, U S Vh against the oracle's truncated reconstruction (relative
Frobenius 1e-12 on the dense embedding; U, Vh themselves are unique only up to signs), and the
isometry of U and Vh block by block.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import svd as OS, dense as OD, contract as OC, layout as OL  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12


def _run(kind, cod, dom, x, p, q, max_dim=0, rel_tol=0.0):
    from paper_2508_10076_b200 import tk
    cplx = np.iscomplexobj(x)
    A = tk.tensor_from_spec({"cod": cod, "dom": dom}, tk.TK_C64 if cplx else tk.TK_F64)
    a = torch.from_numpy(x).cuda()
    nb = tk.tk_svd_workspace(A, p, q)
    ws = torch.empty(nb // 8 + 64, dtype=torch.float64, device="cuda")
    tk.tk_svd(A, a, p, q, ws, ws.numel() * 8)
    spec = tk.tk_svd_spectrum(A, p, q, ws)
    Wsp, U, S, Vh, err, nrm = tk.tk_svd_truncate(A, p, q, ws, max_dim, rel_tol)
    bufs = [torch.full((T.nelems,), float("nan"), dtype=torch.complex128 if cplx else torch.float64, device="cuda")
            for T in (U, S, Vh)]
    tk.tk_svd_extract(A, p, q, ws, U, bufs[0], S, bufs[1], Vh, bufs[2])
    torch.cuda.synchronize()
    wsec, wdeg = Wsp.sectors()
    return spec, dict(zip(wsec, (int(d) for d in wdeg))), err, nrm, [b.cpu().numpy() for b in bufs]


def _check(kind, cod, dom, x, p, q, max_dim=0, rel_tol=0.0):
    lp, xp, Dp = OS.permuted(kind, cod, dom, x, list(p), list(q))
    svds = OS.block_svd(lp, xp)
    keep, err_ref, nrm_ref = OS.truncation(kind, [(c, s) for c, u, s, vh in svds], max_dim, rel_tol)
    spec, wdeg, err, nrm, (u, s, vh) = _run(kind, cod, dom, x, p, q, max_dim, rel_tol)
    # spectra, block by block (both sides list A~'s blocks by ascending coupled label)
    assert len(spec) == len(svds)
    smax = max(float(sv[0]) for _, _, sv, _ in svds if len(sv))
    for got, (c, _, ref, _) in zip(spec, svds):
        assert got.shape == ref.shape
        assert np.abs(got - ref).max(initial=0.0) <= TOL * smax, c
    # truncation decision
    assert {tuple(c): k for (c, *_r), k in zip(svds, keep) if k} == wdeg
    assert abs(err - err_ref) <= TOL * nrm_ref and abs(nrm - nrm_ref) <= TOL * nrm_ref
    assert not (np.isnan(u).any() or np.isnan(s).any() or np.isnan(vh).any())
    # U S Vh == truncated reconstruction (dense embedding; the bond space W from the kept counts)
    Wspace = W.space(kind, [(c, k) for c, k in wdeg.items()])
    lu = OL.homspace_layout(kind, lp.cod, [Wspace])
    ls = OL.homspace_layout(kind, [Wspace], [Wspace])
    lv = OL.homspace_layout(kind, [Wspace], lp.dom)
    n1, n2 = len(lp.cod), len(lp.dom)
    labU = list(range(1, n1 + 1)) + [100]
    labV = [101] + list(range(n1 + 1, n1 + n2 + 1))
    US = OC.contract_einsum(OD.to_dense(lu, u), labU, OD.to_dense(ls, s), [100, 101], labU[:-1] + [101])
    R = OC.contract_einsum(US, labU[:-1] + [101], OD.to_dense(lv, vh), labV, list(range(1, n1 + n2 + 1)))
    ref = OD.to_dense(lp, OS.truncated_reconstruction(lp, svds, keep))
    assert OC.rel_frobenius(R, ref) <= TOL * max(1.0, nrm_ref / max(np.linalg.norm(ref), 1e-300))
    # isometries, block by block: U^T U = 1, Vh Vh^T = 1
    for (c, rows, cols, off) in lu.blocks:
        m = u[off:off + rows * cols].reshape(rows, cols, order="F")
        assert np.abs(m.conj().T @ m - np.eye(cols)).max() <= 1e-12
    for (c, rows, cols, off) in lv.blocks:
        m = vh[off:off + rows * cols].reshape(rows, cols, order="F")
        assert np.abs(m @ m.conj().T - np.eye(rows)).max() <= 1e-12


CASES = [
    ("U1", [((-2,), 5), ((0,), 7), ((1,), 4), ((3,), 3)], [0, 0], [1, 0], [0, 2], [3, 1]),
    ("Z2", [((0,), 9), ((1,), 6)], [0, 1], [0], [0, 1], [2]),
    ("fU1xU1", [((0, 0), 4), ((1, 1), 3), ((1, -1), 5), ((-1, 1), 2)], [0, 0], [0, 1], [1, 0], [3, 2]),
    ("SU2", [((0,), 5), ((1,), 4), ((2,), 3)], [0, 0], [0], [0, 1], [2]),
    ("SU2", [((1,), 3), ((2,), 2), ((3,), 2)], [0, 1], [0, 0], [2, 0], [1, 3]),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_{i}" for i, c in enumerate(CASES)])
@pytest.mark.parametrize("max_dim,rel_tol", [(0, 0.0), (12, 0.0), (0, 0.25)])
def test_svd_small(case, max_dim, rel_tol):
    kind, secs, cod_d, dom_d, p, q = case
    V = W.space(kind, secs)
    cod = [W.dual(V) if d else V for d in cod_d]
    dom = [W.dual(V) if d else V for d in dom_d]
    lt = OL.homspace_layout(kind, cod, dom)
    x = np.random.default_rng(7).standard_normal(lt.nelems)
    _check(kind, cod, dom, x, p, q, max_dim, rel_tol)


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_{i}" for i, c in enumerate(CASES)])
@pytest.mark.parametrize("max_dim,rel_tol", [(0, 0.0), (12, 0.0)])
def test_svd_small_complex(case, max_dim, rel_tol):
    """ComplexF64 (unitary Jacobi: column q rephased by conj(gamma / |gamma|), then a real rotation)."""
    kind, secs, cod_d, dom_d, p, q = case
    V = W.space(kind, secs)
    cod = [W.dual(V) if d else V for d in cod_d]
    dom = [W.dual(V) if d else V for d in dom_d]
    lt = OL.homspace_layout(kind, cod, dom)
    rng = np.random.default_rng(8)
    x = rng.standard_normal(lt.nelems) + 1j * rng.standard_normal(lt.nelems)
    _check(kind, cod, dom, x, p, q, max_dim, rel_tol)


def test_svd_rank_deficient_and_graded():
    """Blocks of low rank (exact zero singular values) and with singular values spread over 12 decades:
    the spectrum stays accurate to eps ||A|| and U, Vh stay isometric."""
    V = W.space("U1", [((-1,), 20), ((0,), 33), ((1,), 17)])
    cod, dom = [V, V], [V]
    lt = OL.homspace_layout("U1", cod, dom)
    rng = np.random.default_rng(11)
    x = np.zeros(lt.nelems)
    for (c, rows, cols, off) in lt.blocks:
        r = max(1, min(rows, cols) // 3)
        m = rng.standard_normal((rows, r)) @ np.diag(10.0 ** -rng.uniform(0, 12, r)) @ rng.standard_normal((r, cols))
        x[off:off + rows * cols] = m.reshape(-1, order="F")
    _check("U1", cod, dom, x, [0, 1], [2], 0, 0.0)


def test_svd_block_larger_than_2048():
    """A single 2200 x 2100 block (min(rows, cols) > 2048: the round-1 limit) runs on an 8-CTA cluster
    with its rows in the workspace."""
    V = W.space("U1", [((0,), 2200)])
    Wd = W.space("U1", [((0,), 2100)])
    lt = OL.homspace_layout("U1", [V], [Wd])
    x = np.random.default_rng(12).standard_normal(lt.nelems)
    _check("U1", [V], [Wd], x, [0], [1], 1000, 0.0)


def _two_site(cfg):
    from tests import harness as H
    spec, idx = cfg["tensors"]["theta"]
    lt = OL.homspace_layout(cfg["kind"], spec["cod"], spec["dom"])
    return spec["cod"], spec["dom"], H.oracle_flat(lt, cfg["cfg"], idx)


@pytest.mark.parametrize("cfgfun,max_dim", [(lambda: W.cfg2(), 512), (lambda: W.cfg2(chi=128), 0),
                                            (lambda: W.cfg3(chi=256), 256)], ids=["cfg2", "cfg2_full", "cfg3"])
def test_svd_two_site(cfgfun, max_dim):
    """The two-site benchmark's truncated SVD (Alg. 12): theta (alpha, s1 ; s2, beta)
    split as (alpha, s1) | (s2, beta) and truncated back to the bond dimension."""
    cfg = cfgfun()
    cod, dom, x = _two_site(cfg)
    _check(cfg["kind"], cod, dom, x, [0, 1], [2, 3], max_dim)


@pytest.mark.parametrize("cfgfun,max_dim", [(lambda: W.cfg2(), 512), (lambda: W.cfg3(chi=256), 256)],
                         ids=["cfg2", "cfg3"])
def test_svd_two_site_complex(cfgfun, max_dim):
    cfg = cfgfun()
    cod, dom, x = _two_site(cfg)
    xi = np.random.default_rng(13).standard_normal(x.shape)
    _check(cfg["kind"], cod, dom, x + 1j * xi, [0, 1], [2, 3], max_dim)


def test_svd_su2_mps():
    cfg = W.cfg6(mults=(6, 9, 8, 6, 4, 3, 2))
    from tests import harness as H
    spec, idx = cfg["tensors"]["A"]
    lt = OL.homspace_layout("SU2", spec["cod"], spec["dom"])
    x = H.oracle_flat(lt, cfg["cfg"], idx)
    _check("SU2", spec["cod"], spec["dom"], x, [0, 1], [2], 20)
    _check("SU2", spec["cod"], spec["dom"], x, [0], [1, 2], 0, 1e-3)


def _check_blocks(kind, cod, dom, x, p, q):
    """Untruncated SVD at the timed sizes, compared block by block (the dense embedding of an
    8192 x 8192 two-site matrix is too large for the oracle's einsum): every block's spectrum against
    numpy LAPACK (1e-12 sigma_max), U_c S_c Vh_c against the oracle's permuted block (1e-12 relative to
    ||A||), and the isometry of U_c and Vh_c."""
    lp, xp, _ = OS.permuted(kind, cod, dom, x, list(p), list(q))
    svds = OS.block_svd(lp, xp)
    spec, wdeg, err, nrm, (u, s, vh) = _run(kind, cod, dom, x, p, q, 0, 0.0)
    smax = max(float(sv[0]) for _, _, sv, _ in svds if len(sv))
    anorm = float(np.linalg.norm(xp))
    assert len(spec) == len(svds)
    for got, (c, _, ref, _) in zip(spec, svds):
        assert np.abs(got - ref).max(initial=0.0) <= TOL * smax, c
    Wspace = W.space(kind, [(c, k) for c, k in wdeg.items()])
    lu = OL.homspace_layout(kind, lp.cod, [Wspace])
    ls = OL.homspace_layout(kind, [Wspace], [Wspace])
    lv = OL.homspace_layout(kind, [Wspace], lp.dom)
    ub = {c: (r, k, o) for c, r, k, o in lu.blocks}
    sb = {c: (k, o) for c, k, _, o in ls.blocks}
    vb = {c: (k, n, o) for c, k, n, o in lv.blocks}
    worst = 0.0
    for (c, rows, cols, off) in lp.blocks:
        m = xp[off:off + rows * cols].reshape(rows, cols, order="F")
        r, k, uo = ub[c]
        mu = u[uo:uo + r * k].reshape(r, k, order="F")
        ms = s[sb[c][1]:sb[c][1] + k * k].reshape(k, k, order="F")
        k2, n, vo = vb[c]
        mv = vh[vo:vo + k2 * n].reshape(k2, n, order="F")
        worst = max(worst, np.linalg.norm(mu @ ms @ mv - m))
        assert np.abs(mu.conj().T @ mu - np.eye(k)).max() <= 1e-12, c
        assert np.abs(mv @ mv.conj().T - np.eye(k2)).max() <= 1e-12, c
    assert worst <= TOL * anorm, worst / anorm


@pytest.mark.parametrize("cfgname", ["cfg2", "cfg3", "cfg7", "cfg8"])
def test_svd_two_site_full_size(cfgname):
    """The two-site tensors at the sizes tools/bench_svd.py times (blocks up to 181 x 181 for cfg3):
    the tile kernel at every cluster size the planner picks."""
    cfg = getattr(W, cfgname)()
    cod, dom, x = _two_site(cfg)
    _check_blocks(cfg["kind"], cod, dom, x, [0, 1], [2, 3])


def test_svd_two_site_full_size_complex():
    cfg = W.cfg3()
    cod, dom, x = _two_site(cfg)
    xi = np.random.default_rng(14).standard_normal(x.shape)
    _check_blocks(cfg["kind"], cod, dom, x + 1j * xi, [0, 1], [2, 3])


# (rows, cols) of a single block: tile kernel at RG 1..8 and cluster sizes 1..8, ragged row tiles, odd
# K (a player sits out), wide blocks (G = A~^H); K > 192 or more than 64 rows per CTA (32 complex) at
# CS 8 go to the shared-memory / workspace cluster kernel
TILE_SHAPES = [(1, 1), (7, 3), (3, 7), (33, 33), (64, 17), (130, 129), (181, 181), (192, 192), (511, 180),
               (513, 100), (200, 193), (300, 257)]


@pytest.mark.parametrize("shape", TILE_SHAPES, ids=[f"{r}x{c}" for r, c in TILE_SHAPES])
@pytest.mark.parametrize("cplx", [False, True], ids=["f64", "c64"])
def test_svd_tile_shapes(shape, cplx):
    rows, cols = shape
    V = W.space("U1", [((0,), rows)])
    Wd = W.space("U1", [((0,), cols)])
    lt = OL.homspace_layout("U1", [V], [Wd])
    rng = np.random.default_rng(rows * 1000 + cols)
    x = rng.standard_normal(lt.nelems)
    if cplx:
        x = x + 1j * rng.standard_normal(lt.nelems)
    _check_blocks("U1", [V], [Wd], x, [0], [1])
