"""Pins of the blockwise-SVD oracle (oracle/svd.py), SURVEY NEXT-1 -- CPU only.

  * Wigner-Eckart block structure: the singular values of the DENSE matrix of permute(A) (rows =
    codomain multi-index, cols = domain multi-index) are exactly the block singular values, each
    repeated d_c times (for abelian kinds d_c = 1) -- an independent route through the
    dense embedding, so a wrong block extraction, permute sign or weight fails it;
  * Eckart-Young: the reported truncation error sqrt(sum_dropped d_c s^2) equals the dense Frobenius
    distance between permute(A) and its truncated reconstruction ("best rank-k approximation");
  * untruncated reconstruction is exact; MaxTotalDim keeps sum_kept d_c <= D and is greedy.
"""
import numpy as np
import pytest

from oracle import svd as OS, dense as Dn, layout as L, sectors
from workloads import configs as W


CASES = [
    ("U1", [((-2,), 2), ((0,), 3), ((1,), 2), ((3,), 1)], [0, 0], [1, 0], (0, 2), (3, 1)),
    ("Z2", [((0,), 3), ((1,), 2)], [0, 1], [0], (0, 1), (2,)),
    ("fU1xU1", [((0, 0), 2), ((1, 1), 1), ((1, -1), 2), ((-1, 1), 1)], [0, 0], [0, 1], (1, 0), (3, 2)),
    ("SU2", [((0,), 2), ((1,), 2), ((2,), 1)], [0, 0], [0], (0, 1), (2,)),
    ("SU2", [((1,), 2), ((2,), 1), ((3,), 1)], [0, 1], [0, 0], (2, 0), (1, 3)),
]


def _case(kind, secs, cod_d, dom_d, seed=0):
    V = W.space(kind, secs)
    cod = [W.dual(V) if d else V for d in cod_d]
    dom = [W.dual(V) if d else V for d in dom_d]
    lt = L.homspace_layout(kind, cod, dom)
    x = np.random.default_rng(seed).standard_normal(lt.nelems)
    return cod, dom, lt, x


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_{i}" for i, c in enumerate(CASES)])
def test_block_spectrum_equals_dense_spectrum(case):
    kind, secs, cod_d, dom_d, p, q = case
    cod, dom, lt, x = _case(kind, secs, cod_d, dom_d)
    lp, xp, Dp = OS.permuted(kind, cod, dom, x, list(p), list(q))
    rows = int(np.prod(Dp.shape[:len(p)]))
    dense_s = np.linalg.svd(Dp.reshape(rows, -1), compute_uv=False)
    blocks = []
    for c, u, s, vh in OS.block_svd(lp, xp):
        blocks.extend(list(s) * int(sectors.qdim(kind, c)))
    blocks = np.sort(np.array(blocks))[::-1]
    nz = dense_s[: len(blocks)]
    assert len(blocks) <= len(dense_s)
    assert np.allclose(blocks, nz, rtol=0, atol=1e-12 * dense_s[0])
    assert np.all(dense_s[len(blocks):] < 1e-12 * dense_s[0])


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_{i}" for i, c in enumerate(CASES)])
@pytest.mark.parametrize("max_dim,rel_tol", [(0, 0.0), (5, 0.0), (0, 0.3), (9, 0.1)])
def test_truncation_error_is_dense_distance(case, max_dim, rel_tol):
    kind, secs, cod_d, dom_d, p, q = case
    cod, dom, lt, x = _case(kind, secs, cod_d, dom_d, seed=3)
    lp, xp, Dp = OS.permuted(kind, cod, dom, x, list(p), list(q))
    svds = OS.block_svd(lp, xp)
    keep, err, nrm = OS.truncation(kind, [(c, s) for c, u, s, vh in svds], max_dim, rel_tol)
    R = Dn.to_dense(lp, OS.truncated_reconstruction(lp, svds, keep))
    assert abs(np.linalg.norm((R - Dp).ravel()) - err) <= 1e-12 * nrm
    assert abs(np.linalg.norm(Dp.ravel()) - nrm) <= 1e-12 * nrm
    kept_dim = sum(k * sectors.qdim(kind, c) for k, (c, *_r) in zip(keep, svds))
    if max_dim > 0:
        assert kept_dim <= max_dim
        # greedy: the next value in global order would not fit
        rest = sorted(((-s[k], sectors.qdim(kind, c)) for k, (c, u, s, vh) in zip(keep, svds) if k < len(s)))
        if rest and rel_tol == 0:
            assert kept_dim + rest[0][1] > max_dim
    if rel_tol > 0 and max_dim == 0:
        assert err <= rel_tol * nrm + 1e-15
    if max_dim == 0 and rel_tol == 0:
        assert err == 0.0 and np.allclose(R, Dp, atol=1e-12)


def test_fermionic_permute_signs_enter_the_spectrum():
    """The fermionic permute changes signs of subblocks, not the dense singular values of the
    unpermuted-order matrix; but the block SVD of permute(A) must still equal the dense SVD of the
    SIGNED permuted array (a sign error in the oracle's permute would mix blocks and fail)."""
    kind, secs, cod_d, dom_d, p, q = CASES[2]
    cod, dom, lt, x = _case(kind, secs, cod_d, dom_d, seed=9)
    lp, xp, Dp = OS.permuted(kind, cod, dom, x, list(p), list(q))
    back = Dn.to_dense(lp, xp)
    assert np.allclose(back, Dp, atol=1e-14)
