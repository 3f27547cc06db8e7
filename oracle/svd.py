"""Oracle for the blockwise truncated SVD of a tensor map -- TEST INFRASTRUCTURE ONLY.

Follows the paper step by step: A~ = permute(A, (p, q)) (the oracle's dense permute with reading C13's
signs, projected back onto the canonical layout of the permuted HomSpace), then "the decompositions
can be carried out block-by-block" (Alg. 9 "Abelian tensor decomposition"; eq. svd,
P:787-809): numpy's LAPACK SVD of every block matrix of A~ (the library primitive is the step). The
global truncation rule is the SPEC TruncationScheme written out as plain loops (values sorted
descending over all blocks, ties by block then block-local index; a value of block c weighs its
quantum dimension d_c; MaxTotalDim keeps greedily while sum_kept d_c <= D; RelError drops the smallest
values while sqrt(sum_dropped d_c s^2) <= eps ||A||).

Pins (tests/test_oracle_svd.py): the multiset of block singular values, each repeated d_c times,
equals the singular values of the dense matrix of permute(A) (Wigner-Eckart block structure); the
truncation error equals the dense Frobenius distance (Eckart-Young); the untruncated reconstruction
is exact.
"""
import math

import numpy as np

from . import sectors
from .contract import permute_dense, permuted_spaces
from .dense import to_dense, from_dense, parity_vector
from .layout import homspace_layout


def permuted(kind, cod, dom, flat, p, q):
    """(layout of A~, reduced flat of A~, dense A~) for A~ = permute(A, (p, q))."""
    lt = homspace_layout(kind, cod, dom)
    D = to_dense(lt, flat)
    par = [parity_vector(sp) for sp in list(cod) + list(dom)]
    Dp = permute_dense(D, par, len(cod), p, q)
    c2, d2 = permuted_spaces(cod, dom, p, q)
    lp = homspace_layout(kind, c2, d2)
    return lp, from_dense(lp, Dp), Dp


def block_matrix(layout, flat, b):
    c, rows, cols, off = layout.blocks[b]
    return np.asarray(flat[off:off + rows * cols]).reshape(rows, cols, order="F")


def block_svd(layout, flat):
    """[(coupled, u, s, vh)] per block of the layout, numpy thin SVD (s descending)."""
    out = []
    for b in range(len(layout.blocks)):
        u, s, vh = np.linalg.svd(block_matrix(layout, flat, b), full_matrices=False)
        out.append((layout.blocks[b][0], u, s, vh))
    return out


def truncation(kind, spectra, max_dim=0, rel_tol=0.0):
    """Kept count per block, truncation error and norm (the rule in the module docstring).

    spectra: [(coupled, s)] with s descending per block."""
    items = []
    n2 = 0.0
    for b, (c, s) in enumerate(spectra):
        dc = sectors.qdim(kind, c)
        for r, x in enumerate(s):
            items.append((-float(x), b, r))
            n2 += dc * float(x) ** 2
    items.sort()
    nkeep = len(items)
    if max_dim > 0:
        tot = 0.0
        i = 0
        while i < len(items):
            dc = sectors.qdim(kind, spectra[items[i][1]][0])
            if tot + dc > max_dim:
                break
            tot += dc
            i += 1
        nkeep = min(nkeep, i)
    if rel_tol > 0:
        dropped = 0.0
        i = len(items)
        while i > 0:
            negs, b, r = items[i - 1]
            w = sectors.qdim(kind, spectra[b][0]) * negs * negs
            if dropped + w > rel_tol * rel_tol * n2:
                break
            dropped += w
            i -= 1
        nkeep = min(nkeep, i)
    keep = [0] * len(spectra)
    d2 = 0.0
    for i, (negs, b, r) in enumerate(items):
        if i < nkeep:
            keep[b] += 1
        else:
            d2 += sectors.qdim(kind, spectra[b][0]) * negs * negs
    return keep, math.sqrt(d2), math.sqrt(n2)


def truncated_reconstruction(layout, svds, keep):
    """Reduced flat of sum_c u_c[:, :k] diag(s[:k]) vh_c[:k] in the layout of A~ (complex blocks give a
    complex flat)."""
    cplx = any(np.iscomplexobj(u) for _, u, _, _ in svds)
    flat = np.zeros(layout.nelems, dtype=np.complex128 if cplx else np.float64)
    for b, (c, u, s, vh) in enumerate(svds):
        k = keep[b]
        _, rows, cols, off = layout.blocks[b]
        m = (u[:, :k] * s[:k]) @ vh[:k]
        flat[off:off + rows * cols] = m.reshape(-1, order="F")
    return flat
