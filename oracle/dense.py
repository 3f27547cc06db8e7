"""Dense embedding of symmetric tensors (oracle side; test infrastructure).

Leg basis: the dense index of a leg runs over the
UNDERLYING space V's sectors in ascending label order; sector a occupies
n_a * d_a consecutive indices, index = off(a) + i * d_a + mu (outer i, inner
mu, m = j - mu). A dual leg V* uses the same index set with dual-basis meaning,
so contracting a V leg with a V* leg is a plain index contraction (the
evaluation map of P:339-344 is delta_ij in the computational basis).

Abelian (Eq. abeliantensorzeros): D[i_1..i_N] = reduced value inside
allowed charge tuples, zero elsewhere.

SU(2) (Wigner-Eckart; canonical trees P:1461-1495; Z on dual legs
P:1649-1654 with reading C7):
    D = sum_{(s,f)} R_{s,f} (x) (X_s o X_f^dagger)
where X_s is the product of CG splitting tensors along the left-to-right tree,
Z^dagger applied on codomain dual legs and Z on domain dual legs.
"""
import math

import numpy as np

from . import sectors, su2
from .layout import underlying, subblock_index


def leg_basis(sp):
    """(dict sector -> (offset, n, d), total dim) for one leg."""
    kind = sp["kind"]
    off = 0
    out = {}
    for lab, n in sorted(sp["sectors"]):
        d = sectors.qdim(kind, lab)
        out[tuple(lab)] = (off, n, d)
        off += n * d
    return out, off


def _splitting_tensor_su2(js_unc, js_chain):
    """X[mu_1..mu_N, mu_c] of ONE SU(2) factor along the canonical left-to-right tree (doubled spins;
    js_chain = inner labels then the coupled label)."""
    n = len(js_unc)
    if n == 0:
        return np.ones((1,))
    if n == 1:
        return np.eye(js_unc[0] + 1)
    X = su2.cg_tensor(js_unc[0], js_unc[1], js_chain[0])
    for k in range(2, n):
        C = su2.cg_tensor(js_chain[k - 2], js_unc[k], js_chain[k - 1])
        X = np.tensordot(X, C, axes=([X.ndim - 1], [0]))
    return X


def _kron_axes(Xs):
    """Per-axis Kronecker product of equal-rank tensors: index mu = (mu_1 * d_2 + mu_2) per axis."""
    X = Xs[0]
    for Y in Xs[1:]:
        nd = X.ndim
        Z = np.multiply.outer(X, Y)
        Z = Z.transpose([a for k in range(nd) for a in (k, nd + k)])
        X = Z.reshape([X.shape[k] * Y.shape[k] for k in range(nd)])
    return X


def _splitting_tensor(kind, uncoupled, inner, coupled):
    """X[mu_1..mu_N, mu_c] for the canonical left-to-right tree: the Kronecker product over the
    SU(2) factors of the kind (Deligne product); a U(1) factor is one-dimensional and
    only selects the sector."""
    chain = list(inner) + [coupled]
    nf = len(sectors.spins2(kind, coupled))
    parts = []
    for f in range(nf):
        js_unc = [sectors.spins2(kind, a)[f] for a in uncoupled]
        js_chain = [sectors.spins2(kind, a)[f] for a in chain]
        parts.append(_splitting_tensor_su2(js_unc, js_chain))
    return _kron_axes(parts)


def _z_flip(kind, X, axis, lab):
    """Z (reading C7) on one leg: the Kronecker product of the factors' Z."""
    js = sectors.spins2(kind, lab)
    if len(js) == 1:
        return su2.z_flip(X, axis, js[0])
    dims = [j + 1 for j in js]
    sh = list(X.shape)
    Y = X.reshape(sh[:axis] + dims + sh[axis + 1:])
    for f, j in enumerate(js):
        Y = su2.z_flip(Y, axis + f, j)
    return Y.reshape(sh)


def basis_tensor(kind, cod, dom, key):
    """Dense basis element X_s o X_f^dagger of tree pair `key`, shape (d_cod..., d_dom...)."""
    s_unc, s_inn, c, f_unc, f_inn = key
    Xs = _splitting_tensor(kind, s_unc, s_inn, c)
    Xf = _splitting_tensor(kind, f_unc, f_inn, c)
    for k, sp in enumerate(cod):
        if sp["dual"]:
            Xs = _z_flip(kind, Xs, k, s_unc[k])
    for k, sp in enumerate(dom):
        if sp["dual"]:
            Xf = _z_flip(kind, Xf, k, f_unc[k])
    return np.tensordot(Xs, Xf, axes=([Xs.ndim - 1], [Xf.ndim - 1]))


def _dense_slices(layout, sb):
    """Per-leg (offset, n, d) of the dense region a subblock occupies."""
    legs = layout.cod + layout.dom
    key = sb.key
    labels = list(key[0]) + list(key[3])
    out = []
    for sp, lab in zip(legs, labels):
        basis, _ = leg_basis(sp)
        out.append(basis[underlying(sp, lab)])
    return out


def dense_shape(layout):
    return tuple(leg_basis(sp)[1] for sp in layout.cod + layout.dom)


def subblock_array(layout, flat, sb):
    """Reduced array of one subblock as an ndarray over (legs...) from the flat buffer."""
    strides = subblock_index(layout, sb)
    item = flat.itemsize
    return np.lib.stride_tricks.as_strided(flat[sb.offset:], shape=sb.extents,
                                           strides=tuple(s * item for s in strides))


def to_dense(layout, flat):
    kind = layout.kind
    flat = np.asarray(flat)
    D = np.zeros(dense_shape(layout), dtype=flat.dtype)
    nl = len(layout.cod) + len(layout.dom)
    for sb in layout.subblocks:
        R = subblock_array(layout, flat, sb)
        sl = _dense_slices(layout, sb)
        if sectors.is_abelian(kind):
            idx = tuple(slice(o, o + n) for o, n, _ in sl)
            D[idx] = R
        else:
            B = basis_tensor(kind, layout.cod, layout.dom, sb.key)
            T = np.multiply.outer(R, B)  # (n_1..n_N, d_1..d_N)
            perm = [x for k in range(nl) for x in (k, nl + k)]
            T = T.transpose(perm).reshape([n * d for _, n, d in sl])
            idx = tuple(slice(o, o + n * d) for o, n, d in sl)
            D[idx] += T
    return D


def from_dense(layout, D):
    """Project a dense array onto the canonical basis: R = <B, D_sub> / d_c (abelian: extraction)."""
    kind = layout.kind
    flat = np.zeros(layout.nelems, dtype=D.dtype)
    nl = len(layout.cod) + len(layout.dom)
    for sb in layout.subblocks:
        sl = _dense_slices(layout, sb)
        dst = subblock_array(layout, flat, sb)
        if sectors.is_abelian(kind):
            idx = tuple(slice(o, o + n) for o, n, _ in sl)
            dst[...] = D[idx]
        else:
            idx = tuple(slice(o, o + n * d) for o, n, d in sl)
            sub = D[idx].reshape([x for _, n, d in sl for x in (n, d)])
            B = basis_tensor(kind, layout.cod, layout.dom, sb.key)
            # contract the inner (d) axes with B
            sub = np.tensordot(sub, B, axes=([2 * k + 1 for k in range(nl)], list(range(nl))))
            dc = sectors.qdim(kind, sb.key[2])
            dst[...] = sub / dc
    return flat


def parity_vector(sp):
    """Fermion parity of every dense index of a leg (0 for bosonic kinds)."""
    basis, dim = leg_basis(sp)
    p = np.zeros(dim, dtype=np.int64)
    for lab, (o, n, d) in basis.items():
        p[o:o + n * d] = sectors.parity(sp["kind"], lab)
    return p


def sector_of_index(sp):
    """Underlying sector label of every dense index of a leg (for symmetry-invariance checks)."""
    basis, dim = leg_basis(sp)
    out = [None] * dim
    for lab, (o, n, d) in basis.items():
        for i in range(o, o + n * d):
            out[i] = lab
    return out


def random_flat(layout, rng, dtype=np.float64):
    x = rng.standard_normal(layout.nelems)
    if dtype == np.complex128:
        x = x + 1j * rng.standard_normal(layout.nelems)
    return x


def norm_dense(D):
    return math.sqrt(float(np.vdot(D, D).real))
