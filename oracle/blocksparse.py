"""Tier 2 oracle: charge-tuple einsum for abelian tensors at full size (test infrastructure).

SURVEY §8(c) step 7. A tensor is a dict keyed by the tuple of tree labels of
all its legs (abelian: the tree pair is fixed by its uncoupled labels) whose
values are ndarrays over (legs...). A contraction sums, for every pair of
A/B keys whose contracted legs refer to the same underlying sector, an
np.einsum of the two arrays over the contracted legs (the dense
array restricted to one allowed charge tuple). No matricisation, no fusion
trees, no planner layout. For fermionic kinds each term carries the product
of the three Alg. 4 permute signs of reading C13, evaluated on the tuple's
parities (the sign is constant over a charge tuple).

Cross-checked against the dense tier 1 (contract.py) at reduced sizes.
"""
import math

import numpy as np

from workloads import gen

from . import sectors
from .contract import tuples_from_labels, output_spaces, koszul_sign_pairs, _LETTERS
from .dense import subblock_array
from .layout import underlying


def to_blocks(layout, flat):
    flat = np.ascontiguousarray(flat)
    out = {}
    for sb in layout.subblocks:
        out[tuple(sb.key[0]) + tuple(sb.key[3])] = np.array(subblock_array(layout, flat, sb))
    return out


def _tree_label(sp, u):
    return sectors.dual(sp["kind"], u) if sp["dual"] else tuple(u)


def _sign(kind, labels, n1, p, q):
    pairs = koszul_sign_pairs(n1, len(labels) - n1, p, q)
    s = 0
    for x, y in pairs:
        s += sectors.parity(kind, labels[x]) * sectors.parity(kind, labels[y])
    return -1.0 if s % 2 else 1.0


def contract_blocks(kind, Ab, A_cod, A_dom, labA, Bb, B_cod, B_dom, labB, labC, n_cod_C, out_keys=None, stats=None):
    """Charge-tuple contraction. Returns dict C key -> ndarray (legs in labC order).

    `stats` (optional dict) accumulates 'flops' = sum over terms of 2 |a| |b| / |contracted|.
    """
    labA, labB, labC = list(labA), list(labB), list(labC)
    A_sp, B_sp = list(A_cod) + list(A_dom), list(B_cod) + list(B_dom)
    C_cod, C_dom = output_spaces(A_cod, A_dom, B_cod, B_dom, labA, labB, labC, n_cod_C)
    C_sp = C_cod + C_dom
    pA, qA, pB, qB, pAB, qAB = tuples_from_labels(labA, labB, labC, n_cod_C)
    ferm = sectors.is_fermionic(kind)
    con = [labA[i] for i in qA]
    openA = [labA[i] for i in pA]
    openB = [labB[j] for j in qB]

    m = {}
    for l in labA + labB:
        m.setdefault(l, _LETTERS[len(m)])
    spec = "".join(m[l] for l in labA) + "," + "".join(m[l] for l in labB) + "->" + "".join(m[l] for l in labC)

    def und(sp_list, lab_list, key, l):
        k = lab_list.index(l)
        return underlying(sp_list[k], key[k])

    A_idx = {}
    for ka in Ab:
        ao = tuple(und(A_sp, labA, ka, l) for l in openA)
        ac = tuple(und(A_sp, labA, ka, l) for l in con)
        A_idx.setdefault(ao, []).append((ka, ac))
    B_idx = {}
    for kb in Bb:
        bo = tuple(und(B_sp, labB, kb, l) for l in openB)
        bc = tuple(und(B_sp, labB, kb, l) for l in con)
        B_idx.setdefault(bo, {})[bc] = kb

    def ckey(u_by_label):
        return tuple(_tree_label(C_sp[i], u_by_label[l]) for i, l in enumerate(labC))

    out = {}
    if out_keys is None:
        pairs_iter = ((ao, bo) for ao in A_idx for bo in B_idx)
    else:
        pairs_iter = []
        for kc in out_keys:
            u = {l: underlying(C_sp[i], kc[i]) for i, l in enumerate(labC)}
            pairs_iter.append((tuple(u[l] for l in openA), tuple(u[l] for l in openB)))
    for ao, bo in pairs_iter:
        if ao not in A_idx or bo not in B_idx:
            continue
        bmap = B_idx[bo]
        for ka, ac in A_idx[ao]:
            kb = bmap.get(ac)
            if kb is None:
                continue
            u = dict(zip(openA, ao))
            u.update(zip(openB, bo))
            kc = ckey(u)
            xa, xb = Ab[ka], Bb[kb]
            term = np.einsum(spec, xa, xb, optimize=True)
            if stats is not None:
                ncon = 1
                for l in con:
                    ncon *= xa.shape[labA.index(l)]
                stats["flops"] = stats.get("flops", 0.0) + 2.0 * xa.size * xb.size / max(ncon, 1)
            if ferm:
                ct_labels = [ka[i] for i in pA] + [kb[j] for j in qB]
                s = (_sign(kind, list(ka), len(A_cod), pA, qA) * _sign(kind, list(kb), len(B_cod), pB, qB)
                     * _sign(kind, ct_labels, len(pA), pAB, qAB))
                term = s * term
            if kc in out:
                out[kc] += term
            else:
                out[kc] = term
    return out, (C_cod, C_dom)


class LazyBlocks(dict):
    """Charge-tuple blocks of an input tensor, generated on first access (keyed values are
    independent of placement, so block[key] = values reshaped column-major over the legs)."""

    def __init__(self, layout, cfg, tidx, complex_=False):
        super().__init__()
        self._sub = {tuple(sb.key[0]) + tuple(sb.key[3]): sb for sb in layout.subblocks}
        self._cfg, self._tidx, self._complex = cfg, tidx, complex_

    def __iter__(self):
        return iter(self._sub)

    def __contains__(self, k):
        return k in self._sub

    def __len__(self):
        return len(self._sub)

    def __getitem__(self, k):
        if not dict.__contains__(self, k):
            sb = self._sub[k]
            v = gen.subblock_values(self._cfg, self._tidx, sb.key, math.prod(sb.extents), self._complex)
            dict.__setitem__(self, k, v.reshape(sb.extents, order="F"))
        return dict.__getitem__(self, k)

    def keys(self):
        return self._sub.keys()
