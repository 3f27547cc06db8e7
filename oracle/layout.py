"""Canonical block layout, re-derived on the oracle side from the text of readings C4/C5.

(Test infrastructure; shares no code with the library's planner.)

A HomSpace is (kind, cod spaces, dom spaces). For each side we enumerate the
canonical left-to-right fusion trees: uncoupled labels a_1..a_N
(a dual leg carries the label of its dual sector, "use the sector as if it were
a normal space", reading C6), inner labels e_2..e_{N-1} with
e_k in e_{k-1} (x) a_k, coupled label c = e_N.

Reading C4 (orders): sectors ascending by label; blocks by coupled label
ascending; trees within a block by (uncoupled tuple, first leg most
significant), then inner labels. The trivial-grouping offsets follow
Eq. abeliangrouping / the embedding G^{c;s_I}.

Reading C5 (storage): block c is a column-major rows(c) x cols(c) matrix; blocks
are concatenated in block order; the reduced array of tree pair (s, f) is the
strided region starting at (row_off(s), col_off(f)) with column-major element
order over (codomain legs..., domain legs...) (Eq. linearindex).
Subblocks are enumerated block by block, fusion tree (column) major, splitting
tree (row) minor.
"""
from dataclasses import dataclass
import itertools
import math

from . import sectors


def tree_sectors(sp):
    """[(tree label, degeneracy)] of one leg, ascending by tree label (reading C6)."""
    kind = sp["kind"]
    out = [((sectors.dual(kind, lab) if sp["dual"] else tuple(lab)), deg) for lab, deg in sp["sectors"]]
    return sorted(out)


def underlying(sp, tree_label):
    """Sector of the underlying non-dual space V that a tree label on this leg refers to."""
    return sectors.dual(sp["kind"], tree_label) if sp["dual"] else tuple(tree_label)


@dataclass(frozen=True)
class Tree:
    uncoupled: tuple
    inner: tuple
    coupled: tuple
    dims: tuple  # degeneracies of the uncoupled legs


def _inner_sequences(kind, uncoupled):
    """All admissible (inner labels, coupled) for a left-to-right tree, in lexicographic order."""
    n = len(uncoupled)
    if n == 0:
        return [((), sectors.unit(kind))]
    if n == 1:
        return [((), uncoupled[0])]
    seqs = []

    def rec(e, k, inner):
        if k == n:
            seqs.append((tuple(inner[:-1]), e))
            return
        for e2 in sectors.fuse(kind, e, uncoupled[k]):
            rec(e2, k + 1, inner + [e2])

    rec(uncoupled[0], 1, [])
    return sorted(seqs)


def enumerate_trees(kind, spaces):
    """dict coupled -> [Tree] in canonical order (reading C4)."""
    per_leg = [tree_sectors(sp) for sp in spaces]
    groups = {}
    for combo in itertools.product(*per_leg):  # first leg most significant
        unc = tuple(l for l, _ in combo)
        dims = tuple(d for _, d in combo)
        for inner, c in _inner_sequences(kind, unc):
            groups.setdefault(c, []).append(Tree(unc, inner, c, dims))
    return groups


@dataclass(frozen=True)
class Subblock:
    key: tuple          # (cod uncoupled, cod inner, coupled, dom uncoupled, dom inner)
    block: int
    row_off: int
    col_off: int
    extents: tuple      # cod degeneracies..., dom degeneracies...
    offset: int         # flat offset of element (0,...,0)
    ld: int             # rows of the block


@dataclass
class Layout:
    kind: str
    cod: list
    dom: list
    blocks: list        # [(coupled, rows, cols, offset)]
    subblocks: list     # [Subblock]
    nelems: int


def homspace_layout(kind, cod, dom):
    ct = enumerate_trees(kind, cod)
    dt = enumerate_trees(kind, dom)
    blocks, subs = [], []
    off = 0
    for bi, c in enumerate(sorted(set(ct) & set(dt))):
        rows = sum(math.prod(t.dims) for t in ct[c])
        cols = sum(math.prod(t.dims) for t in dt[c])
        blocks.append((c, rows, cols, off))
        col_off = 0
        for f in dt[c]:
            row_off = 0
            for s in ct[c]:
                subs.append(Subblock((s.uncoupled, s.inner, c, f.uncoupled, f.inner), bi, row_off, col_off,
                                     s.dims + f.dims, off + row_off + rows * col_off, rows))
                row_off += math.prod(s.dims)
            col_off += math.prod(f.dims)
        off += rows * cols
    return Layout(kind, list(cod), list(dom), blocks, subs, off)


def subblock_index(layout, sb):
    """Flat indices (numpy-free helper) are built by dense.py; this returns the strides.

    Element (i_1..i_N1; j_1..j_N2) of subblock sb sits at
      sb.offset + i_1 + n_1 i_2 + ... + ld * (j_1 + m_1 j_2 + ...)
    """
    n1 = len(layout.cod)
    ext = sb.extents
    strides = []
    s = 1
    for k in range(n1):
        strides.append(s)
        s *= ext[k]
    s = sb.ld
    for k in range(n1, len(ext)):
        strides.append(s)
        s *= ext[k]
    return strides
