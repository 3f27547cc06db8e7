"""The paper's worked examples, reproduced by the oracle (golden fixtures in tests/golden/).

Each fixture cites the PAPER.md lines it transcribes. The oracle computes the
transfer matrices from its dense Clebsch-Gordan embedding (a method the paper
names at P:1534-1542), i.e. independently of any fusion-tree manipulation.
"""
import math
import os

import numpy as np

from oracle import layout as L, dense as Dn, contract as C

GOLD = os.path.join(os.path.dirname(__file__), "golden")
V_SU2 = {"kind": "SU2", "sectors": [((0,), 1), ((1,), 1)], "dual": False}
V_Z2 = {"kind": "Z2", "sectors": [((0,), 1), ((1,), 1)], "dual": False}


def load_matrix(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([0.0 if tok == "." else float(eval(tok, {"sqrt": math.sqrt})) for tok in line.split()])
    return np.array(rows)


def su2_transfer(op_dense, cod_out, dom_out):
    lt = L.homspace_layout("SU2", [V_SU2, V_SU2], [V_SU2, V_SU2])
    ls = L.homspace_layout("SU2", cod_out, dom_out)
    M = np.zeros((lt.nelems, ls.nelems))
    for i in range(lt.nelems):
        x = np.zeros(lt.nelems)
        x[i] = 1.0
        M[i] = Dn.from_dense(ls, op_dense(Dn.to_dense(lt, x)))
    return M


def test_su2_bookkeeping_P1750():
    # five splitting trees, 9 reduced elements (vs 81), blocks 2x2, 2x2, 1x1
    lt = L.homspace_layout("SU2", [V_SU2, V_SU2], [V_SU2, V_SU2])
    trees = L.enumerate_trees("SU2", [V_SU2, V_SU2])
    assert sum(len(v) for v in trees.values()) == 5
    assert lt.nelems == 9 and len(lt.subblocks) == 9
    assert [(b[1], b[2]) for b in lt.blocks] == [(2, 2), (2, 2), (1, 1)]
    assert int(np.prod(Dn.dense_shape(lt))) == 81


def test_su2_transpose_P1805():
    p, q = (1, 3), (0, 2)  # reading C11: ((2,4),(1,3)) 1-based
    cod, dom = C.permuted_spaces([V_SU2, V_SU2], [V_SU2, V_SU2], p, q)
    assert [s["dual"] for s in cod] == [False, True] and [s["dual"] for s in dom] == [True, False]
    M = su2_transfer(lambda D: np.transpose(D, p + q), cod, dom)
    assert np.abs(M - load_matrix("su2_transpose_P1805.txt")).max() < 1e-15


def test_su2_permute_P1850():
    p, q = (1, 0), (3, 2)
    cod, dom = C.permuted_spaces([V_SU2, V_SU2], [V_SU2, V_SU2], p, q)
    M = su2_transfer(lambda D: np.transpose(D, p + q), cod, dom)
    assert np.abs(M - load_matrix("su2_permute_P1850.txt")).max() < 1e-15


def test_su2_partial_trace_P1892():
    # codomain leg 2 traced with domain leg 2 (reading C11)
    M = su2_transfer(lambda D: np.einsum("akbk->ab", D), [V_SU2], [V_SU2])
    assert np.abs(M - load_matrix("su2_trace_P1892.txt")).max() < 1e-15
    # tracing leg 1 with leg 1 instead does NOT reproduce the printed matrix
    M1 = su2_transfer(lambda D: np.einsum("kakb->ab", D), [V_SU2], [V_SU2])
    assert np.abs(M1 - load_matrix("su2_trace_P1892.txt")).max() > 0.1


def _channels(name):
    out = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#")[0].strip()
        if line:
            out.append(line)
    return out


def test_z2_grouping_P1043():
    lt = L.homspace_layout("Z2", [V_Z2, V_Z2], [V_Z2, V_Z2])
    got = {}
    for sb in lt.subblocks:
        cod, dom = sb.key[0], sb.key[3]
        got[(cod[0][0], cod[1][0], dom[0][0], dom[1][0])] = lt.blocks[sb.block][0][0]
    want = {}
    for line in _channels("z2_grouping_P1043.txt"):
        c, rest = line.split(None, 1)
        left, right = rest.split(";")
        a = tuple(int(x) for x in left.split())
        b = tuple(int(x) for x in right.split())
        want[a + b] = int(c)
    assert got == want
    assert [(b[1], b[2]) for b in lt.blocks] == [(2, 2), (2, 2)]


def test_z2_bend_P1112():
    # bend the second domain leg to the codomain: (a1 a2 ; b1 b2) -> (a1 a2 b2* ; b1)
    lt = L.homspace_layout("Z2", [V_Z2, V_Z2], [V_Z2, V_Z2])
    p, q = (0, 1, 3), (2,)
    cod, dom = C.permuted_spaces([V_Z2, V_Z2], [V_Z2, V_Z2], p, q)
    ls = L.homspace_layout("Z2", cod, dom)
    for line in _channels("z2_bend_P1112.txt"):
        src, dst = line.split("->")
        s_c, s_d = src.split(";")
        src_key = tuple(int(x) for x in s_c.split()) + tuple(int(x) for x in s_d.split())
        d_c, rest = dst.split(";")
        d_dom, blk = rest.split("block")
        dst_key = tuple(int(x) for x in d_c.split()) + tuple(int(x) for x in d_dom.split())
        x = np.zeros(lt.nelems)
        for sb in lt.subblocks:
            if tuple(l[0] for l in sb.key[0] + sb.key[3]) == src_key:
                x[sb.offset] = 7.0
        y = Dn.from_dense(ls, np.transpose(Dn.to_dense(lt, x), p + q))
        hit = [sb for sb in ls.subblocks if y[sb.offset] != 0.0]
        assert len(hit) == 1 and y[hit[0].offset] == 7.0
        assert tuple(l[0] for l in hit[0].key[0] + hit[0].key[3]) == dst_key
        assert ls.blocks[hit[0].block][0][0] == int(blk)
