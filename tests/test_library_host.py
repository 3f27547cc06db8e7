"""CPU tests of the C-ABI library's host side (no GPU needed).

  * the library loads and exports every symbol include/tk.h declares
  * block layouts and sector bookkeeping equal the oracle's, integer for integer (reading C25)
  * the planner's F / R tables equal the oracle's exact 6j / CG values
  * permute transfer matrices (fusion-tree moves in C++) equal the oracle's dense
    Clebsch-Gordan projections -- including the paper's §4.3 matrices -- and, for
    fermions, the dense Koszul permute
  * error statuses for malformed input
"""
import itertools
import os
import re

import numpy as np
import pytest

from paper_2508_10076_b200 import tk
from oracle import layout as OL, dense as OD, contract as OC, su2 as OS
from workloads import configs as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "tk.h")).read()
    names = sorted(set(re.findall(r"\b(tk_[a-z_0-9]+)\s*\(", hdr)))
    assert len(names) >= 25
    for n in names:
        assert hasattr(tk._lib, n), n
    assert set(names) == set(tk.EXPORTED)


def oracle_layout(spec):
    kind = spec["cod"][0]["kind"] if spec["cod"] else spec["dom"][0]["kind"]
    return OL.homspace_layout(kind, spec["cod"], spec["dom"])


def assert_same_layout(spec):
    t = tk.tensor_from_spec(spec)
    lo = oracle_layout(spec)
    assert t.nelems == lo.nelems
    cp, rows, cols, off = t.blocks()
    assert [tuple(x) for x in cp] == [tuple(b[0]) for b in lo.blocks]
    assert list(rows) == [b[1] for b in lo.blocks] and list(cols) == [b[2] for b in lo.blocks]
    assert list(off) == [b[3] for b in lo.blocks]
    from paper_2508_10076_b200 import layout_io
    keys = layout_io.decode_keys(t)
    sb = t.subblocks()
    assert len(keys) == len(lo.subblocks)
    n = len(spec["cod"]) + len(spec["dom"])
    for i, s in enumerate(lo.subblocks):
        assert keys[i] == s.key
        assert sb["block"][i] == s.block and sb["row_off"][i] == s.row_off and sb["col_off"][i] == s.col_off
        assert tuple(sb["extents"][i][:n]) == s.extents and sb["offset"][i] == s.offset


@pytest.mark.parametrize("cfgfun", [W.cfg1, lambda: W.cfg2(), lambda: W.cfg3(chi=256), lambda: W.cfg4(d_leg=64),
                                    lambda: W.cfg5(), lambda: W.cfg6(), lambda: W.cfg7(n_mult=200),
                                    lambda: W.cfg8(n_mult=60)])
def test_layout_equals_oracle(cfgfun):
    cfg = cfgfun()
    for name, (spec, _) in cfg["tensors"].items():
        assert_same_layout(spec)


def test_layout_duals_and_empty_codomain():
    V = W.space("U1", [((-1,), 2), ((0,), 1), ((2,), 3)])
    S = W.space("SU2", [((0,), 2), ((1,), 1), ((2,), 2)])
    for spec in ({"cod": [V, W.dual(V)], "dom": [V]}, {"cod": [], "dom": [V, W.dual(V)]},
                 {"cod": [W.dual(V), V, V], "dom": []}, {"cod": [S, W.dual(S), S], "dom": [S]},
                 {"cod": [], "dom": [S, S]}):
        assert_same_layout(spec)


def test_topological_data_equals_oracle():
    for j1, j2, j3, j4 in itertools.product(range(5), repeat=4):
        for e in range(9):
            for f in range(9):
                ref = OS.fsymbol(j1, j2, j3, j4, e, f)
                got = tk.tk_fsymbol("SU2", [j1], [j2], [j3], [j4], [e], [f])
                assert abs(got - ref) < 1e-14
    for a, b in itertools.product(range(7), repeat=2):
        for c in range(14):
            assert tk.tk_rsymbol("SU2", [a], [b], [c]) == OS.rsymbol(a, b, c)
    assert tk.tk_rsymbol("fU1xU1", [1, 1], [-1, 1], [0, 2]) == -1.0
    assert tk.tk_rsymbol("fU1xU1", [2, 0], [1, 1], [3, 1]) == 1.0


# ------------------------------------------------------------ permute transfer
def oracle_transfer(kind, cod, dom, p, q):
    lt = OL.homspace_layout(kind, cod, dom)
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    ls = OL.homspace_layout(kind, c2, d2)
    par = [OD.parity_vector(s) for s in cod + dom]
    M = np.zeros((len(lt.subblocks), len(ls.subblocks)))
    for i, sb in enumerate(lt.subblocks):
        x = np.zeros(lt.nelems)
        x[sb.offset] = 1.0  # first element of the subblock: tree-pair coefficient (all-degeneracy-1 spaces)
        y = OD.from_dense(ls, OC.permute_dense(OD.to_dense(lt, x), par, len(cod), p, q))
        for j, sc in enumerate(ls.subblocks):
            M[i, j] = y[sc.offset]
    return M, c2, d2


def lib_transfer(kind, cod, dom, p, q):
    A = tk.tensor_from_spec({"cod": cod, "dom": dom})
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    C = tk.tensor_from_spec({"cod": c2, "dom": d2})
    return tk.tk_permute_transfer(A, p, q, C)


def test_transfer_golden_P1805_P1850():
    from tests.test_oracle_golden import load_matrix
    V = W.space("SU2", [((0,), 1), ((1,), 1)])
    M = lib_transfer("SU2", [V, V], [V, V], [1, 3], [0, 2])
    assert np.abs(M - load_matrix("su2_transpose_P1805.txt")).max() < 1e-14
    M = lib_transfer("SU2", [V, V], [V, V], [1, 0], [3, 2])
    assert np.abs(M - load_matrix("su2_permute_P1850.txt")).max() < 1e-14


def _random_perms(N, rng, n):
    out = []
    for _ in range(n):
        perm = list(rng.permutation(N))
        k = int(rng.integers(0, N + 1))
        out.append((perm[:k], perm[k:]))
    return out


@pytest.mark.parametrize("kind,secs", [
    ("SU2", [((0,), 1), ((1,), 1), ((2,), 1)]),
    ("SU2", [((1,), 1), ((2,), 1), ((3,), 1)]),
    ("fU1xU1", [((0, 0), 1), ((1, 1), 1), ((1, -1), 1), ((2, 0), 1)]),
    ("fZ2", [((0,), 1), ((1,), 1)]),
    ("U1", [((-1,), 1), ((0,), 1), ((1,), 1)]),
    ("fU1xSU2", [((0, 0), 1), ((1, 1), 1), ((-1, 1), 1), ((2, 0), 1)]),
    ("fU1xSU2", [((0, 2), 1), ((1, 1), 1), ((-1, 3), 1)]),
    ("fSU2xSU2", [((0, 0), 1), ((1, 1), 1), ((0, 2), 1)]),
    ("fSU2xSU2", [((0, 1), 1), ((1, 0), 1), ((2, 2), 1)]),
])
def test_transfer_random_vs_oracle(kind, secs):
    rng = np.random.default_rng(42)
    V = W.space(kind, secs)
    Vd = W.dual(V)
    shapes = [([V, Vd], [V]), ([V], [V, V]), ([V, V], [Vd, V]), ([Vd, V, V], [V]), ([V, V, Vd, V], [])]
    for cod, dom in shapes:
        N = len(cod) + len(dom)
        for p, q in _random_perms(N, rng, 6):
            ref, _, _ = oracle_transfer(kind, cod, dom, p, q)
            got = lib_transfer(kind, cod, dom, p, q)
            assert np.abs(got - ref).max() < 1e-13, (cod, dom, p, q)


# ------------------------------------------------------------------ errors
def test_error_statuses():
    V = tk.tk_space_parse("U1[-1:2, 0:1, 1:2]")
    assert V.info()[:3] == (3, 5, False)
    with pytest.raises(tk.TKError) as e:
        tk.tk_space_create("Z3", [[0]], [1])
    assert e.value.status == "TK_ERR_UNKNOWN_LABEL"
    with pytest.raises(tk.TKError) as e:
        tk.tk_space_create("Z2", [[0], [0]], [1, 2])
    assert e.value.status == "TK_ERR_INVALID_ARGUMENT"
    A = tk.tk_tensor_create(tk.TK_F64, [V, V], [V])
    B = tk.tk_tensor_create(tk.TK_F64, [V], [V])
    with pytest.raises(tk.TKError) as e:   # contracted legs both kets
        tk.tk_contract_output(A, [1, 2, 3], B, [2, 4], [1, 3, 4], 2)
    assert e.value.status == "TK_ERR_SPACE_MISMATCH"
    with pytest.raises(tk.TKError) as e:   # labC repeats an open label
        tk.tk_contract_output(A, [1, 2, 3], B, [3, 4], [1, 1, 4], 1)
    assert e.value.status == "TK_ERR_MALFORMED_NETWORK"
    with pytest.raises(tk.TKError) as e:   # labC names a contracted label
        tk.tk_contract_output(A, [1, 2, 3], B, [3, 4], [1, 2, 3], 1)
    assert e.value.status == "TK_ERR_UNKNOWN_LABEL"
    with pytest.raises(tk.TKError) as e:
        tk.tk_permute_transfer(A, [0, 0], [1], A)
    assert e.value.status == "TK_ERR_INVALID_PERMUTATION"
    with pytest.raises(tk.TKError) as e:   # wrong output spaces
        tk.tk_permute_transfer(A, [1, 0], [2], B)
    assert e.value.status == "TK_ERR_SPACE_MISMATCH"
    S = tk.tk_space_parse("SU2[0:1, 1/2:2]'")
    n, dim, dual, w = S.info()
    assert (n, dim, dual) == (2, 5, True)
    with pytest.raises(tk.TKError) as e:
        tk.tk_tensor_create(tk.TK_F64, [V], [S])
    assert e.value.status == "TK_ERR_SECTOR_MISMATCH"


@pytest.mark.parametrize("cfgfun", [W.cfg1, lambda: W.cfg2(chi=64), lambda: W.cfg3(chi=64), lambda: W.cfg4(d_leg=32),
                                    lambda: W.cfg5(mults=(2, 2, 1, 1, 1, 1, 1)),
                                    lambda: W.cfg6(mults=(2, 2, 1, 1, 1, 1, 1)), lambda: W.cfg7(n_mult=60),
                                    lambda: W.cfg8(n_mult=20)])
def test_contract_output_spaces(cfgfun):
    cfg = cfgfun()
    specs = {k: v[0] for k, v in cfg["tensors"].items()}
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        A, B = tk.tensor_from_spec(specs[na]), tk.tensor_from_spec(specs[nb])
        C = tk.tk_contract_output(A, la, B, lb, lc, ncod)
        cod, dom = OC.output_spaces(specs[na]["cod"], specs[na]["dom"], specs[nb]["cod"], specs[nb]["dom"],
                                    la, lb, lc, ncod)
        specs[nc] = {"cod": cod, "dom": dom}
        assert_same_layout(specs[nc])
        assert C.nelems == OL.homspace_layout(cfg["kind"], cod, dom).nelems


# ------------------------------------------------- planar route and anyons
def _cyclic(n1, N, r, n1p):
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    T = [S[(i + r) % N] for i in range(N)]
    return T[:n1p], list(reversed(T[n1p:]))


def test_planar_route_su2():
    """The library's planar route (rotations + bends, forced through the test hook) equals the dense
    SU(2) oracle for every cyclic transpose with dual legs; kappa = chi_{a1} is the only one that does."""
    for secs in ([((0,), 1), ((1,), 1), ((2,), 1)], [((1,), 1), ((2,), 1)]):
        V = W.space("SU2", secs)
        Vd = W.dual(V)
        for cod, dom in (([V, Vd], [V]), ([V, V], [Vd, V]), ([Vd, V, V], [V])):
            n1, N = len(cod), len(cod) + len(dom)
            for r in range(N):
                for n1p in range(N + 1):
                    p, q = _cyclic(n1, N, r, n1p)
                    ref, c2, d2 = oracle_transfer("SU2", cod, dom, p, q)
                    A, C = tk.tensor_from_spec({"cod": cod, "dom": dom}), tk.tensor_from_spec({"cod": c2, "dom": d2})
                    assert np.abs(tk.tk_permute_transfer_planar(A, p, q, C) - ref).max() < 1e-13
    # kappa = 1 fails for half-integer spins (chi = -1)
    V = W.space("SU2", [((1,), 1), ((2,), 1)])
    p, q = _cyclic(2, 3, 1, 2)
    ref, c2, d2 = oracle_transfer("SU2", [V, V], [V], p, q)
    A, C = tk.tensor_from_spec({"cod": [V, V], "dom": [V]}), tk.tensor_from_spec({"cod": c2, "dom": d2})
    assert np.abs(tk.tk_permute_transfer_planar(A, p, q, C, 0) - ref).max() > 0.5
    tk.tk_permute_transfer_planar(A, p, q, C, 1)  # restore the library convention


@pytest.mark.parametrize("kind,secs", [("Fib", [((0,), 1), ((1,), 1)]), ("Ising", [((0,), 1), ((1,), 1), ((2,), 1)])])
def test_anyon_transfer_equals_planar_oracle(kind, secs):
    from oracle import planar as OP
    V = W.space(kind, secs)
    Vd = W.dual(V)
    for cod, dom in (([V, Vd], [V]), ([V, V], [Vd, V]), ([V], [V, V]), ([V, V], [V, V])):
        n1, N = len(cod), len(cod) + len(dom)
        for r in range(N):
            for n1p in range(N + 1):
                p, q = _cyclic(n1, N, r, n1p)
                M, lt, ls = OP.planar_transfer(kind, cod, dom, p, q)
                A, C = tk.tensor_from_spec({"cod": cod, "dom": dom}), tk.tensor_from_spec({"cod": ls.cod, "dom": ls.dom})
                assert np.abs(tk.tk_permute_transfer(A, p, q, C) - M).max() < 1e-13, (cod, dom, p, q)
    # braiding is unavailable: a non-planar permutation is refused
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V]})
    C = tk.tensor_from_spec({"cod": [V, V], "dom": [V]})
    with pytest.raises(tk.TKError) as e:
        tk.tk_permute_transfer(A, [1, 0], [2], C)
    assert e.value.status == "TK_ERR_BRAIDING_UNAVAILABLE"
    with pytest.raises(tk.TKError) as e:
        tk.tk_rsymbol(kind, [1], [1], [0])
    assert e.value.status == "TK_ERR_BRAIDING_UNAVAILABLE"


def test_anyon_fsymbols_equal_oracle():
    from oracle import planar as OP
    for kind, L in (("Fib", [0, 1]), ("Ising", [0, 1, 2])):
        for a, b, c, d, e, f in itertools.product(L, repeat=6):
            ref = OP.fsymbol(kind, (a,), (b,), (c,), (d,), (e,), (f,))
            assert abs(tk.tk_fsymbol(kind, [a], [b], [c], [d], [e], [f]) - ref) < 1e-15


# --------------------------------------------------------------- partial trace (NEXT-4)
def test_trace_golden_P1892():
    """§4.3's printed partial-trace matrix (reading C11: codomain leg 2 with domain leg 2)."""
    from tests.test_oracle_golden import load_matrix
    V = W.space("SU2", [((0,), 1), ((1,), 1)])
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V, V]})
    C = tk.tk_trace_output(A, [1], [3], [0], [2])
    M = tk.tk_trace_transfer(A, [1], [3], [0], [2], C)
    assert np.abs(M - load_matrix("su2_trace_P1892.txt")).max() < 1e-14


def _dense_trace_transfer(kind, cod, dom, pt, qt, p, q):
    lt = OL.homspace_layout(kind, cod, dom)
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    lc = OL.homspace_layout(kind, c2, d2)
    M = np.zeros((len(lt.subblocks), len(lc.subblocks)))
    for i, sb in enumerate(lt.subblocks):
        x = np.zeros(lt.nelems)
        x[sb.offset] = 1.0
        R, _, _ = OC.partial_trace_dense(OD.to_dense(lt, x), cod, dom, pt, qt, p, q)
        y = OD.from_dense(lc, R)
        for j, sc in enumerate(lc.subblocks):
            M[i, j] = y[sc.offset]
    return M, c2, d2


@pytest.mark.parametrize("kind,secs", [("U1", [((-1,), 1), ((0,), 1), ((1,), 1)]),
                                       ("SU2", [((0,), 1), ((1,), 1), ((2,), 1)]),
                                       ("SU2", [((1,), 1), ((2,), 1)])])
def test_trace_transfer_vs_dense(kind, secs):
    V = W.space(kind, secs)
    Vd = W.dual(V)
    cases = [([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [0], [2], [3], [1]),
             ([V, V], [V, V], [0], [3], [1], [2]), ([V, Vd, V], [V, V], [2], [4], [1, 0], [3]),
             ([V, V], [V, V], [0, 1], [2, 3], [], []), ([Vd, V], [Vd, V], [0], [2], [1], [3]),
             ([V, Vd, V], [V], [0], [1], [2], [3])]   # a codomain V with a codomain V*: ket/bra
    for cod, dom, pt, qt, p, q in cases:
        ref, c2, d2 = _dense_trace_transfer(kind, cod, dom, pt, qt, p, q)
        A = tk.tensor_from_spec({"cod": cod, "dom": dom})
        C = tk.tk_trace_output(A, pt, qt, p, q)   # rank 0 for full traces
        assert np.abs(tk.tk_trace_transfer(A, pt, qt, p, q, C) - ref).max() < 1e-13, (pt, qt, p, q)


def test_trace_errors():
    V = W.space("U1", [((-1,), 1), ((1,), 2)])
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V, V]})
    with pytest.raises(tk.TKError) as e:   # two kets of V
        tk.tk_trace_output(A, [0], [1], [2], [3])
    assert e.value.status == "TK_ERR_SPACE_MISMATCH"
    F = W.space("fU1xU1", [((0, 0), 1), ((1, 1), 1)])
    B = tk.tensor_from_spec({"cod": [F, F], "dom": [F, F]})
    with pytest.raises(tk.TKError) as e:
        tk.tk_trace_output(B, [1], [3], [0], [2])
    assert e.value.status == "TK_ERR_UNSUPPORTED"


@pytest.mark.parametrize("kind,secs", [("Fib", [((0,), 1), ((1,), 1)]), ("Ising", [((0,), 1), ((1,), 1), ((2,), 1)])])
def test_anyon_trace_vs_planar_oracle(kind, secs):
    from oracle import planar as OP
    V = W.space(kind, secs)
    for cod, dom, pt, qt, p, q in (([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [2], [0], [1, 3], []),
                                   ([V, V], [V, V], [0, 1], [2, 3], [], [])):
        lt = OL.homspace_layout(kind, cod, dom)
        A = tk.tensor_from_spec({"cod": cod, "dom": dom})
        C = tk.tk_trace_output(A, pt, qt, p, q)
        got = tk.tk_trace_transfer(A, pt, qt, p, q, C)
        for i, sb in enumerate(lt.subblocks):
            x = np.zeros(lt.nelems)
            x[sb.offset] = 1.0
            y, lc = OP.trace_planar(kind, cod, dom, x, pt, qt, p, q)
            ref = np.array([y[sc.offset] for sc in lc.subblocks])
            assert np.abs(got[i] - ref).max() < 1e-13


def test_contract_tuples_output_and_errors():
    """tk_contract_tuples_output (Alg. 4 with explicit tuples): C~ = (pA legs ; qB legs) permuted
    by (pAB, qAB) -- the same HomSpace the oracle's selection rule gives; the reading-C2 tuples reproduce
    tk_contract_output; malformed tuples fail before any work."""
    V = W.space("fU1xU1", [((0, 0), 2), ((1, 1), 3), ((1, -1), 1)])
    A_sp, B_sp = {"cod": [V, V, V], "dom": [V]}, {"cod": [V], "dom": [V, W.dual(V)]}
    A, B = tk.tensor_from_spec(A_sp), tk.tensor_from_spec(B_sp)
    Asp, Bsp = A_sp["cod"] + A_sp["dom"], B_sp["cod"] + B_sp["dom"]
    for tup in (([0, 1], [2, 3], [1, 0], [2], [2, 0], [1]), ([1, 0], [3, 2], [0, 1], [2], [0], [2, 1])):
        C = tk.tk_contract_tuples_output(A, *tup[:2], B, *tup[2:])
        at_cod, _ = OC.permuted_spaces(A_sp["cod"], A_sp["dom"], tup[0], tup[1])
        _, bt_dom = OC.permuted_spaces(B_sp["cod"], B_sp["dom"], tup[2], tup[3])
        cod, dom = OC.permuted_spaces(at_cod, bt_dom, tup[4], tup[5])
        assert C.nelems == OL.homspace_layout("fU1xU1", cod, dom).nelems
        assert C.info()["n_cod"] == len(tup[4])
    # reading C2 tuples of A[1,2,3,4] B[4,3,5] -> C[5,1;2]
    C1 = tk.tk_contract_tuples_output(A, [0, 1], [2, 3], B, [1, 0], [2], [2, 0], [1])
    C2 = tk.tk_contract_output(A, [1, 2, 3, 4], B, [4, 3, 5], [5, 1, 2], 2)
    assert np.array_equal(C1.blocks()[1], C2.blocks()[1]) and np.array_equal(C1.blocks()[2], C2.blocks()[2])
    bad = [(([0, 0], [2, 3], [1, 0], [2], [2, 0], [1]), "TK_ERR_INVALID_PERMUTATION"),   # repeated leg
           (([0, 1], [2, 3], [0], [1, 2], [0, 1], [2]), "TK_ERR_INVALID_PERMUTATION"),   # |qA| != |pB|
           (([0, 1], [2, 3], [1, 0], [2], [2, 2], [1]), "TK_ERR_INVALID_PERMUTATION"),   # pAB not a permutation
           (([0, 1], [2, 3], [2, 0], [1], [2, 0], [1]), "TK_ERR_SPACE_MISMATCH")]        # A2 (V) with B2 (V* dom)
    for tup, status in bad:
        with pytest.raises(tk.TKError) as e:
            tk.tk_contract_tuples_output(A, *tup[:2], B, *tup[2:])
        assert e.value.status == status, tup


def test_parse_deligne_spellings():
    """The fermionic product kinds parse under their Deligne spellings (reading C14)."""
    pairs = [("fZ2 x U1 x SU2[(0,0):1, (1,1/2):2]", "fU1xSU2[(0,0):1, (1,1/2):2]"),
             ("fZ2xSU2xSU2[(0,0):1, (1/2,1/2):3]'", "fSU2xSU2[(0,0):1, (1/2,1/2):3]'"),
             ("fZ2 x U1 x U1[(1,1):2, (0,0):1]", "fU1xU1[(1,1):2, (0,0):1]")]
    for a, b in pairs:
        sa, sb = tk.tk_space_parse(a), tk.tk_space_parse(b)
        assert sa.info() == sb.info()
        la, da = sa.sectors()
        lb, db = sb.sectors()
        assert np.array_equal(la, lb) and np.array_equal(da, db)


def test_ncon_output_and_errors():
    """tk_ncon_output (include/tk.h): the HomSpace the pairwise replay gives; malformed networks rejected."""
    V = W.space("U1", [((-1,), 2), ((0,), 3), ((1,), 2)])
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V]})
    B = tk.tensor_from_spec({"cod": [V], "dom": [V, V]})
    M = tk.tensor_from_spec({"cod": [V], "dom": [V]})
    C = tk.tk_ncon_output([A, B, M], [[-1, 1, 2], [2, -2, 3], [3, 1]], [2, 3, 1], 1)
    # replay: A.B over label 2 -> (-1, 1 ; -2, 3), then with M over 3 and 1 -> (-1 ; -2)
    T1 = tk.tk_contract_output(A, [-1, 1, 2], B, [2, -2, 3], [-1, 1, -2, 3], 2)
    C2 = tk.tk_contract_output(T1, [-1, 1, -2, 3], M, [3, 1], [-1, -2], 1)
    assert C.nelems == C2.nelems and C.info() == C2.info()
    assert tk.tk_ncon_workspace([A, B, M], [[-1, 1, 2], [2, -2, 3], [3, 1]], [2, 3, 1], 1) > 0
    bad = [([[-1, 1, 2], [2, -2, 3], [3, 4]], [1, 2, 3], "TK_ERR_MALFORMED_NETWORK"),    # 4 appears once
           ([[-1, 1, 1], [2, -2, 3], [3, 2, 1]], [1, 2, 3], "TK_ERR_MALFORMED_NETWORK"),  # 1 three times
           ([[-1, 1, 2], [2, -3, 3], [3, 1]], [1, 2, 3], "TK_ERR_MALFORMED_NETWORK"),    # open labels -1, -3
           ([[-1, 1, 2], [2, -2, 3], [3, 1]], [1, 2], "TK_ERR_MALFORMED_NETWORK"),       # order misses 3
           ([[-1, 1, 2], [2, -2, 3], [3, 1]], [1, 2, 9], "TK_ERR_UNKNOWN_LABEL")]        # order names 9
    for labels, order, status in bad:
        with pytest.raises(tk.TKError) as e:
            tk.tk_ncon_output([A, B, M] if len(labels[2]) == 2 else [A, B, A], labels, order, 1)
        assert e.value.status == status, (labels, order)
    # a label twice on one tensor is a partial trace (done first): A[-1, 1, 1] is the trace over legs 2, 3
    Ct = tk.tk_ncon_output([A, M], [[-1, 1, 1], [-2, -3]], [1], 1)
    T1 = tk.tk_trace_output(A, [1], [2], [0], [])
    Cr = tk.tk_contract_output(T1, [-1], M, [-2, -3], [-1, -2, -3], 1)
    assert Ct.nelems == Cr.nelems and Ct.info() == Cr.info()


# ------------------------------------------------------------------ plan cache (host side)
def _tiny_pair(tag):
    V = W.space("U1", [((-1,), 1), ((0,), 3), ((1,), 2), ((tag,), 1)])
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V]})
    B = tk.tensor_from_spec({"cod": [V], "dom": [V, V]})
    return A, B


def test_plan_cache_keys_and_bound():
    """Plans are memoised per (structure, labels, device): a repeated query reuses the plan, other labels
    or other spaces make new ones, the LRU keeps at most 512 per cache, tk_cache_clear empties it."""
    tk.tk_cache_clear()
    assert tk.tk_cache_size() == 0
    A, B = _tiny_pair(3)
    la, lb, lc = [1, 2, 3], [3, 4, 5], [1, 4, 2, 5]
    C = tk.tk_contract_output(A, la, B, lb, lc, 2)
    w1 = tk.tk_contract_workspace(A, la, B, lb, C, lc)
    assert tk.tk_cache_size() == 1
    assert tk.tk_contract_workspace(A, la, B, lb, C, lc) == w1
    assert tk.tk_cache_size() == 1                        # same key: cached
    lc2 = [4, 1, 2, 5]
    C2 = tk.tk_contract_output(A, la, B, lb, lc2, 2)
    tk.tk_contract_workspace(A, la, B, lb, C2, lc2)
    assert tk.tk_cache_size() == 2                        # other output labels: a new plan
    A3, B3 = _tiny_pair(4)
    C3 = tk.tk_contract_output(A3, la, B3, lb, lc, 2)
    tk.tk_contract_workspace(A3, la, B3, lb, C3, lc)
    assert tk.tk_cache_size() == 3                        # other spaces: a new plan
    for d in range(5, 5 + 520):                           # bounded LRU
        Ad, Bd = _tiny_pair(d)
        Cd = tk.tk_contract_output(Ad, la, Bd, lb, lc, 2)
        tk.tk_contract_workspace(Ad, la, Bd, lb, Cd, lc)
    assert tk.tk_cache_size() == 512
    tk.tk_cache_clear()
    assert tk.tk_cache_size() == 0


def test_ncon_plan_is_cached():
    """A network's plan (pairwise steps, intermediate HomSpaces, workspace) is memoised by the inputs'
    structure, labels, order and n_cod_out: a repeated query with NEW tensor objects of the same structure
    builds nothing, returns the same workspace size and an output of the same HomSpace; another order or
    other labels make a new plan; tk_cache_clear drops it."""
    from workloads import configs as W
    cfg = W.cfg2()
    names, labels, order, ncod, out_name = W.chain_as_ncon(cfg)
    tk.tk_cache_clear()
    T1 = [tk.tensor_from_spec(cfg["tensors"][nm][0]) for nm in names]
    w1 = tk.tk_ncon_workspace(T1, labels, order, ncod)
    n1 = tk.tk_cache_size()
    assert n1 > 0
    T2 = [tk.tensor_from_spec(cfg["tensors"][nm][0]) for nm in names]   # fresh objects, same structure
    assert tk.tk_ncon_workspace(T2, labels, order, ncod) == w1
    assert tk.tk_cache_size() == n1
    O1 = tk.tk_ncon_output(T1, labels, order, ncod)
    O2 = tk.tk_ncon_output(T2, labels, order, ncod)
    assert tk.tk_cache_size() == n1
    assert O1.info() == O2.info() and O1.nelems == O2.nelems
    del T1, O1                                                          # the cached plan does not borrow them
    assert tk.tk_ncon_workspace(T2, labels, order, ncod) == w1
    tk.tk_ncon_output(T2, labels, order, ncod - 1)                      # another output split: a new plan
    assert tk.tk_cache_size() > n1
    tk.tk_cache_clear()
    assert tk.tk_cache_size() == 0
    assert tk.tk_ncon_workspace(T2, labels, order, ncod) == w1          # rebuilt after the clear


def test_binding_rejects_bad_labels():
    A, B = _tiny_pair(3)
    with pytest.raises(ValueError):
        tk.tk_contract_output(A, [1, 2], B, [3, 4, 5], [1, 4, 2, 5], 2)


@pytest.mark.parametrize("cfgfun", [lambda: W.cfg3(), lambda: W.cfg4(), lambda: W.cfg4(d_leg=320),
                                    lambda: W.cfg7(), lambda: W.cfg8(), lambda: W.cfg2()],
                         ids=["cfg3_chi2048", "cfg4_d384", "cfg4_d320", "cfg7_m700", "cfg8_m270", "cfg2"])
def test_layout_equals_oracle_bench_sizes(cfgfun):
    """Reading C25 at the sizes bench.py / tools/bench_configs.py time: every input tensor AND every
    intermediate / output of the chain (tk_contract_output vs the oracle's output spaces) has the
    oracle's block and subblock layout, integer for integer."""
    cfg = cfgfun()
    T = {n: (spec, tk.tensor_from_spec(spec)) for n, (spec, _) in cfg["tensors"].items()}
    for spec, _ in T.values():
        assert_same_layout(spec)
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        (sa, A), (sb, B) = T[na], T[nb]
        Ct = tk.tk_contract_output(A, la, B, lb, lc, ncod)
        cod, dom = OC.output_spaces(sa["cod"], sa["dom"], sb["cod"], sb["dom"], la, lb, lc, ncod)
        spec = {"cod": cod, "dom": dom}
        assert Ct.nelems == oracle_layout(spec).nelems
        assert_same_layout(spec)
        T[nc] = (spec, Ct)


def _pair_descs(cfg, i):
    steps = cfg["steps"]
    T = {n: tk.tensor_from_spec(spec) for n, (spec, _) in cfg["tensors"].items()}
    for (na, la, nb, lb, nc, lc, ncod) in steps[:i + 2]:
        T[nc] = tk.tk_contract_output(T[na], la, T[nb], lb, lc, ncod)
    (na, la, nb, lb, nc, lc, _), (_, la2, nb2, lb2, nc2, lc2, _) = steps[i], steps[i + 1]
    return (T[na], la, T[nb], lb, T[nc], lc, T[nb2], lb2, T[nc2], lc2)


@pytest.mark.parametrize("cfgfun,fused", [(W.cfg2, [False, True, False]), (lambda: W.cfg3(chi=96), [False, True, False]),
                                          (W.cfg5, []), (W.cfg6, [False, False]),
                                          (lambda: W.cfg7(n_mult=24), [False, False, False])],
                         ids=["cfg2", "cfg3_chi96", "cfg5", "cfg6", "cfg7_m24"])
def test_contract2_fusion_decision(cfgfun, fused):
    """Host-only plan query: which consecutive pairs tk_contract2 runs as one kernel (the abelian MPO pair
    T1.W1 -> T2, T2.W2 -> T3), and the workspace of the others (T plus the larger step workspace)."""
    cfg = cfgfun()
    steps = cfg["steps"]
    got = []
    for i in range(len(steps) - 1):
        d = _pair_descs(cfg, i)
        n, fu = tk.tk_contract2_workspace(*d, want_fused=True)
        got.append(fu)
        if fu:
            assert n == 0
        else:
            A, la, B1, lb1, Tm, lt, B2, lb2, C, lc = d
            n1 = tk.tk_contract_workspace(A, la, B1, lb1, Tm, lt)
            n2 = tk.tk_contract_workspace(Tm, lt, B2, lb2, C, lc)
            assert n >= Tm.nelems * 8 + max(n1, n2)
    assert got == fused


def test_contract2_errors():
    cfg = W.cfg2()
    A, la, B1, lb1, Tm, lt, B2, lb2, C, lc = _pair_descs(cfg, 1)
    with pytest.raises(tk.TKError):  # T is not A.B1's output HomSpace
        tk.tk_contract2_workspace(A, la, B1, lb1, C, lc, B2, lb2, C, lc)
    with pytest.raises(ValueError):
        tk.tk_contract2_workspace(A, la[:-1], B1, lb1, Tm, lt, B2, lb2, C, lc)
