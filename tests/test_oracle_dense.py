"""Pins of the oracle's dense embedding and contraction (abelian, fermionic, SU(2)).

Pins used (SURVEY §8(c) "What pins each part of the oracle"):
  * brute force: explicit loops over every dense index on tiny inputs
  * symmetry invariance: dense tensors vanish outside allowed charge tuples
     / commute with Wigner-D rotations (SU(2))
  * dim(fuse(P)) = prod dim for the layout
  * round trip from_dense o to_dense = id; tier 2 == tier 1 at reduced size
  * associativity of bosonic contraction orders
  * fermions (reading C13): bosonic limit, odd-odd swap = -1,
    permute o inverse = id, bubble-sort accumulation, cyclic bends = +1
"""
import itertools
import math

import numpy as np
import pytest

from oracle import layout as L, dense as Dn, contract as C, blocksparse as BS, sectors
from workloads import configs as W


def sp(kind, secs, dual=False):
    return W.space(kind, secs, dual)


def rand_tensor(kind, cod, dom, seed):
    lt = L.homspace_layout(kind, cod, dom)
    x = np.random.default_rng(seed).standard_normal(lt.nelems)
    return lt, x


# ------------------------------------------------------------------ layout
@pytest.mark.parametrize("kind,secs", [
    ("Z2", [((0,), 2), ((1,), 3)]),
    ("U1", [((-1,), 2), ((0,), 1), ((2,), 3)]),
    ("fU1xU1", [((0, 0), 1), ((1, 1), 2), ((1, -1), 1), ((-1, 1), 2)]),
    ("SU2", [((0,), 2), ((1,), 1), ((2,), 2)]),
    ("fU1xSU2", [((0, 0), 2), ((1, 1), 1), ((-1, 1), 2), ((2, 0), 1), ((0, 2), 1)]),
    ("fSU2xSU2", [((0, 0), 2), ((1, 1), 1), ((0, 2), 1), ((2, 0), 1), ((1, 3), 1)]),
])
def test_fuse_dimension(kind, secs):
    # sum_c rows(c) * d_c over ALL coupled sectors == prod of leg dims
    V = sp(kind, secs)
    for legs in ([V], [V, W.dual(V)], [V, V, W.dual(V)]):
        trees = L.enumerate_trees(kind, legs)
        tot = sum(math.prod(t.dims) * sectors.qdim(kind, c) for c, ts in trees.items() for t in ts)
        assert tot == math.prod(Dn.leg_basis(l)[1] for l in legs)


def test_config_layout_counts():
    # counts re-derived in SURVEY App. B (independent survey scripts)
    c1 = W.cfg1()
    A = c1["tensors"]["A"][0]
    lt = L.homspace_layout("Z2", A["cod"], A["dom"])
    assert [(b[1], b[2]) for b in lt.blocks] == [(128, 128), (128, 128)] and len(lt.subblocks) == 8
    c2 = W.cfg2()
    th = c2["tensors"]["theta"][0]
    lt = L.homspace_layout("U1", th["cod"], th["dom"])
    assert (lt.nelems, len(lt.subblocks), len(lt.blocks)) == (98032, 66, 17)
    c5 = W.cfg5()
    Lt, At = c5["tensors"]["L"][0], c5["tensors"]["A"][0]
    # closed-form block sizes from the SU(2) triangle rule, counted by hand:
    # L: V <- V (x) W, W = 2(0)+(1): rows(j) = n_j, cols(j) = 2 n_j + sum_{j' (x) 1 ni j} n_j'
    n = [24, 40, 40, 32, 24, 12, 6]
    nn = lambda j: n[j] if 0 <= j < len(n) else 0
    adj = lambda j: sum(nn(k) for k in (j - 1, j, j + 1) if k >= 0 and (k > 0 or j == 1) and (j > 0 or k == 1))
    L_tot = sum(nn(j) * (2 * nn(j) + adj(j)) for j in range(7))
    A_tot = sum(adj(j) * nn(j) for j in range(7))
    assert (L_tot, A_tot) == (26028, 14916)
    assert L.homspace_layout("SU2", Lt["cod"], Lt["dom"]).nelems == L_tot
    assert L.homspace_layout("SU2", At["cod"], At["dom"]).nelems == A_tot


# ----------------------------------------------------------- abelian dense
def test_roundtrip_and_invariance_u1():
    V = sp("U1", [((-1,), 2), ((0,), 1), ((2,), 3)])
    cod, dom = [V, W.dual(V)], [V]
    lt, x = rand_tensor("U1", cod, dom, 0)
    D = Dn.to_dense(lt, x)
    assert np.array_equal(Dn.from_dense(lt, D), x)
    # zero outside allowed charge tuples: sum(ket) - sum(bra) == 0
    q = [np.array([s[0] * (-1 if l["dual"] else 1) for s in Dn.sector_of_index(l)]) for l in cod + dom]
    tot = q[0][:, None, None] + q[1][None, :, None] - q[2][None, None, :]
    assert np.all(D[tot != 0] == 0) and np.count_nonzero(D[tot == 0]) == lt.nelems


def test_brute_force_z2_contraction():
    # cfg1 pattern at V = Z2(0=>2, 1=>2): explicit loops vs einsum on the dense embeddings
    V = sp("Z2", [((0,), 2), ((1,), 2)])
    la, xa = rand_tensor("Z2", [V, V], [V, V], 1)
    lb, xb = rand_tensor("Z2", [V, W.dual(V)], [V, V], 2)
    A, B = Dn.to_dense(la, xa), Dn.to_dense(lb, xb)
    Cd = C.contract_einsum(A, [1, 3, 2, 4], B, [4, 3, 5, 6], [1, 2, 5, 6])
    n = 4
    ref = np.zeros((n, n, n, n))
    for a, b, e, f, c, d in itertools.product(range(n), repeat=6):
        ref[a, b, e, f] += A[a, c, b, d] * B[d, c, e, f]
    assert np.abs(Cd - ref).max() < 1e-13
    # result is Z2-symmetric: parity of (a + b + e + f) even
    par = np.array([0, 0, 1, 1])
    tot = (par[:, None, None, None] + par[None, :, None, None] + par[None, None, :, None] + par[None, None, None, :]) % 2
    assert np.all(Cd[tot == 1] == 0)


def _chain_dense(cfg):
    out = {}
    for name, (t, idx) in cfg["tensors"].items():
        lt, x = rand_tensor(cfg["kind"], t["cod"], t["dom"], 100 + idx)
        out[name] = (Dn.to_dense(lt, x), t["cod"] + t["dom"], len(t["cod"]))
    return out


def test_associativity_bosonic_chain():
    # all contraction paths of a consistent framework agree (bosonic: cfg2 shape)
    cfg = W.cfg2(chi=24)
    T = _chain_dense(cfg)
    Ld, th, W1, W2, R = (T[k][0] for k in ("L", "theta", "W1", "W2", "R"))
    al_, al, a, s1, s2, be, s1p, b, s2p, c, bep = range(1, 12)
    x = C.contract_einsum(Ld, [al_, al, a], th, [al, s1, s2, be], [al_, a, s1, s2, be])
    x = C.contract_einsum(x, [al_, a, s1, s2, be], W1, [a, s1p, s1, b], [al_, s2, be, s1p, b])
    x = C.contract_einsum(x, [al_, s2, be, s1p, b], W2, [b, s2p, s2, c], [al_, be, s1p, s2p, c])
    ref = C.contract_einsum(x, [al_, be, s1p, s2p, c], R, [c, bep, be], [al_, s1p, s2p, bep])
    # other order: (W1 W2) R first, then L theta
    y = C.contract_einsum(W1, [a, s1p, s1, b], W2, [b, s2p, s2, c], [a, s1p, s1, s2p, s2, c])
    y = C.contract_einsum(y, [a, s1p, s1, s2p, s2, c], R, [c, bep, be], [a, s1p, s1, s2p, s2, bep, be])
    z = C.contract_einsum(Ld, [al_, al, a], th, [al, s1, s2, be], [al_, a, s1, s2, be])
    out = C.contract_einsum(z, [al_, a, s1, s2, be], y, [a, s1p, s1, s2p, s2, bep, be], [al_, s1p, s2p, bep])
    assert C.rel_frobenius(out, ref) < 1e-13


@pytest.mark.parametrize("cfgfun", [lambda: W.cfg4(d_leg=24), lambda: W.cfg2(chi=40), lambda: W.cfg3(chi=40)])
def test_tier2_equals_tier1(cfgfun):
    cfg = cfgfun()
    kind = cfg["kind"]
    tens = {}
    for name, (t, idx) in cfg["tensors"].items():
        lt, x = rand_tensor(kind, t["cod"], t["dom"], 7 + idx)
        tens[name] = (t["cod"], t["dom"], lt, x)
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        Acod, Adom, lta, xa = tens[na]
        Bcod, Bdom, ltb, xb = tens[nb]
        ref = C.contract(kind, Dn.to_dense(lta, xa), Acod + Adom, len(Acod), la,
                         Dn.to_dense(ltb, xb), Bcod + Bdom, len(Bcod), lb, lc, ncod)
        blocks, (Ccod, Cdom) = BS.contract_blocks(kind, BS.to_blocks(lta, xa), Acod, Adom, la,
                                                  BS.to_blocks(ltb, xb), Bcod, Bdom, lb, lc, ncod)
        ltc = L.homspace_layout(kind, Ccod, Cdom)
        flat = np.zeros(ltc.nelems)
        for sb in ltc.subblocks:
            k = tuple(sb.key[0]) + tuple(sb.key[3])
            if k in blocks:
                Dn.subblock_array(ltc, flat, sb)[...] = blocks[k]
        got = Dn.to_dense(ltc, flat)
        assert C.rel_frobenius(got, ref) < 1e-13
        # the dense result is supported only on the output layout (symmetry invariance)
        assert C.rel_frobenius(Dn.to_dense(ltc, Dn.from_dense(ltc, ref)), ref) < 1e-14
        tens[nc] = (Ccod, Cdom, ltc, Dn.from_dense(ltc, ref))


# ---------------------------------------------------------------- fermions
def test_fermion_bosonic_limit():
    V = sp("U1xU1", [((0, 0), 2), ((1, 1), 1), ((2, 0), 2)])
    la, xa = rand_tensor("U1xU1", [V, V], [V], 3)
    lb, xb = rand_tensor("U1xU1", [V], [V, W.dual(V)], 4)
    A, B = Dn.to_dense(la, xa), Dn.to_dense(lb, xb)
    r1 = C.contract_alg4(A, [V, V, V], 2, [1, 2, 3], B, [V, V, W.dual(V)], 1, [3, 4, 5], [2, 5, 1, 4], 2)
    r2 = C.contract_einsum(A, [1, 2, 3], B, [3, 4, 5], [2, 5, 1, 4])
    assert C.rel_frobenius(r1, r2) < 1e-14


def test_fermion_odd_odd_swap_sign():
    # P:2361 R^{JJ}_I = -1: swapping two odd legs negates the block; even-odd does not
    V = sp("fZ2", [((0,), 1), ((1,), 1)])
    D = np.zeros((2, 2))
    D[1, 1] = 1.0   # odd (x) odd channel
    D[0, 0] = 1.0   # even (x) even
    par = [Dn.parity_vector(V)] * 2
    out = C.permute_dense(D, par, 2, (1, 0), ())
    assert out[1, 1] == -1.0 and out[0, 0] == 1.0


def test_fermion_permute_inverse_and_bubble_sort():
    rng = np.random.default_rng(5)
    V = sp("fU1xU1", [((0, 0), 1), ((1, 1), 2), ((1, -1), 1), ((2, 0), 1)])
    cod, dom = [V, V, W.dual(V)], [V, V]
    lt, x = rand_tensor("fU1xU1", cod, dom, 6)
    D = Dn.to_dense(lt, x)
    par = [Dn.parity_vector(s) for s in cod + dom]
    N, n1 = 5, 3
    for _ in range(20):
        perm = list(rng.permutation(N))
        k = int(rng.integers(0, N + 1))
        p, q = perm[:k], perm[k:]
        P = C.permute_dense(D, par, n1, p, q)
        # inverse: legs of P are (p..., q...) with codomain count k
        order = p + q
        inv = [order.index(i) for i in range(N)]
        back = C.permute_dense(P, [par[i] for i in order], k, inv[:n1], inv[n1:])
        assert np.array_equal(back, D)
        # bubble sort: the sign equals the product of adjacent-swap signs on the
        # fully bent ordering S -> T
        S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
        T = list(p) + list(reversed(q))
        cur = S[:]
        swaps = []
        for i in range(N):
            for j in range(N - 1 - i):
                if T.index(cur[j]) > T.index(cur[j + 1]):
                    swaps.append((cur[j], cur[j + 1]))
                    cur[j], cur[j + 1] = cur[j + 1], cur[j]
        assert cur == T
        assert sorted(tuple(sorted(s)) for s in swaps) == sorted(C.koszul_sign_pairs(n1, N - n1, p, q))


def test_fermion_pure_bends_sign_free():
    # right bends only re-partition the bent order S (T == S): no sign (reading C13; P:2355-2361
    # chi_J = d_J = 1, F trivial => B-symbols are 1). A genuine rotation of S moves an odd leg
    # past the others; on an even-parity tensor that is the twist theta_J = -1.
    N, n1 = 5, 2
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    for k in range(N + 1):
        p, q = S[:k], list(reversed(S[k:]))
        assert C.koszul_sign_pairs(n1, N - n1, p, q) == []
    V = sp("fZ2", [((0,), 1), ((1,), 1)])
    D = np.zeros((2, 2, 2))
    D[1, 1, 0] = 1.0     # odd, odd ; even  (total parity even)
    par = [Dn.parity_vector(V)] * 3
    rot = C.permute_dense(D, par, 2, (1, 2), (0,))   # S=(0,1,2) -> T=(1,2,0): leg 0 moved around
    assert rot[1, 0, 1] == -1.0


# ------------------------------------------------------------------- SU(2)
def _wigner_D(j, th):
    from scipy.linalg import expm
    from oracle import su2
    Jz, Jp, Jm = su2.spin_matrices(j)
    return expm(-1j * (th[0] * (Jp + Jm) / 2 + th[1] * (Jp - Jm) / 2j + th[2] * Jz))


def _leg_rep(spc, th):
    blocks = []
    for lab, n in sorted(spc["sectors"]):
        Dj = _wigner_D(lab[0], th)
        for _ in range(n):
            blocks.append(Dj)
    from scipy.linalg import block_diag
    M = block_diag(*blocks)
    return M.conj() if spc["dual"] else M


def test_su2_equivariance_roundtrip():
    V = sp("SU2", [((0,), 2), ((1,), 1), ((2,), 2)])
    P = sp("SU2", [((2,), 1)])
    th = np.array([0.3, -1.1, 0.7])
    for cod, dom in (([V, P], [V]), ([V, W.dual(V)], [P]), ([W.dual(P), V], [V, W.dual(P)])):
        lt, x = rand_tensor("SU2", cod, dom, 9)
        D = Dn.to_dense(lt, x)
        assert np.abs(Dn.from_dense(lt, D) - x).max() < 1e-13
        Mc = np.ones((1, 1))
        for s in cod:
            Mc = np.kron(Mc, _leg_rep(s, th))
        Md = np.ones((1, 1))
        for s in dom:
            Md = np.kron(Md, _leg_rep(s, th))
        T = D.reshape(Mc.shape[0], Md.shape[0])
        assert np.abs(Mc @ T - T @ Md).max() < 1e-12


@pytest.mark.parametrize("cfgfun", [lambda: W.cfg5(mults=(2, 2, 1, 1, 1, 1, 1)),
                                    lambda: W.cfg6(mults=(2, 2, 1, 1, 1, 1, 1))], ids=["cfg5", "cfg6"])
def test_su2_contraction_supported_on_output_layout(cfgfun):
    """Every step's dense einsum result lies in the span of the output layout's CG basis (it is an
    SU(2) intertwiner): projecting onto the reduced blocks and back loses nothing."""
    cfg = cfgfun()
    specs = {k: v[0] for k, v in cfg["tensors"].items()}
    dense = {}
    for i, (k, (spec, _)) in enumerate(cfg["tensors"].items()):
        lt, x = rand_tensor("SU2", spec["cod"], spec["dom"], 11 + i)
        dense[k] = Dn.to_dense(lt, x)
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        out = C.contract_einsum(dense[na], la, dense[nb], lb, lc)
        Ccod, Cdom = C.output_spaces(specs[na]["cod"], specs[na]["dom"], specs[nb]["cod"], specs[nb]["dom"],
                                     la, lb, lc, ncod)
        specs[nc] = {"cod": Ccod, "dom": Cdom}
        lc_ = L.homspace_layout("SU2", Ccod, Cdom)
        back = Dn.to_dense(lc_, Dn.from_dense(lc_, out))
        assert C.rel_frobenius(back, out) < 1e-13
        dense[nc] = out


# ------------------------------------------------------ fZ2 x U1 x SU2
def _leg_rep_u1su2(spc, th, phi):
    """U(1) x SU(2) action on one fU1xSU2 leg: exp(i N phi) (x) D^j(th) per multiplet."""
    from scipy.linalg import block_diag
    blocks = []
    for lab, n in sorted(spc["sectors"]):
        Dj = np.exp(1j * lab[0] * phi) * _wigner_D(lab[1], th)
        blocks.extend([Dj] * n)
    M = block_diag(*blocks)
    return M.conj() if spc["dual"] else M


HUB = [((0, 0), 2), ((1, 1), 1), ((-1, 1), 2), ((2, 0), 1), ((1, 3), 1)]


def test_u1su2_equivariance_roundtrip():
    """Deligne product embedding: the dense tensor is invariant under U(1) x SU(2)
    (charge phase times Wigner-D on every leg), and from_dense o to_dense = id."""
    V = sp("fU1xSU2", HUB)
    P = sp("fU1xSU2", [((0, 0), 1), ((1, 1), 1), ((2, 0), 1)])
    th, phi = np.array([0.4, -0.9, 1.3]), 0.77
    for cod, dom in (([V, P], [V]), ([V, W.dual(V)], [P]), ([W.dual(P), V], [V, W.dual(P)])):
        lt, x = rand_tensor("fU1xSU2", cod, dom, 21)
        D = Dn.to_dense(lt, x)
        assert np.abs(Dn.from_dense(lt, D) - x).max() < 1e-13
        Mc = np.ones((1, 1))
        for s_ in cod:
            Mc = np.kron(Mc, _leg_rep_u1su2(s_, th, phi))
        Md = np.ones((1, 1))
        for s_ in dom:
            Md = np.kron(Md, _leg_rep_u1su2(s_, th, phi))
        T = D.reshape(Mc.shape[0], Md.shape[0])
        assert np.abs(Mc @ T - T @ Md).max() < 1e-12


def test_u1su2_even_charges_reduce_to_su2():
    """Bosonic limit of the product: with every charge even the fermionic Alg. 4 contraction equals the
    plain einsum, and the dense embedding equals the SU(2) one (same reduced values, same CG)."""
    # sectors listed so that the (N, 2j) order equals the 2j order: both legs index the same basis
    Vh = sp("fU1xSU2", [((0, 0), 2), ((2, 2), 1), ((4, 4), 1)])
    Vs = sp("SU2", [((0,), 2), ((2,), 1), ((4,), 1)])  # the same spins, charges dropped
    la, xa = rand_tensor("fU1xSU2", [Vh, Vh], [Vh], 31)
    ls, xs = rand_tensor("SU2", [Vs, Vs], [Vs], 31)
    Dh, Ds = Dn.to_dense(la, xa), Dn.to_dense(ls, xs)
    assert Dh.shape == Ds.shape
    lb, xb = rand_tensor("fU1xSU2", [Vh], [Vh, W.dual(Vh)], 32)
    B = Dn.to_dense(lb, xb)
    r1 = C.contract_alg4(Dh, [Vh, Vh, Vh], 2, [1, 2, 3], B, [Vh, Vh, W.dual(Vh)], 1, [3, 4, 5], [2, 5, 1, 4], 2)
    r2 = C.contract_einsum(Dh, [1, 2, 3], B, [3, 4, 5], [2, 5, 1, 4])
    assert C.rel_frobenius(r1, r2) < 1e-14
    # where the U(1) charges allow a block, the fU1xSU2 tensor IS an SU(2) intertwiner: its dense array
    # is supported on the SU(2) layout of the same legs (projection onto the SU(2) basis loses nothing)
    back = Dn.to_dense(ls, Dn.from_dense(ls, Dh))
    assert C.rel_frobenius(back, Dh) < 1e-13


def test_u1su2_fermion_permute_inverse():
    rng = np.random.default_rng(8)
    V = sp("fU1xSU2", HUB)
    cod, dom = [V, W.dual(V)], [V, V]
    lt, x = rand_tensor("fU1xSU2", cod, dom, 33)
    D = Dn.to_dense(lt, x)
    par = [Dn.parity_vector(s_) for s_ in cod + dom]
    N, n1 = 4, 2
    for _ in range(10):
        perm = list(rng.permutation(N))
        k = int(rng.integers(0, N + 1))
        p, q = perm[:k], perm[k:]
        Pd = C.permute_dense(D, par, n1, p, q)
        order = p + q
        inv = [order.index(i) for i in range(N)]
        back = C.permute_dense(Pd, [par[i] for i in order], k, inv[:n1], inv[n1:])
        assert np.array_equal(back, D)
        # the permuted dense tensor is again an intertwiner of the permuted HomSpace
        c2, d2 = C.permuted_spaces(cod, dom, p, q)
        l2 = L.homspace_layout("fU1xSU2", c2, d2)
        assert C.rel_frobenius(Dn.to_dense(l2, Dn.from_dense(l2, Pd)), Pd) < 1e-13


# --------------------------------------------- fZ2 x SU2 x SU2 (half filling)
SO4 = [((0, 0), 2), ((1, 1), 1), ((0, 2), 1), ((2, 0), 2), ((1, 3), 1)]


def _leg_rep_su2su2(spc, thc, ths):
    from scipy.linalg import block_diag
    blocks = []
    for lab, n in sorted(spc["sectors"]):
        blocks.extend([np.kron(_wigner_D(lab[0], thc), _wigner_D(lab[1], ths))] * n)
    M = block_diag(*blocks)
    return M.conj() if spc["dual"] else M


def test_su2su2_equivariance_roundtrip():
    """Deligne product embedding: invariant under SU(2) x SU(2) (charge and spin rotations)."""
    V = sp("fSU2xSU2", SO4)
    P = sp("fSU2xSU2", [((0, 1), 1), ((1, 0), 1)])
    thc, ths = np.array([0.2, 1.1, -0.5]), np.array([-0.7, 0.3, 0.9])
    # V's sectors have j_c + j_s integer, P's half-integer (one site): pair the P legs
    for cod, dom in (([V, P], [V, P]), ([V, W.dual(V)], [P, P]), ([W.dual(P), V], [V, W.dual(P)])):
        lt, x = rand_tensor("fSU2xSU2", cod, dom, 41)
        assert lt.nelems > 0
        D = Dn.to_dense(lt, x)
        assert np.abs(Dn.from_dense(lt, D) - x).max() < 1e-13
        Mc = np.ones((1, 1))
        for s_ in cod:
            Mc = np.kron(Mc, _leg_rep_su2su2(s_, thc, ths))
        Md = np.ones((1, 1))
        for s_ in dom:
            Md = np.kron(Md, _leg_rep_su2su2(s_, thc, ths))
        T = D.reshape(Mc.shape[0], Md.shape[0])
        assert np.abs(Mc @ T - T @ Md).max() < 1e-12


@pytest.mark.parametrize("factor", [0, 1])
def test_su2su2_single_factor_reduces_to_su2(factor):
    """With one factor trivial (j = 0 on every leg) the product embedding IS the SU(2) one."""
    js = [0, 2, 4]
    lab = (lambda j: (0, j)) if factor == 1 else (lambda j: (j, 0))
    Vh = sp("fSU2xSU2", [(lab(j), n) for j, n in zip(js, (2, 1, 1))])
    Vs = sp("SU2", [((j,), n) for j, n in zip(js, (2, 1, 1))])
    for cod_d, dom_d in (([0, 0], [0]), ([0, 1], [0, 0])):
        ch = [W.dual(Vh) if d else Vh for d in cod_d], [W.dual(Vh) if d else Vh for d in dom_d]
        cs = [W.dual(Vs) if d else Vs for d in cod_d], [W.dual(Vs) if d else Vs for d in dom_d]
        lh, xh = rand_tensor("fSU2xSU2", *ch, 51)
        ls, xs = rand_tensor("SU2", *cs, 51)
        assert lh.nelems == ls.nelems
        assert np.array_equal(Dn.to_dense(lh, xh), Dn.to_dense(ls, xs))


def test_su2su2_fermion_permute_inverse():
    rng = np.random.default_rng(9)
    V = sp("fSU2xSU2", SO4)
    cod, dom = [V, W.dual(V)], [V, V]
    lt, x = rand_tensor("fSU2xSU2", cod, dom, 43)
    D = Dn.to_dense(lt, x)
    par = [Dn.parity_vector(s_) for s_ in cod + dom]
    N, n1 = 4, 2
    for _ in range(8):
        perm = list(rng.permutation(N))
        k = int(rng.integers(0, N + 1))
        p, q = perm[:k], perm[k:]
        Pd = C.permute_dense(D, par, n1, p, q)
        order = p + q
        inv = [order.index(i) for i in range(N)]
        assert np.array_equal(C.permute_dense(Pd, [par[i] for i in order], k, inv[:n1], inv[n1:]), D)
        c2, d2 = C.permuted_spaces(cod, dom, p, q)
        l2 = L.homspace_layout("fSU2xSU2", c2, d2)
        assert C.rel_frobenius(Dn.to_dense(l2, Dn.from_dense(l2, Pd)), Pd) < 1e-13


# ------------------------------------------------------------ Alg. 4 with explicit tuples
def test_alg4_tuples_bosonic_equals_einsum():
    """Dense Alg. 4 with arbitrary tuple orders reproduces the plain einsum (bosonic: the
    permutes are basis relabelings, so every (pA, qA, pB, qB, pAB, qAB) gives the same C)."""
    rng = np.random.default_rng(21)
    V = sp("U1", [((-1,), 2), ((0,), 3), ((1,), 2)])
    la, xa = rand_tensor("U1", [V, V], [V], 1)
    lb, xb = rand_tensor("U1", [V], [V, V], 2)
    A, B = Dn.to_dense(la, xa), Dn.to_dense(lb, xb)
    want = C.contract_einsum(A, [1, 2, 3], B, [3, 2, 5], [5, 1])
    for _ in range(6):
        ka = [int(x) for x in rng.permutation([1, 2])]   # contracted A legs (labels 2, 3 at A legs 1, 2)
        qA = ka
        pB = [{1: 1, 2: 0}[i] for i in qA]                # label 2 is B leg 1, label 3 is B leg 0
        got = C.contract_alg4_tuples(A, [V, V, V], 2, B, [V, V, V], 1, [0], qA, pB, [2], [1], [0])
        assert C.rel_frobenius(got, want) < 1e-14


def test_alg4_tuples_fermionic_reorder_invariance():
    """Reading C13 makes the Koszul sign a group action (permute o inverse = id), so under Alg. 4:
    (i) reordering A~'s codomain legs pA (with pAB compensating) leaves C unchanged, and (ii) reordering
    the contracted legs jointly in qA and pB leaves C unchanged (paired legs carry equal parities, so
    the two domain/codomain signs cancel)."""
    V = sp("fU1xU1", [((0, 0), 1), ((1, 1), 2), ((1, -1), 1), ((-1, 1), 1), ((-1, -1), 1), ((2, 0), 1)])
    la, xa = rand_tensor("fU1xU1", [V, V, V], [V], 7)      # A: V V V <- V, legs 0..3
    lb, xb = rand_tensor("fU1xU1", [V], [V, W.dual(V)], 8)  # B: V <- V V*, legs 0..2
    A, B = Dn.to_dense(la, xa), Dn.to_dense(lb, xb)
    Asp, Bsp = [V, V, V, V], [V, V, W.dual(V)]
    # ket/bra pairs: A leg 2 (codomain V) with B leg 1 (domain V), A leg 3 (domain V) with B leg 0 (codomain V)
    base = C.contract_alg4_tuples(A, Asp, 3, B, Bsp, 1, [0, 1], [2, 3], [1, 0], [2], [2, 0], [1])
    # (i) pA reversed; C~ legs are now (1, 0, B2), so pAB/qAB must name them accordingly
    r1 = C.contract_alg4_tuples(A, Asp, 3, B, Bsp, 1, [1, 0], [2, 3], [1, 0], [2], [2, 1], [0])
    assert np.allclose(r1, base, rtol=0, atol=1e-14)
    # (ii) contracted legs in the other order on both sides
    r2 = C.contract_alg4_tuples(A, Asp, 3, B, Bsp, 1, [0, 1], [3, 2], [0, 1], [2], [2, 0], [1])
    assert np.allclose(r2, base, rtol=0, atol=1e-14)
    # the same checks on an output permute that crosses A1 and B2 (C[1,5;2]): there the signs are not
    # trivial -- dropping them (bosonic einsum) differs -- and the invariances still hold
    cross = C.contract_alg4_tuples(A, Asp, 3, B, Bsp, 1, [0, 1], [2, 3], [1, 0], [2], [0, 2], [1])
    bos = C.contract_einsum(A, [1, 2, 3, 4], B, [4, 3, 5], [1, 5, 2])
    assert C.rel_frobenius(bos, cross) > 1e-3
    r3 = C.contract_alg4_tuples(A, Asp, 3, B, Bsp, 1, [1, 0], [3, 2], [0, 1], [2], [1, 2], [0])
    assert np.allclose(r3, cross, rtol=0, atol=1e-14)


# ----------------------------------------------------------- SURVEY App. B integers (timed sizes)
def _step_stats(cfg):
    """Per step of a config, from the oracle's layouts only: (elements, subblocks) of the operands and of
    C~, and the useful GEMM flops sum_c 2 M_c K_c N_c of A~ B~ under the reading-C2 tuples."""
    kind = cfg["kind"]
    spaces = {n: (t["cod"], t["dom"]) for n, (t, _) in cfg["tensors"].items()}
    out = []
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        (Ac, Ad), (Bc, Bd) = spaces[na], spaces[nb]
        pA, qA, pB, qB, pAB, qAB = C.tuples_from_labels(la, lb, lc, ncod)
        at = L.homspace_layout(kind, *C.permuted_spaces(Ac, Ad, pA, qA))
        bt = L.homspace_layout(kind, *C.permuted_spaces(Bc, Bd, pB, qB))
        bcols = {b[0]: (b[1], b[2]) for b in bt.blocks}
        flops = sum(2 * r * k * bcols[c][1] for (c, r, k, _) in at.blocks if c in bcols)
        cod, dom = C.output_spaces(Ac, Ad, Bc, Bd, la, lb, lc, ncod)
        ct = L.homspace_layout(kind, cod, dom)
        spaces[nc] = (cod, dom)
        out.append({"A": (at.nelems, len(at.subblocks)), "B": (bt.nelems, len(bt.subblocks)),
                    "C": (ct.nelems, len(ct.subblocks)), "flops": flops})
    return out


def test_appendix_b_cfg2_cfg3_chains():
    """SURVEY App. B tables (independent survey scripts): cfg2 and cfg3 per-step operand sizes and flops."""
    s2 = _step_stats(W.cfg2())
    assert [x["flops"] for x in s2] == [53773296, 3322556, 3322556, 53773296]
    assert sum(x["flops"] for x in s2) == 114191704
    assert [x["A"] for x in s2] == [(122884, 49), (484894, 194), (484894, 194), (484894, 194)]
    assert [x["B"] for x in s2] == [(98032, 66), (34, 10), (34, 10), (122884, 49)]
    assert [x["C"] for x in s2] == [(484894, 194)] * 3 + [(98032, 66)]
    s3 = _step_stats(W.cfg3())
    assert [x["flops"] for x in s3] == [433399764, 60924864, 60924864, 433419928]
    assert sum(x["flops"] for x in s3) == 988669420
    assert [x["A"] for x in s3] == [(521456, 701), (6732096, 9756), (6732096, 9756), (6732096, 9756)]
    assert [x["B"] for x in s3] == [(708260, 2008), (176, 44), (176, 44), (521456, 701)]
    assert [x["C"] for x in s3] == [(6732096, 9756)] * 3 + [(708260, 2008)]
    th = W.cfg3()["tensors"]["theta"][0]
    lt = L.homspace_layout("fU1xU1", th["cod"], th["dom"])
    assert (lt.nelems, len(lt.subblocks), len(lt.blocks)) == (708260, 2008, 157)


@pytest.mark.parametrize("d_leg,elems,subs,blocks,flops", [
    (64, 854974, 4579, 37, 409405460),
    (128, 13569540, 5340, 39, 25757272064),
    (320, 534794900, 6181, 41, 6401382315008),
    (384, 1110720212, 6181, 41, 19215054235248),
])
def test_appendix_b_cfg4(d_leg, elems, subs, blocks, flops):
    """stored elements, subblocks, GEMM blocks and useful flops per D_leg
    (ComplexF64 at D_leg 320: 4x the real count, reading C21)."""
    cfg = W.cfg4(d_leg=d_leg)
    A = cfg["tensors"]["A"][0]
    lt = L.homspace_layout("U1", A["cod"], A["dom"])
    assert (lt.nelems, len(lt.subblocks)) == (elems, subs)
    st = _step_stats(cfg)[0]
    assert st["flops"] == flops and st["C"][0] == elems
    (_, la, _, lb, _, lc, ncod) = cfg["steps"][0]
    pA, qA, _, _, _, _ = C.tuples_from_labels(la, lb, lc, ncod)
    at = L.homspace_layout("U1", *C.permuted_spaces(A["cod"], A["dom"], pA, qA))
    assert len(at.blocks) == blocks
