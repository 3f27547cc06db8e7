"""The five BASELINE.json configs as plain data (spaces, tensors, contraction order).

Spaces are dicts {"kind": str, "sectors": [(label, degeneracy), ...], "dual": bool}
with labels as tuples of ints: Z2 (0|1,), U1 (q,), U1xU1/fU1xU1 (N, 2Sz), SU2 (2j,).
`sectors` always lists the sectors of the underlying (non-dual) space V; a dual
space V* is the same dict with "dual": True (reading C6).

Readings: C3 leg spaces/arrows from the paper's benchmark
spaces, C15 Gaussian rounding, C16 sigma units, C17 literal 13x13
cfg3 grid, C18 cfg3 MPO charges, C19 cfg5 MPO multiplets, C20 cfg4 leg-dim knob.
No arithmetic of the method lives here.
"""
import math


def space(kind, sectors, dual=False):
    return {"kind": kind, "sectors": sorted((tuple(l), int(d)) for l, d in sectors if d > 0), "dual": dual}


def dual(sp):
    return {"kind": sp["kind"], "sectors": list(sp["sectors"]), "dual": not sp["dual"]}


def gaussian_degeneracies(labels, weights, total, tie_key):
    """Reading C15: n = floor(T w / sum w), then largest remainder.

    Ties in the remainder are broken by `tie_key(label)` (smaller first: |q| or
    |N|+|2Sz|), then by ascending label. Zero degeneracies are dropped.
    """
    wsum = sum(weights)
    exact = [total * w / wsum for w in weights]
    base = [int(math.floor(x)) for x in exact]
    rem = total - sum(base)
    order = sorted(range(len(labels)), key=lambda i: (-(exact[i] - base[i]), tie_key(labels[i]), labels[i]))
    for i in order[:rem]:
        base[i] += 1
    return [(labels[i], base[i]) for i in range(len(labels)) if base[i] > 0]


# ---------------------------------------------------------------- config 1 (Z2)
def cfg1():
    V = space("Z2", [((0,), 8), ((1,), 8)])
    A = {"cod": [V, V], "dom": [V, V]}            # legs (a, c; b, d)
    B = {"cod": [V, dual(V)], "dom": [V, V]}      # legs (d, c; e, f)
    a, b, c, d, e, f = 1, 2, 3, 4, 5, 6
    return {
        "cfg": 1, "kind": "Z2", "dtype": "f64",
        "tensors": {"A": (A, 0), "B": (B, 1)},
        "steps": [("A", [a, c, b, d], "B", [d, c, e, f], "C", [a, b, e, f], 2)],
    }


# -------------------------------------------------------- config 2 (U(1) DMRG)
def _u1_bond(chi, qmax, sigma):
    labels = [(q,) for q in range(-qmax, qmax + 1, 2)]
    weights = [math.exp(-q * q / (2 * sigma * sigma)) for (q,) in labels]
    return gaussian_degeneracies(labels, weights, chi, lambda l: abs(l[0]))


def _dmrg_chain(cfg, kind, P, W, V):
    # C3: L = FL: V <- V (x) W ; theta: V (x) P (x) P <- V ; W = O: W (x) P <- P (x) W ;
    #     R = FR: W (x) V* <- V*
    L = {"cod": [V], "dom": [V, W]}                        # (alpha', alpha, a)
    TH = {"cod": [V, P, P], "dom": [V]}                    # (alpha, s1, s2, beta)
    W1 = {"cod": [W, P], "dom": [P, W]}                    # (a, s1', s1, b)
    W2 = {"cod": [W, P], "dom": [P, W]}                    # (b, s2', s2, c)
    R = {"cod": [W, dual(V)], "dom": [dual(V)]}            # (c, beta', beta)
    al_, al, a, s1, s2, be, s1p, b, s2p, c, bep = range(1, 12)
    return {
        "cfg": cfg, "kind": kind, "dtype": "f64",
        "tensors": {"L": (L, 0), "theta": (TH, 1), "W1": (W1, 2), "W2": (W2, 3), "R": (R, 4)},
        "steps": [
            ("L", [al_, al, a], "theta", [al, s1, s2, be], "T1", [al_, a, s1, s2, be], 2),
            ("T1", [al_, a, s1, s2, be], "W1", [a, s1p, s1, b], "T2", [al_, s2, be, s1p, b], 3),
            ("T2", [al_, s2, be, s1p, b], "W2", [b, s2p, s2, c], "T3", [al_, be, s1p, s2p, c], 3),
            ("T3", [al_, be, s1p, s2p, c], "R", [c, bep, be], "out", [al_, s1p, s2p, bep], 3),
        ],
    }


def cfg2(chi=512):
    P = space("U1", [((1,), 1), ((-1,), 1)])
    W = space("U1", [((0,), 3), ((2,), 1), ((-2,), 1)])
    V = space("U1", _u1_bond(chi, 16, 6.0))
    return _dmrg_chain(2, "U1", P, W, V)


# ------------------------------------------- config 3 (fermionic U(1)xU(1) Hubbard)
def _u1u1_bond(chi, sigma_n=2.5, sigma_s=2.5):
    labels = [(n, s) for n in range(-6, 7) for s in range(-6, 7)]  # reading C17: literal 13x13 grid
    weights = [math.exp(-n * n / (2 * sigma_n ** 2) - s * s / (2 * sigma_s ** 2)) for n, s in labels]
    return gaussian_degeneracies(labels, weights, chi, lambda l: abs(l[0]) + abs(l[1]))


def cfg3(chi=2048):
    P = space("fU1xU1", [((0, 0), 1), ((1, 1), 1), ((1, -1), 1), ((2, 0), 1)])
    # C18: identity channels + four single-fermion operators, D = 10
    W = space("fU1xU1", [((0, 0), 2), ((1, 1), 2), ((1, -1), 2), ((-1, 1), 2), ((-1, -1), 2)])
    V = space("fU1xU1", _u1u1_bond(chi))
    return _dmrg_chain(3, "fU1xU1", P, W, V)


# ------------------------------------------------------- config 4 (U(1) PEPS)
def cfg4_leg(d_leg):
    labels = [(q,) for q in range(-10, 11)]
    weights = [math.exp(-q * q / (2 * 4.0 ** 2)) for (q,) in labels]
    return space("U1", gaussian_degeneracies(labels, weights, d_leg, lambda l: abs(l[0])))


def cfg4(d_leg=384, complex_=False):
    V = cfg4_leg(d_leg)
    A = {"cod": [V, V], "dom": [V, V]}   # (x1, x2; x3, x4)
    B = {"cod": [V, V], "dom": [V, V]}   # (y1, y2; y3, y4)
    x1, x2, x3, x4, y2, y4 = 1, 2, 3, 4, 5, 6
    # contract x2-y3 and x4-y1: B's legs (y1, y2; y3, y4) = (x4, y2; x2, y4)
    return {
        "cfg": 4, "kind": "U1", "dtype": "c64" if complex_ else "f64", "d_leg": d_leg,
        "tensors": {"A": (A, 0), "B": (B, 1)},
        "steps": [("A", [x1, x2, x3, x4], "B", [x4, y2, x2, y4], "C", [x1, y2, x3, y4], 2)],
    }


# --------------------------------------------------------------- config 5 (SU(2))
def cfg5(mults=(24, 40, 40, 32, 24, 12, 6)):
    P = space("SU2", [((2,), 1)])                                   # spin 1
    V = space("SU2", [((2 * j,), m) for j, m in enumerate(mults)])  # j = 0..6
    W = space("SU2", [((0,), 2), ((2,), 1)])                        # C19: 2 x (0) + 1 x (1)
    L = {"cod": [V], "dom": [V, W]}      # FL: V <- V (x) W  (alpha'; alpha, a)
    A = {"cod": [V, P], "dom": [V]}      # V (x) P <- V      (alpha, s; beta)
    al_, al, a, s, be = 1, 2, 3, 4, 5
    return {
        "cfg": 5, "kind": "SU2", "dtype": "f64",
        "tensors": {"L": (L, 0), "A": (A, 1)},
        "steps": [("L", [al_, al, a], "A", [al, s, be], "C", [al_, s, a, be], 2)],
    }


# ------------------------------- config 6 (single-site SU(2) chain)
def cfg6(mults=(24, 40, 40, 32, 24, 12, 6)):
    """Single-site effective Hamiltonian A' = FL . A . O . FR (Alg. 11) with the paper's
    spin-1 Heisenberg spaces P = (1), W = 2 (0) + (1), V = sum_i d_i (i + 1/2).
    The d_i live in an external benchmark repo (absent here): the cfg5 multiplicities are reused,
    shifted to half-integer spins 1/2 .. 13/2 (dim V = sum d_i (2i + 2) = 1172)."""
    P = space("SU2", [((2,), 1)])
    V = space("SU2", [((2 * j + 1,), m) for j, m in enumerate(mults)])
    W = space("SU2", [((0,), 2), ((2,), 1)])
    FL = {"cod": [V], "dom": [V, W]}                 # (alpha'; alpha, a)
    A = {"cod": [V, P], "dom": [V]}                  # (alpha, s; beta)
    O = {"cod": [W, P], "dom": [P, W]}               # (a, s'; s, b)
    FR = {"cod": [W, dual(V)], "dom": [dual(V)]}     # (b, beta'; beta)
    al_, al, a, s, be, sp, b, bep = range(1, 9)
    return {
        "cfg": 6, "kind": "SU2", "dtype": "f64",
        "tensors": {"FL": (FL, 0), "A": (A, 1), "O": (O, 2), "FR": (FR, 3)},
        "steps": [
            ("FL", [al_, al, a], "A", [al, s, be], "T1", [al_, a, s, be], 2),
            ("T1", [al_, a, s, be], "O", [a, sp, s, b], "T2", [al_, sp, be, b], 2),
            ("T2", [al_, sp, be, b], "FR", [b, bep, be], "out", [al_, sp, bep], 2),
        ],
    }


# ------------------------- config 7 (non-abelian fermionic Hubbard, fZ2 x U1 x SU2)
def _u1su2_bond(n_mult, sigma_n=2.5, sigma_j=1.5):
    """Multiplets (N, 2j) with N = -6..6, 2j = 0..6 and N = 2j (mod 2) (the sectors a Hubbard chain
    reaches from the physical space), multiplicities ~ exp(-N^2/2s_N^2 - j^2/2s_j^2) by reading C15."""
    labels = [(n, tj) for n in range(-6, 7) for tj in range(0, 7) if (n - tj) % 2 == 0]
    weights = [math.exp(-n * n / (2 * sigma_n ** 2) - (tj / 2) ** 2 / (2 * sigma_j ** 2)) for n, tj in labels]
    return gaussian_degeneracies(labels, weights, n_mult, lambda l: abs(l[0]) + l[1])


def cfg7(n_mult=700):
    """Hubbard two-site update with fZ2 x U1 x SU2, the cfg3 chain with the spin promoted
    to SU(2): P = (0,0) + (1,1/2) + (2,0) (dim 4); W = 2 (0,0) + 2 (1,1/2) + 2 (-1,1/2) (dim 10: the
    cfg3 channels of reading C18 grouped into doublets); V: 700 multiplets, dim 2058 (~ cfg3's 2048)."""
    P = space("fU1xSU2", [((0, 0), 1), ((1, 1), 1), ((2, 0), 1)])
    W = space("fU1xSU2", [((0, 0), 2), ((1, 1), 2), ((-1, 1), 2)])
    V = space("fU1xSU2", _u1su2_bond(n_mult))
    return _dmrg_chain(7, "fU1xSU2", P, W, V)


# ----------------------- config 8 (Hubbard at half filling, fZ2 x SU2 x SU2)
def _su2su2_bond(n_mult, sigma_c=1.2, sigma_s=1.5):
    """Multiplets (2jc, 2js), 0..6 each, with jc + js integer (bonds cut after an even number of sites),
    multiplicities ~ exp(-jc^2/2s_c^2 - js^2/2s_s^2) by reading C15."""
    labels = [(c, t) for c in range(0, 7) for t in range(0, 7) if (c + t) % 2 == 0]
    weights = [math.exp(-(c / 2) ** 2 / (2 * sigma_c ** 2) - (t / 2) ** 2 / (2 * sigma_s ** 2)) for c, t in labels]
    return gaussian_degeneracies(labels, weights, n_mult, lambda l: l[0] + l[1])


def cfg8(n_mult=270):
    """Hubbard two-site update at half filling with fZ2 x SU2(charge) x SU2(spin): the cfg3
    chain with P = (1/2, 0) + (0, 1/2) (charge doublet: empty/double; spin doublet: single, odd),
    W = 2 (0,0) + 2 (1/2,1/2) (the D = 10 channels: identity and the four single-fermion operators as
    one SO(4) vector, odd), V: 270 multiplets (dim ~ 2000, as cfg3)."""
    P = space("fSU2xSU2", [((1, 0), 1), ((0, 1), 1)])
    W = space("fSU2xSU2", [((0, 0), 2), ((1, 1), 2)])
    V = space("fSU2xSU2", _su2su2_bond(n_mult))
    return _dmrg_chain(8, "fSU2xSU2", P, W, V)


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5, 6: cfg6, 7: cfg7, 8: cfg8}


def chain_as_ncon(cfg):
    """The chain of a config as ONE ncon network (tk_ncon): (tensor names, labels per tensor, order,
    n_cod_out, output name). Labels contracted along the chain stay positive; the final output's legs
    become -1..-m in its label order; `order` lists each step's contracted labels, step by step, so the
    network is contracted in the chain's own pairwise order. Pure relabelling, no arithmetic."""
    steps = cfg["steps"]
    inputs = list(cfg["tensors"])
    lab = {}
    for (na, la, nb, lb, nc, lc, ncod) in steps:
        for name, l in ((na, la), (nb, lb)):
            if name in cfg["tensors"]:
                lab[name] = list(l)
    na, la, nb, lb, out_name, lout, n_cod_out = steps[-1]
    open_map = {x: -(i + 1) for i, x in enumerate(lout)}
    labels = [[open_map.get(x, x) for x in lab[name]] for name in inputs]
    order = []
    for (na, la, nb, lb, nc, lc, ncod) in steps:
        order += [x for x in la if x in lb and x not in order]
    return inputs, labels, order, n_cod_out, out_name
