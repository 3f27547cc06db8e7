"""Sector algebra for the kinds the configs use (oracle side; test infrastructure).

Labels are tuples of ints:
  Z2      (g,)      g in {0,1}; fusion = xor
  fZ2     (g,)      fermion parity (SVect) g in {0,1}
  U1      (q,)      fusion = addition, dual = negation
  U1xU1   (N, 2Sz)  Deligne product of two U1, componentwise
  fU1xU1  (N, 2Sz)  as U1xU1 with fermion parity N mod 2 (BASELINE cfg3, reading C14)
  SU2     (2j,)     N^{j1 j2}_{j3} = 1 iff |j1-j2| <= j3 <= j1+j2 (and integrality), d = 2j+1
                    P:2303-2312
  fU1xSU2 (N, 2j)   Hubbard fZ2 x U1 x SU2 as a Deligne product:
                    charges add, spins by the SU2 rule, d = 2j+1, fermion parity N mod 2 (reading C14)
  fSU2xSU2 (2jc, 2js) Hubbard at half filling, fZ2 x SU2(charge) x SU2(spin): both
                    factors by the SU2 rule, d = (2jc+1)(2js+1), fermion parity 2js mod 2
  Fib     (0|1,)    {I, tau}: tau x tau = I + tau, d_tau = golden ratio
  Ising   (0|1|2,)  {I, sigma, psi}: sigma x sigma = I + psi, sigma x psi = sigma, psi x psi = I,
                    d_sigma = sqrt 2. No dense embedding (planar oracle: oracle/planar.py)
"""
import math

KINDS = ("Z2", "fZ2", "U1", "U1xU1", "fU1xU1", "SU2", "fU1xSU2", "fSU2xSU2", "Fib", "Ising")
GOLDEN = (1 + math.sqrt(5)) / 2


def width(kind):
    return 2 if kind in ("U1xU1", "fU1xU1", "fU1xSU2", "fSU2xSU2") else 1


def spins2(kind, a):
    """Doubled spins of the SU(2) factors of a label, in factor order ([] for abelian kinds)."""
    if kind == "SU2":
        return [a[0]]
    if kind == "fU1xSU2":
        return [a[1]]
    if kind == "fSU2xSU2":
        return [a[0], a[1]]
    return []


def spin2(kind, a):
    """Doubled spin of the single SU(2) factor (0 for kinds without one)."""
    js = spins2(kind, a)
    return js[0] if js else 0


def unit(kind):
    return (0, 0) if width(kind) == 2 else (0,)


def dual(kind, a):
    if kind in ("Z2", "fZ2", "SU2", "fSU2xSU2", "Fib", "Ising"):
        return tuple(a)  # self-dual (SU2: "all irreps are self-dual")
    if kind == "fU1xSU2":
        return (-a[0], a[1])  # Deligne product: componentwise duals
    return tuple(-x for x in a)


def fuse(kind, a, b):
    """All c with N^{ab}_c = 1, ascending (multiplicity-free for every kind here)."""
    if kind in ("Z2", "fZ2"):
        return [((a[0] + b[0]) % 2,)]
    if kind == "U1":
        return [(a[0] + b[0],)]
    if kind in ("U1xU1", "fU1xU1"):
        return [(a[0] + b[0], a[1] + b[1])]
    if kind == "SU2":
        lo, hi = abs(a[0] - b[0]), a[0] + b[0]
        return [(j,) for j in range(lo, hi + 1, 2)]
    if kind == "fU1xSU2":
        lo, hi = abs(a[1] - b[1]), a[1] + b[1]
        return [(a[0] + b[0], j) for j in range(lo, hi + 1, 2)]
    if kind == "fSU2xSU2":
        return [(jc, js) for jc in range(abs(a[0] - b[0]), a[0] + b[0] + 1, 2)
                for js in range(abs(a[1] - b[1]), a[1] + b[1] + 1, 2)]
    if kind == "Fib":
        if a[0] == 0:
            return [tuple(b)]
        if b[0] == 0:
            return [tuple(a)]
        return [(0,), (1,)]
    if kind == "Ising":
        x, y = a[0], b[0]
        if x == 0:
            return [tuple(b)]
        if y == 0:
            return [tuple(a)]
        if x == 1 and y == 1:
            return [(0,), (2,)]
        if x == 2 and y == 2:
            return [(0,)]
        return [(1,)]
    raise ValueError(kind)


def qdim(kind, a):
    if kind == "Fib":
        return GOLDEN if a[0] == 1 else 1.0
    if kind == "Ising":
        return math.sqrt(2.0) if a[0] == 1 else 1.0
    d = 1
    for j in spins2(kind, a):
        d *= j + 1
    return d


def parity(kind, a):
    """Fermion parity (0 for bosonic kinds). fU1xU1: N mod 2 (BASELINE cfg3)."""
    if kind == "fZ2":
        return a[0] % 2
    if kind in ("fU1xU1", "fU1xSU2"):
        return a[0] % 2
    if kind == "fSU2xSU2":
        return a[1] % 2
    return 0


def is_fermionic(kind):
    return kind in ("fZ2", "fU1xU1", "fU1xSU2", "fSU2xSU2")


def is_abelian(kind):
    return kind not in ("SU2", "fU1xSU2", "fSU2xSU2", "Fib", "Ising")
