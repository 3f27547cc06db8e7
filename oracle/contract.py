"""Dense contraction -- the plain definition (oracle side; test infrastructure).

Bosonic sectors (Z2, U1, U1xU1, SU2): a dense einsum over leg labels in float64
(composition = matmul P:591-609; pairwise contraction Alg. 4 P:634-647 reduces,
without symmetry structure, to a plain index contraction -- P:384-386).

Fermionic sectors (fZ2, fU1xU1): a dense Alg. 4 in the fixed pairwise order:
permute each operand to (open ; contracted) with the per-element Koszul sign of
reading C13, reshape, matmul, reshape, permute the result with the same rule.

Reading C13 (sign of a permute with tuples (p, q) of a rank-(N1, N2) tensor):
    S = (1, ..., N1, N1+N2, ..., N1+1),   T = (p_1, ..., p_N1', q_N2', ..., q_1)
    sign = prod over leg pairs (x, y) whose relative order differs between S and T
           of (-1)^{pi_x pi_y}
where pi_x is the fermion parity of the sector of leg x's index. Compose carries
no sign. (Bends are sign-free in the unitary convention.)

Reading C2 (labels -> tuples): A~ = (open A in A order ; contracted in A order),
B~ = (same contracted order ; open B in B order), C~ = (open A ; open B), then
permute C~ to labC.
"""
import numpy as np

from . import sectors
from .dense import parity_vector


def permuted_spaces(cod, dom, p, q):
    """Space selection rule of Alg. 2: V'_i = p_i-th of (V_1.., W_1*..),
    W'_j = q_j-th of (V_1*.., W_1..). Indices are 0-based."""
    def flip(sp):
        return {"kind": sp["kind"], "sectors": sp["sectors"], "dual": not sp["dual"]}
    as_cod = list(cod) + [flip(w) for w in dom]
    as_dom = [flip(v) for v in cod] + list(dom)
    return [as_cod[i] for i in p], [as_dom[j] for j in q]


def tuples_from_labels(labA, labB, labC, n_cod_C):
    """Reading C2. Returns (pA, qA, pB, qB, pAB, qAB), 0-based."""
    labA, labB, labC = list(labA), list(labB), list(labC)
    con = [l for l in labA if l in labB]
    openA = [l for l in labA if l not in labB]
    openB = [l for l in labB if l not in labA]
    pA = [labA.index(l) for l in openA]
    qA = [labA.index(l) for l in con]
    pB = [labB.index(l) for l in con]
    qB = [labB.index(l) for l in openB]
    ct = openA + openB
    pAB = [ct.index(l) for l in labC[:n_cod_C]]
    qAB = [ct.index(l) for l in labC[n_cod_C:]]
    return pA, qA, pB, qB, pAB, qAB


def output_spaces(A_cod, A_dom, B_cod, B_dom, labA, labB, labC, n_cod_C):
    pA, qA, pB, qB, pAB, qAB = tuples_from_labels(labA, labB, labC, n_cod_C)
    At_cod, _ = permuted_spaces(A_cod, A_dom, pA, qA)
    _, Bt_dom = permuted_spaces(B_cod, B_dom, pB, qB)
    return permuted_spaces(At_cod, Bt_dom, pAB, qAB)


def koszul_sign_pairs(n1, n2, p, q):
    """Leg pairs (x, y) whose relative order differs between S and T (reading C13)."""
    N = n1 + n2
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    T = list(p) + list(reversed(q))
    ps = {leg: i for i, leg in enumerate(S)}
    pt = {leg: i for i, leg in enumerate(T)}
    pairs = []
    for x in range(N):
        for y in range(x + 1, N):
            if (ps[x] < ps[y]) != (pt[x] < pt[y]):
                pairs.append((x, y))
    return pairs


def permute_dense(D, parities, n1, p, q):
    """Dense permute with the Koszul sign of reading C13.

    D has legs (cod..., dom...) in the tensor's order; `parities[k]` is the
    parity vector of leg k (all zeros for bosons). Returns the array with legs
    ordered (p..., q...).
    """
    N = D.ndim
    order = list(p) + list(q)
    out = np.transpose(D, order).copy()
    pos = {leg: i for i, leg in enumerate(order)}
    for x, y in koszul_sign_pairs(n1, N - n1, p, q):
        px, py = parities[x], parities[y]
        if not (px.any() and py.any()):
            continue
        shape_x = [1] * N
        shape_x[pos[x]] = px.size
        shape_y = [1] * N
        shape_y[pos[y]] = py.size
        odd = px.reshape(shape_x) * py.reshape(shape_y)
        out *= 1 - 2 * (odd % 2)
    return out


_LETTERS = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"


def contract_einsum(A, labA, B, labB, labC):
    """Bosonic plain definition: C[labC] = sum over shared labels A[labA] B[labB]."""
    m = {}
    for l in list(labA) + list(labB):
        if l not in m:
            m[l] = _LETTERS[len(m)]
    spec = "".join(m[l] for l in labA) + "," + "".join(m[l] for l in labB) + "->" + "".join(m[l] for l in labC)
    return np.einsum(spec, A, B, optimize=True)


def contract_alg4(A, A_spaces, nA, labA, B, B_spaces, nB, labB, labC, n_cod_C):
    """Dense Alg. 4 (Alg. 8 P:1276-1300 with reading C1: B uses (p^B, q^B)).

    A_spaces / B_spaces: the leg spaces in (cod..., dom...) order; nA, nB the codomain counts.
    """
    pA, qA, pB, qB, pAB, qAB = tuples_from_labels(labA, labB, labC, n_cod_C)
    return contract_alg4_tuples(A, A_spaces, nA, B, B_spaces, nB, pA, qA, pB, qB, pAB, qAB)


def contract_alg4_tuples(A, A_spaces, nA, B, B_spaces, nB, pA, qA, pB, qB, pAB, qAB):
    """Dense Alg. 4 with explicit tuples: A~ = permute(A, (pA, qA)), B~ = permute(B, (pB, qB))
    (reading C1), C~ = A~ o B~ (a matmul over the qA / pB legs), C = permute(C~, (pAB, qAB)).
    Permutes carry the Koszul sign of reading C13 (+1 for bosonic kinds)."""
    parA = [parity_vector(sp) for sp in A_spaces]
    parB = [parity_vector(sp) for sp in B_spaces]
    At = permute_dense(A, parA, nA, pA, qA)
    Bt = permute_dense(B, parB, nB, pB, qB)
    m = int(np.prod([A.shape[i] for i in pA], dtype=np.int64))
    k = int(np.prod([A.shape[i] for i in qA], dtype=np.int64))
    n = int(np.prod([B.shape[j] for j in qB], dtype=np.int64))
    Ct = (At.reshape(m, k) @ Bt.reshape(k, n)).reshape([A.shape[i] for i in pA] + [B.shape[j] for j in qB])
    parC = [parA[i] for i in pA] + [parB[j] for j in qB]
    return permute_dense(Ct, parC, len(pA), pAB, qAB)


def contract(kind, A, A_spaces, nA, labA, B, B_spaces, nB, labB, labC, n_cod_C):
    """The oracle's contraction: einsum for bosons, dense Alg. 4 with signs for fermions."""
    if sectors.is_fermionic(kind):
        return contract_alg4(A, A_spaces, nA, labA, B, B_spaces, nB, labB, labC, n_cod_C)
    return contract_einsum(A, labA, B, labB, labC)


def rel_frobenius(X, Y):
    """||X - Y||_F / ||Y||_F."""
    ny = np.linalg.norm(Y.ravel())
    return float(np.linalg.norm((X - Y).ravel()) / (ny if ny > 0 else 1.0))


def partial_trace_dense(D, cod, dom, pt, qt, p, q):
    """Plain partial trace (Alg. 3) of a dense bosonic tensor: legs pt[i] and qt[i] carry the
    same dense index set (ket/bra pair) and are summed with a delta (the evaluation map),
    then the remaining legs are arranged as (p..., q...). Returns (dense result, C cod, C dom)."""
    N = D.ndim
    letters = [_LETTERS[i] for i in range(N)]
    for a, b in zip(pt, qt):
        letters[b] = letters[a]
    out = "".join(letters[i] for i in list(p) + list(q))
    R = np.einsum("".join(letters) + "->" + out, D)
    c2, d2 = permuted_spaces(cod, dom, p, q)
    return R, c2, d2
