"""Randomised parity sweep of tk_contract against the oracle -- needs a B200.

Seeded random contractions over every sector kind of the configs: random leg spaces, ranks 2-4,
codomain/domain splits, dual flags, one or two contracted legs, output leg order and split, alpha /
beta. Small dense sizes, so each case is checked against the plain definition (dense embedding +
einsum; fermions through the dense Alg. 4 with reading C2 / C13). The cases run whichever kernel
paths the planner picks for them (seg, recoupling, gathered, small / skinny GEMMs, split-K).
"""
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import layout as OL, dense as OD, contract as OC  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12
SECTORS = {
    "Z2": [(0,), (1,)],
    "fZ2": [(0,), (1,)],
    "U1": [(-2,), (-1,), (0,), (1,), (2,)],
    "U1xU1": [(0, 0), (1, 1), (1, -1), (-1, 1), (-1, -1), (2, 0)],
    "fU1xU1": [(0, 0), (1, 1), (1, -1), (-1, 1), (-1, -1), (2, 0)],
    "SU2": [(0,), (1,), (2,)],
    "fU1xSU2": [(0, 0), (1, 1), (-1, 1), (2, 0), (0, 2)],
    "fSU2xSU2": [(0, 0), (1, 1), (0, 2), (2, 0), (1, 0), (0, 1)],
}


def _space(rng, kind):
    labs = SECTORS[kind]
    pick = sorted(rng.choice(len(labs), size=int(rng.integers(2, min(4, len(labs)) + 1)), replace=False))
    return W.space(kind, [(labs[i], int(rng.integers(1, 4))) for i in pick])


def _case(rng, kind):
    """Random A, B (as HomSpace specs), labels, output order; B's contracted legs mirror A's."""
    NA = int(rng.integers(2, 5))
    legsA = [(_space(rng, kind), bool(rng.integers(0, 2))) for _ in range(NA)]  # (space, dual)
    nA = int(rng.integers(1, NA))                                               # A codomain count
    nc = int(rng.integers(1, min(2, NA) + 1))                                   # contracted legs
    cA = sorted(rng.choice(NA, size=nc, replace=False))
    NBo = int(rng.integers(0, 3))                                               # open legs of B
    # B legs: contracted mirrors (same space, opposite side) + open legs
    bcod, bdom, labB_cod, labB_dom = [], [], [], []
    labA = list(range(1, NA + 1))
    for i in cA:
        sp, du = legsA[i]
        S = W.dual(sp) if du else sp
        if i < nA:            # A codomain leg -> B domain leg of the same space
            bdom.append(S)
            labB_dom.append(labA[i])
        else:                 # A domain leg -> B codomain leg of the same space
            bcod.append(S)
            labB_cod.append(labA[i])
    for j in range(NBo):
        sp = _space(rng, kind)
        S = W.dual(sp) if rng.integers(0, 2) else sp
        lab = 100 + j
        if rng.integers(0, 2):
            bcod.append(S)
            labB_cod.append(lab)
        else:
            bdom.append(S)
            labB_dom.append(lab)
    Aspec = {"cod": [(W.dual(s) if d else s) for s, d in legsA[:nA]],
             "dom": [(W.dual(s) if d else s) for s, d in legsA[nA:]]}
    Bspec = {"cod": bcod, "dom": bdom}
    labB = labB_cod + labB_dom
    open_ = [l for i, l in enumerate(labA) if i not in cA] + [l for l in labB if l >= 100]
    labC = [open_[i] for i in rng.permutation(len(open_))]
    ncod = int(rng.integers(0, len(labC) + 1))
    return Aspec, labA, Bspec, labB, labC, ncod


@pytest.mark.parametrize("kind,cplx", [(k, False) for k in SECTORS] + [(k, True) for k in ("U1", "fU1xU1", "SU2",
                                                                                          "fSU2xSU2")])
def test_random_contractions_vs_oracle(kind, cplx):
    from paper_2508_10076_b200 import tk
    rng = np.random.default_rng(zlib.crc32((kind + str(cplx)).encode()))  # stable across processes
    done = 0
    for trial in range(150):
        Aspec, labA, Bspec, labB, labC, ncod = _case(rng, kind)
        la = OL.homspace_layout(kind, Aspec["cod"], Aspec["dom"])
        lb = OL.homspace_layout(kind, Bspec["cod"], Bspec["dom"])
        if la.nelems == 0 or lb.nelems == 0:
            continue
        try:
            cod, dom = OC.output_spaces(Aspec["cod"], Aspec["dom"], Bspec["cod"], Bspec["dom"], labA, labB, labC, ncod)
        except Exception:
            continue
        lc = OL.homspace_layout(kind, cod, dom)
        if max(int(np.prod(OD.dense_shape(la))), int(np.prod(OD.dense_shape(lb))),
               int(np.prod(OD.dense_shape(lc)))) > 200000:
            continue
        def draw(n):
            x = rng.standard_normal(n)
            return x + 1j * rng.standard_normal(n) if cplx else x
        xa, xb, y0 = draw(la.nelems), draw(lb.nelems), draw(lc.nelems)
        alpha, beta = float(rng.choice([1.0, -0.5, 2.0])), float(rng.choice([0.0, 0.0, 0.75]))
        conjA, conjB = (bool(rng.integers(0, 2)), bool(rng.integers(0, 2))) if cplx else (False, False)
        dt, tdt = (tk.TK_C64, torch.complex128) if cplx else (tk.TK_F64, torch.float64)
        A, B = tk.tensor_from_spec(Aspec, dt), tk.tensor_from_spec(Bspec, dt)
        C = tk.tk_contract_output(A, labA, B, labB, labC, ncod)
        assert C.nelems == lc.nelems
        a, b = torch.from_numpy(xa).to(tdt).cuda(), torch.from_numpy(xb).to(tdt).cuda()
        c = torch.from_numpy(y0.copy()).to(tdt).cuda() if beta != 0 else torch.full((lc.nelems,), float("nan"),
                                                                                     dtype=tdt, device="cuda")
        nws = tk.tk_contract_workspace(A, labA, B, labB, C, labC)
        ws = torch.empty(max(nws // 8 + 32, 1), dtype=torch.float64, device="cuda")
        tk.tk_contract(A, a, labA, B, b, labB, C, c, labC, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8,
                       conjA=conjA, conjB=conjB)
        torch.cuda.synchronize()
        DA, DB = OD.to_dense(la, xa), OD.to_dense(lb, xb)
        DA, DB = (np.conj(DA) if conjA else DA), (np.conj(DB) if conjB else DB)
        D = OC.contract(kind, DA, Aspec["cod"] + Aspec["dom"], len(Aspec["cod"]), labA,
                        DB, Bspec["cod"] + Bspec["dom"], len(Bspec["cod"]), labB, labC, ncod)
        want = alpha * D + (beta * OD.to_dense(lc, y0) if beta != 0 else 0.0)
        got = OD.to_dense(lc, c.cpu().numpy())
        # symmetry can force the result to vanish (e.g. an output space without the unit sector): then
        # the dense oracle returns rounding noise ~1e-16 |A||B| and the comparison is absolute
        scale = np.linalg.norm(DA.ravel()) * np.linalg.norm(DB.ravel()) * abs(alpha) + abs(beta) * np.linalg.norm(y0)
        if np.linalg.norm(want.ravel()) <= 1e-13 * scale:
            assert np.linalg.norm(got.ravel()) <= 1e-13 * scale, (trial, labA, labB, labC, ncod)
        else:
            err = OC.rel_frobenius(got, want)
            assert err <= TOL, (trial, Aspec, labA, Bspec, labB, labC, ncod, err)
        done += 1
    assert done >= 50


@pytest.mark.parametrize("kind", list(SECTORS))
def test_random_tuples_vs_oracle(kind):
    """tk_contract_tuples with random explicit Alg. 4 tuples (any order of pA / qB / the contracted pairs,
    any split of C~'s legs) against the oracle's dense Alg. 4 with the same tuples."""
    from paper_2508_10076_b200 import tk
    rng = np.random.default_rng(zlib.crc32(("tuples" + kind).encode()))
    done = 0
    for trial in range(100):
        Aspec, labA, Bspec, labB, labC, ncod = _case(rng, kind)
        la = OL.homspace_layout(kind, Aspec["cod"], Aspec["dom"])
        lb = OL.homspace_layout(kind, Bspec["cod"], Bspec["dom"])
        if la.nelems == 0 or lb.nelems == 0:
            continue
        # tuples: contracted pairs from the labels, then everything shuffled
        pairs = [(i, labB.index(l)) for i, l in enumerate(labA) if l in labB]
        pairs = [pairs[k] for k in rng.permutation(len(pairs))]
        qA, pB = [p[0] for p in pairs], [p[1] for p in pairs]
        pA = [i for i in range(len(labA)) if i not in qA]
        pA = [pA[k] for k in rng.permutation(len(pA))]
        qB = [j for j in range(len(labB)) if j not in pB]
        qB = [qB[k] for k in rng.permutation(len(qB))]
        n = len(pA) + len(qB)
        perm = [int(x) for x in rng.permutation(n)]
        k = int(rng.integers(0, n + 1))
        pAB, qAB = perm[:k], perm[k:]
        Asp, Bsp = Aspec["cod"] + Aspec["dom"], Bspec["cod"] + Bspec["dom"]
        # C~ = (A~ codomain ; B~ domain), each by the selection rule of Alg. 2
        at_cod, _ = OC.permuted_spaces(Aspec["cod"], Aspec["dom"], pA, qA)
        _, bt_dom = OC.permuted_spaces(Bspec["cod"], Bspec["dom"], pB, qB)
        cod, dom = OC.permuted_spaces(at_cod, bt_dom, pAB, qAB)
        lc = OL.homspace_layout(kind, cod, dom)
        if max(int(np.prod(OD.dense_shape(la))), int(np.prod(OD.dense_shape(lb))),
               int(np.prod(OD.dense_shape(lc)))) > 200000:
            continue
        xa, xb = rng.standard_normal(la.nelems), rng.standard_normal(lb.nelems)
        A, B = tk.tensor_from_spec(Aspec), tk.tensor_from_spec(Bspec)
        C = tk.tk_contract_tuples_output(A, pA, qA, B, pB, qB, pAB, qAB)
        assert C.nelems == lc.nelems
        c = torch.full((lc.nelems,), float("nan"), dtype=torch.float64, device="cuda")
        nws = tk.tk_contract_tuples_workspace(A, pA, qA, B, pB, qB, C, pAB, qAB)
        ws = torch.empty(max(nws // 8 + 32, 1), dtype=torch.float64, device="cuda")
        tk.tk_contract_tuples(A, torch.from_numpy(xa).cuda(), pA, qA, B, torch.from_numpy(xb).cuda(), pB, qB, C, c,
                              pAB, qAB, ws=ws, ws_bytes=ws.numel() * 8)
        torch.cuda.synchronize()
        DA, DB = OD.to_dense(la, xa), OD.to_dense(lb, xb)
        want = OC.contract_alg4_tuples(DA, Asp, len(Aspec["cod"]), DB, Bsp, len(Bspec["cod"]), pA, qA, pB, qB,
                                       pAB, qAB)
        got = OD.to_dense(lc, c.cpu().numpy())
        scale = np.linalg.norm(DA.ravel()) * np.linalg.norm(DB.ravel())
        if np.linalg.norm(want.ravel()) <= 1e-13 * scale:
            assert np.linalg.norm(got.ravel()) <= 1e-13 * scale, trial
        else:
            assert OC.rel_frobenius(got, want) <= TOL, (trial, pA, qA, pB, qB, pAB, qAB)
        done += 1
    assert done >= 30
