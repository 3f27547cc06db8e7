"""tk_ncon (network contraction) against the oracle -- needs a B200.

The oracle side replays the network pair by pair exactly as include/tk.h specifies (each step
contracts the two tensors holding the next label of `order` over all labels they share -- a left fold:
the running intermediate is the left operand A, two inputs in list order; the last step into -1, -2,
...), with the dense oracle contraction for every step; for bosonic kinds it is also checked against one
einsum over the whole network. (The library may store intermediates in any leg order: that changes no
value, so the replay keeps them (open A ; open B).)
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import layout as OL, dense as OD, contract as OC, sectors as OS  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12


def oracle_ncon(kind, specs, denses, labels, order, n_cod_out):
    items = []
    for s, D, l in zip(specs, denses, labels):
        l = list(l)
        rep = [x for x in set(l) if l.count(x) == 2]
        if rep:  # partial trace first (Alg. 3), remaining legs keep their side and order
            N1 = len(s["cod"])
            legs = s["cod"] + s["dom"]
            pt, qt = [], []
            for x in rep:
                i, j = [k for k, y in enumerate(l) if y == x]
                ket_i = not (legs[i]["dual"] ^ (i >= N1))
                pt.append(i if ket_i else j)
                qt.append(j if ket_i else i)
            keep = [k for k in range(len(l)) if l[k] not in rep]
            p = [k for k in keep if k < N1]
            q = [k for k in keep if k >= N1]
            D, c2, d2 = OC.partial_trace_dense(D, s["cod"], s["dom"], pt, qt, p, q)
            s = {"cod": c2, "dom": d2}
            l = [l[k] for k in p + q]
        items.append((s["cod"], s["dom"], D, l))
    alive = [True] * len(items)
    m = sum(1 for l in labels for x in l if x < 0)

    def pair(a, b):
        Ac, Ad, A, la = items[a]
        Bc, Bd, B, lb = items[b]
        oa = [x for x in la if x not in lb]
        ob = [x for x in lb if x not in la]
        last = sum(alive) == 2
        lc, nc = ([-k for k in range(1, m + 1)], n_cod_out) if last else (oa + ob, len(oa))
        D = OC.contract(kind, A, Ac + Ad, len(Ac), la, B, Bc + Bd, len(Bc), lb, lc, nc)
        cod, dom = OC.output_spaces(Ac, Ad, Bc, Bd, la, lb, lc, nc)
        alive[a] = alive[b] = False
        items.append((cod, dom, D, lc))
        alive.append(True)

    n_in = len(items)
    for x in order:
        hold = [i for i, it in enumerate(items) if alive[i] and x in it[3]]
        if hold:
            a, b = hold[0], hold[1]
            if b >= n_in and a < n_in:  # left fold: the intermediate is A
                a, b = b, a
            pair(a, b)
    while sum(alive) > 1:
        al = [i for i in range(len(items)) if alive[i]]
        pair(al[0], al[1])
    cod, dom, D, _ = items[-1]
    return cod, dom, D


def _network_cfg2(chi=64):
    cfg = W.cfg2(chi=chi)
    t = {k: v[0] for k, v in cfg["tensors"].items()}
    # L(a', a, w) th(a, s1, s2, b) W1(w, s1', s1, w2) W2(w2, s2', s2, w3) R(w3, b', b): the DMRG H.theta
    specs = [t["L"], t["theta"], t["W1"], t["W2"], t["R"]]
    labels = [[-1, 1, 2], [1, 3, 4, 5], [2, -2, 3, 6], [6, -3, 4, 7], [7, -4, 5]]
    return "U1", specs, labels, [1, 2, 3, 6, 4, 5, 7], 3


def _network_cfg3(chi=96):
    cfg = W.cfg3(chi=chi)
    t = {k: v[0] for k, v in cfg["tensors"].items()}
    specs = [t["L"], t["theta"], t["W1"], t["W2"], t["R"]]
    labels = [[-1, 1, 2], [1, 3, 4, 5], [2, -2, 3, 6], [6, -3, 4, 7], [7, -4, 5]]
    return "fU1xU1", specs, labels, [1, 2, 3, 6, 4, 5, 7], 3


def _network_su2():
    V = W.space("SU2", [((0,), 3), ((1,), 2), ((2,), 2)])
    A = {"cod": [V, V], "dom": [V]}
    B = {"cod": [V], "dom": [V, V]}
    M = {"cod": [V], "dom": [V]}
    # A[-1, 1, 2] B[2, -2, 3] M[3, 1]: a ring with two open legs; and a disconnected piece M2[-3, -4]
    return "SU2", [A, B, M, M], [[-1, 1, 2], [2, -2, 3], [3, 1], [-3, -4]], [2, 3, 1], 2


def _network_trace():
    V = W.space("U1", [((-1,), 2), ((0,), 3), ((1,), 2)])
    A = {"cod": [V, V], "dom": [V, V]}
    B = {"cod": [V], "dom": [V, V]}
    # A[-1, 1, 2, 1] traces its legs 1 and 3, then meets B[2, -2, -3]
    return "U1", [A, B], [[-1, 1, 2, 1], [2, -2, -3]], [1, 2], 1


@pytest.mark.parametrize("maker", [_network_cfg2, _network_cfg3, _network_su2, _network_trace],
                         ids=["cfg2", "cfg3", "su2", "trace"])
def test_ncon_vs_oracle(maker):
    from paper_2508_10076_b200 import tk
    kind, specs, labels, order, n_cod_out = maker()
    rng = np.random.default_rng(7)
    lays = [OL.homspace_layout(kind, s["cod"], s["dom"]) for s in specs]
    xs = [rng.standard_normal(l.nelems) for l in lays]
    T = [tk.tensor_from_spec(s) for s in specs]
    C = tk.tk_ncon_output(T, labels, order, n_cod_out)
    cod, dom, D = oracle_ncon(kind, specs, [OD.to_dense(l, x) for l, x in zip(lays, xs)], labels, order, n_cod_out)
    lc = OL.homspace_layout(kind, cod, dom)
    assert C.nelems == lc.nelems
    y0 = rng.standard_normal(lc.nelems)
    c = torch.from_numpy(y0.copy()).cuda()
    nws = tk.tk_ncon_workspace(T, labels, order, n_cod_out)
    ws = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
    tk.tk_ncon(T, [torch.from_numpy(x).cuda() for x in xs], labels, order, n_cod_out, C, c, alpha=-0.5, beta=0.25,
               ws=ws, ws_bytes=ws.numel() * 8)
    torch.cuda.synchronize()
    want = -0.5 * D + 0.25 * OD.to_dense(lc, y0)
    assert OC.rel_frobenius(OD.to_dense(lc, c.cpu().numpy()), want) <= TOL
    if not OS.is_fermionic(kind):  # bosonic: the whole network is one einsum (ncon semantics)
        letters = {}
        def L(x):
            return letters.setdefault(x, "abcdefghijklmnopqrstuvwxyz"[len(letters)])
        dens = [OD.to_dense(l, x) for l, x in zip(lays, xs)]
        m = sum(1 for l in labels for x in l if x < 0)
        spec = ",".join("".join(L(x) for x in l) for l in labels) + "->" + "".join(L(-k) for k in range(1, m + 1))
        E = np.einsum(spec, *dens, optimize=True)
        assert OC.rel_frobenius(-0.5 * E + 0.25 * OD.to_dense(lc, y0), want) <= 1e-12


@pytest.mark.parametrize("maker", [_network_cfg3, _network_su2], ids=["cfg3", "su2"])
def test_ncon_cached_plan_serves_new_tensor_objects(maker):
    """A planned network is memoised by structure: a second call with FRESH tensor objects (the first ones
    released) and other data reuses the plan -- its input slots are filled from the current call, the
    intermediates are the plan's own -- and still matches the oracle."""
    import gc
    from paper_2508_10076_b200 import tk
    kind, specs, labels, order, n_cod_out = maker()
    lays = [OL.homspace_layout(kind, s["cod"], s["dom"]) for s in specs]
    tk.tk_cache_clear()
    for seed in (11, 12):
        rng = np.random.default_rng(seed)
        xs = [rng.standard_normal(l.nelems) for l in lays]
        T = [tk.tensor_from_spec(s) for s in specs]          # new host objects every round
        C = tk.tk_ncon_output(T, labels, order, n_cod_out)
        n_plans = tk.tk_cache_size()
        nws = tk.tk_ncon_workspace(T, labels, order, n_cod_out)
        assert tk.tk_cache_size() == n_plans                  # output and workspace: one plan
        ws = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
        c = torch.full((C.nelems,), float("nan"), dtype=torch.float64, device="cuda")
        tk.tk_ncon(T, [torch.from_numpy(x).cuda() for x in xs], labels, order, n_cod_out, C, c, ws=ws,
                   ws_bytes=ws.numel() * 8)
        torch.cuda.synchronize()
        if seed == 11:
            after_first = tk.tk_cache_size()
        else:
            assert tk.tk_cache_size() == after_first          # nothing new was planned
        cod, dom, D = oracle_ncon(kind, specs, [OD.to_dense(l, x) for l, x in zip(lays, xs)], labels, order,
                                  n_cod_out)
        lc = OL.homspace_layout(kind, cod, dom)
        assert OC.rel_frobenius(OD.to_dense(lc, c.cpu().numpy()), D) <= TOL
        del T, C
        gc.collect()
