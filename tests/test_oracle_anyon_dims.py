"""Quantum-dimension pins of the planar anyon oracle (oracle/planar.py) -- values fixed by the category.

The planar oracle replays the paper's moves (bends with B-symbols, F-rotations with chi, tadpole
d_c/d_e). Its SU(2) results are pinned against the dense CG oracle
(test_oracle_planar.py), but the factors only anyons exercise -- non-integer quantum dimensions inside
sqrt(d_c/d_e) and d_c/d_e, the Fib/Ising B-symbols -- need anchors of their own. The quantum (pivotal)
trace fixes them (Fib P:2418-2421: d_tau = phi; Ising P:2440-2447: d_sigma = sqrt 2; textbook):

  * tr(id_{V (x) W}) = dim_q(V) dim_q(W), dim_q(V) = sum_a deg_a d_a;
  * tr_2(id_{V (x) V}) = dim_q(V) id_V; the left partial trace (through the cyclic rotation: F-moves, chi,
    B-symbols) is dim_q(V) times the bent id_V, whose entries are sqrt(d_a) (loop value dim_q(V));
  * the projector P_c onto the fusion channel c of a (x) b has tr(P_c) = d_c and tr_2(P_c) = (d_c / d_a) id_a
    (the Markov trace of the Temperley-Lieb / Fibonacci projectors: for tau (x) tau, 1/phi and 1).
"""
import math

import numpy as np
import pytest

from oracle import layout as L, planar as OP, sectors
from workloads import configs as W

PHI = (1 + math.sqrt(5)) / 2


def _identity_flat(kind, cod, dom):
    lt = L.homspace_layout(kind, cod, dom)
    x = np.zeros(lt.nelems)
    for (c, r, k, off) in lt.blocks:
        assert r == k
        x[off:off + r * k] = np.eye(r).ravel()
    return lt, x


def _projector_flat(kind, cod, dom, channel):
    lt = L.homspace_layout(kind, cod, dom)
    x = np.zeros(lt.nelems)
    for (c, r, k, off) in lt.blocks:
        if tuple(c) == tuple(channel):
            x[off:off + r * k] = np.eye(r).ravel()
    return lt, x


def _qdim(kind, secs):
    return sum(n * sectors.qdim(kind, a) for a, n in secs)


CASES = [("Fib", [((0,), 2), ((1,), 3)], 2 + 3 * PHI),
         ("Fib", [((1,), 1)], PHI),
         ("Ising", [((0,), 1), ((1,), 2), ((2,), 1)], 2 + 2 * math.sqrt(2)),
         ("Ising", [((1,), 1)], math.sqrt(2))]


@pytest.mark.parametrize("kind,secs,dq", CASES)
def test_full_trace_of_identity_is_qdim_squared(kind, secs, dq):
    assert abs(_qdim(kind, secs) - dq) < 1e-14  # the kind's d_a are the paper's
    V = W.space(kind, secs)
    lt, x = _identity_flat(kind, [V, V], [V, V])
    got, lc = OP.trace_planar(kind, [V, V], [V, V], x, [0, 1], [2, 3], [], [])
    assert lc.nelems == 1
    assert abs(got[0] - dq * dq) < 1e-12 * dq * dq


@pytest.mark.parametrize("kind,secs,dq", CASES)
def test_right_partial_trace_of_identity_is_qdim_times_identity(kind, secs, dq):
    V = W.space(kind, secs)
    lt, x = _identity_flat(kind, [V, V], [V, V])
    got, lc = OP.trace_planar(kind, [V, V], [V, V], x, [1], [3], [0], [2])
    want = np.zeros(lc.nelems)
    for (c, r, k, off) in lc.blocks:
        want[off:off + r * k] = dq * np.eye(r).ravel()
    assert np.abs(got - want).max() < 1e-12 * dq


@pytest.mark.parametrize("kind,secs,dq", CASES)
def test_left_partial_trace_through_rotation_is_qdim_times_cup(kind, secs, dq):
    """Closing V1 with V1' of id_{V1 V2 <- V1' V2'} leaves the strand V2 -- V2' bent into a cup (the planar
    route rotates the tree: F-moves, chi, B-symbols) times one loop, dim_q(V). The cup is the bent id_V,
    whose squared entries sum to the loop value dim_q(V) = sum_a deg_a d_a, each entry being sqrt(d_a)."""
    V = W.space(kind, secs)
    lt, x = _identity_flat(kind, [V, V], [V, V])
    got, lc = OP.trace_planar(kind, [V, V], [V, V], x, [2], [0], [1, 3], [])
    l1, x1 = _identity_flat(kind, [V], [V])
    cup, lcup = OP.apply_planar(kind, [V], [V], x1, [0, 1], [])
    assert lc.nelems == lcup.nelems
    assert abs(float(cup @ cup) - dq) < 1e-12 * dq
    nz = np.sort(np.abs(cup[np.abs(cup) > 1e-15]))
    want_nz = np.sort(np.concatenate([[math.sqrt(sectors.qdim(kind, a))] * n for a, n in secs]))
    assert np.allclose(nz, want_nz, rtol=0, atol=1e-14)
    assert np.abs(got - dq * cup).max() < 1e-12 * dq


@pytest.mark.parametrize("kind,a,channels", [
    ("Fib", (1,), [((0,), 1.0), ((1,), PHI)]),
    ("Ising", (1,), [((0,), 1.0), ((2,), 1.0)]),
    ("Ising", (2,), [((0,), 1.0)]),
])
def test_channel_projector_traces(kind, a, channels):
    V = W.space(kind, [(a, 1)])
    da = sectors.qdim(kind, a)
    for ch, dc in channels:
        assert abs(sectors.qdim(kind, ch) - dc) < 1e-14
        lt, x = _projector_flat(kind, [V, V], [V, V], ch)
        full, _ = OP.trace_planar(kind, [V, V], [V, V], x, [0, 1], [2, 3], [], [])
        assert abs(full[0] - dc) < 1e-12
        part, lc = OP.trace_planar(kind, [V, V], [V, V], x, [1], [3], [0], [2])
        assert len(lc.blocks) == 1 and lc.nelems == 1
        assert abs(part[0] - dc / da) < 1e-12, ch


def test_pins_reject_plausible_wrong_factors(monkeypatch):
    """Not vacuous: a B-symbol off by sqrt(d_a), or a flipped Frobenius-Schur indicator chi on a non-trivial
    label, fails the trace pins."""
    kind, secs, dq = CASES[0]
    ob, oc = OP.bsymbol, OP.chi
    monkeypatch.setattr(OP, "bsymbol", lambda k, a, b, c: ob(k, a, b, c) * math.sqrt(sectors.qdim(k, a)))
    with pytest.raises(AssertionError):
        test_right_partial_trace_of_identity_is_qdim_times_identity(kind, secs, dq)
    monkeypatch.setattr(OP, "bsymbol", ob)
    monkeypatch.setattr(OP, "chi", lambda k, a: -oc(k, a) if sectors.qdim(k, a) > 1.2 else oc(k, a))
    with pytest.raises(AssertionError):
        test_left_partial_trace_through_rotation_is_qdim_times_cup(kind, secs, dq)
