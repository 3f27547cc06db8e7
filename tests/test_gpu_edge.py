"""Degenerate and edge cases of the CUDA path against the oracle -- needs a B200.

  * empty tensors (no allowed sector) and outputs with no coupled sector shared by A~ and B~
    (every block K = 0: C = beta * C);
  * full contractions to a scalar (rank-0 output) and outer products (no contracted leg);
  * alpha = 0 (C = beta * C, inputs may hold NaN-free garbage), beta = 1 accumulation, negative alpha;
  * ragged subblocks (single-element sectors next to large ones), every kind;
  * the workspace contract: too small -> TK_ERR_WORKSPACE_TOO_SMALL with C untouched.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import layout as OL, dense as OD, contract as OC  # noqa: E402
from workloads import configs as W  # noqa: E402

TOL = 1e-12


def _run(kind, A_sp, labA, B_sp, labB, labC, ncod, alpha=1.0, beta=0.0, seed=0, c0=None):
    from paper_2508_10076_b200 import tk
    la = OL.homspace_layout(kind, A_sp["cod"], A_sp["dom"])
    lb = OL.homspace_layout(kind, B_sp["cod"], B_sp["dom"])
    rng = np.random.default_rng(seed)
    xa, xb = rng.standard_normal(la.nelems), rng.standard_normal(lb.nelems)
    A, B = tk.tensor_from_spec(A_sp), tk.tensor_from_spec(B_sp)
    C = tk.tk_contract_output(A, labA, B, labB, labC, ncod)
    cod, dom = OC.output_spaces(A_sp["cod"], A_sp["dom"], B_sp["cod"], B_sp["dom"], labA, labB, labC, ncod)
    lc = OL.homspace_layout(kind, cod, dom)
    assert C.nelems == lc.nelems
    y0 = rng.standard_normal(lc.nelems) if c0 is None else c0
    a, b = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    c = torch.from_numpy(y0.copy()).cuda()
    nws = tk.tk_contract_workspace(A, labA, B, labB, C, labC)
    ws = torch.empty(max(nws // 8 + 32, 1), dtype=torch.float64, device="cuda")
    tk.tk_contract(A, a, labA, B, b, labB, C, c, labC, alpha=alpha, beta=beta, ws=ws, ws_bytes=ws.numel() * 8)
    torch.cuda.synchronize()
    D = OC.contract(kind, OD.to_dense(la, xa), A_sp["cod"] + A_sp["dom"], len(A_sp["cod"]), labA,
                    OD.to_dense(lb, xb), B_sp["cod"] + B_sp["dom"], len(B_sp["cod"]), labB, labC, ncod)
    want = alpha * D + (beta * OD.to_dense(lc, y0) if beta != 0 else 0.0)
    got = OD.to_dense(lc, c.cpu().numpy())
    return got, want, lc


def _check(got, want):
    if np.linalg.norm(want.ravel()) == 0:
        assert np.abs(got).max(initial=0.0) == 0.0
    else:
        assert OC.rel_frobenius(got, want) <= TOL


def test_all_blocks_zero_k():
    """A~ and B~ share no coupled sector: every GEMM group has K = 0 and C = beta * C."""
    V = W.space("U1", [((0,), 3), ((1,), 2)])
    X = W.space("U1", [((5,), 2)])        # contracted leg: charges 5 cannot balance V's
    A = {"cod": [V], "dom": [X]}
    B = {"cod": [X], "dom": [V]}
    for beta in (0.0, 0.5):
        got, want, lc = _run("U1", A, [1, 2], B, [2, 3], [1, 3], 1, beta=beta)
        _check(got, want)


def test_empty_operand():
    """An operand with no allowed sector (nelems 0): the output is beta * C."""
    V = W.space("U1", [((1,), 3)])
    A = {"cod": [V, V], "dom": [V]}       # charge 2 <- 1: nothing allowed
    B = {"cod": [V], "dom": [V]}
    from paper_2508_10076_b200 import tk
    assert tk.tensor_from_spec(A).nelems == 0
    got, want, lc = _run("U1", A, [1, 2, 3], B, [3, 4], [1, 2, 4], 2, beta=-1.0)
    _check(got, want)


@pytest.mark.parametrize("kind,secs", [
    ("U1", [((-1,), 1), ((0,), 17), ((1,), 2)]),
    ("fU1xU1", [((0, 0), 1), ((1, 1), 9), ((1, -1), 1), ((2, 0), 5)]),
    ("SU2", [((0,), 1), ((1,), 7), ((2,), 1)]),
    ("fU1xSU2", [((0, 0), 1), ((1, 1), 6), ((-1, 1), 1)]),
])
def test_scalar_and_outer_product(kind, secs):
    """Full contraction to a rank-0 tensor (trace of A^T B) and the outer product (no shared leg)."""
    V = W.space(kind, secs)
    A = {"cod": [V, V], "dom": [V]}
    B = {"cod": [V], "dom": [V, V]}
    got, want, lc = _run(kind, A, [1, 2, 3], B, [3, 1, 2], [], 0)
    assert lc.nelems <= 1
    _check(got, want)
    S = {"cod": [V], "dom": [V]}
    got, want, lc = _run(kind, S, [1, 2], S, [3, 4], [1, 3, 2, 4], 2, seed=2)
    _check(got, want)


@pytest.mark.parametrize("alpha,beta", [(0.0, 1.0), (0.0, 0.0), (-1.5, 1.0), (2.0, -0.25)])
def test_alpha_beta_degenerate(alpha, beta):
    cfg = W.cfg2(chi=96)
    (na, la_, nb, lb_, nc, lc_, ncod) = cfg["steps"][0]
    A, B = cfg["tensors"][na][0], cfg["tensors"][nb][0]
    got, want, lc = _run("U1", A, la_, B, lb_, lc_, ncod, alpha=alpha, beta=beta, seed=5)
    _check(got, want)


def test_workspace_too_small_leaves_output():
    from paper_2508_10076_b200 import tk
    cfg = W.cfg4(d_leg=16)
    (na, la_, nb, lb_, nc, lc_, ncod) = cfg["steps"][0]
    A, B = tk.tensor_from_spec(cfg["tensors"][na][0]), tk.tensor_from_spec(cfg["tensors"][nb][0])
    C = tk.tk_contract_output(A, la_, B, lb_, lc_, ncod)
    a = torch.zeros(A.nelems, dtype=torch.float64, device="cuda")
    b = torch.zeros(B.nelems, dtype=torch.float64, device="cuda")
    c = torch.full((C.nelems,), 7.0, dtype=torch.float64, device="cuda")
    nws = tk.tk_contract_workspace(A, la_, B, lb_, C, lc_)
    assert nws > 0
    ws = torch.empty(nws // 8 + 32, dtype=torch.float64, device="cuda")
    with pytest.raises(tk.TKError) as e:
        tk.tk_contract(A, a, la_, B, b, lb_, C, c, lc_, ws=ws, ws_bytes=nws - 8)
    assert e.value.status == "TK_ERR_WORKSPACE_TOO_SMALL"
    torch.cuda.synchronize()
    assert bool((c == 7.0).all())


# ------------------------------------------------------------------ seg jobs (latency-regime permutes)
# Permutes below 2^24 elements run as kJobSeg jobs (tk_kernels.hpp): chunks of <= 32 groups and
# <= 1024 rows per job, one row longer than a job taking a job of its own, transposing groups walked
# along the source-fastest leg. Each case below drives one of those limits.
def test_seg_long_row():
    V = [((0,), 10000)]
    S = [((0,), 1), ((1,), 1)]
    # V (x) S <- S, permuted to (S, V ; S): one 10000-element row per block (> job_elems = 512)
    err = _perm_case_spaces("U1", [W.space("U1", V), W.space("U1", S)], [W.space("U1", S)], [1, 0], [2])
    assert err <= TOL


def test_seg_many_tiny_groups():
    from tests.test_gpu_parity import _perm_case
    secs = [((q,), 1) for q in range(-3, 4)]  # 1-element subblocks: > 32 groups per job
    assert _perm_case("U1", secs, [0, 0], [0, 0], [2, 0], [3, 1], alpha=-1.5) <= TOL
    assert _perm_case("fU1xU1", [((0, 0), 1), ((1, 1), 1), ((1, -1), 1), ((2, 0), 1), ((-1, 1), 1)],
                      [0, 1], [0], [2, 1], [0]) <= TOL


def test_seg_transposes():
    from tests.test_gpu_parity import _perm_case
    secs = [((0,), 40), ((1,), 30), ((-1,), 20)]
    assert _perm_case("U1", secs, [0, 1], [], [1, 0], [], beta=0.5) <= TOL
    assert _perm_case("U1", secs, [0], [0, 1], [2, 1], [0]) <= TOL
    # 3.2 M elements in rows of 2: job_elems ~ 2700 > 1024 rows x 2, so the row limit of a job binds
    V1 = W.space("U1", [((0,), 2), ((1,), 2), ((-1,), 2)])
    V = W.space("U1", [((0,), 40), ((1,), 40), ((-1,), 40), ((2,), 20)])
    assert _perm_case_spaces("U1", [V1, V], [V, V], [0, 2], [1, 3]) <= TOL


def _perm_case_spaces(kind, cod, dom, p, q, seed=0):
    from paper_2508_10076_b200 import tk
    lt = OL.homspace_layout(kind, cod, dom)
    x = np.random.default_rng(seed).standard_normal(lt.nelems)
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    ls = OL.homspace_layout(kind, c2, d2)
    par = [OD.parity_vector(s) for s in cod + dom]
    ref = OC.permute_dense(OD.to_dense(lt, x), par, len(cod), p, q)
    A = tk.tensor_from_spec({"cod": cod, "dom": dom})
    C = tk.tensor_from_spec({"cod": c2, "dom": d2})
    c = torch.full((ls.nelems,), float("nan"), dtype=torch.float64, device="cuda")
    tk.tk_permute(A, torch.from_numpy(x).cuda(), p, q, C, c)
    torch.cuda.synchronize()
    return OC.rel_frobenius(OD.to_dense(ls, c.cpu().numpy()), ref)


# ------------------------------------------------------------------ gathered skinny GEMM
# The T.W steps of the DMRG chains (every GEMM block K, N <= 16, abelian) run as one gathered GEMM:
# A~ and B~ are read straight from A and B with the permutes' offsets and signs (tk_kernels.hpp,
# GatherSeg). Cases: fermionic signs, alpha / beta accumulation, and an output permute after it.
@pytest.mark.parametrize("cfgfun,kind", [(lambda: W.cfg3(chi=96), "fU1xU1"), (lambda: W.cfg2(chi=128), "U1")])
def test_gather_gemm_alpha_beta_and_output_permute(cfgfun, kind):
    cfg = cfgfun()
    specs = {k: v[0] for k, v in cfg["tensors"].items()}
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][0]
    cod, dom = OC.output_spaces(specs[na]["cod"], specs[na]["dom"], specs[nb]["cod"], specs[nb]["dom"],
                                la, lb, lc, ncod)
    T1 = {"cod": cod, "dom": dom}
    (_, la2, nb2, lb2, _, lc2, ncod2) = cfg["steps"][1]
    for alpha, beta in ((1.0, 0.0), (-0.5, 0.75)):
        got, want, lc_ = _run(kind, T1, la2, specs[nb2], lb2, lc2, ncod2, alpha=alpha, beta=beta, seed=11)
        _check(got, want)
    # a non-identity output permute after the gathered GEMM (C~ -> C with alpha / beta)
    lc3 = [lc2[2], lc2[0], lc2[4], lc2[1], lc2[3]]
    got, want, _ = _run(kind, T1, la2, specs[nb2], lb2, lc3, 2, alpha=2.0, beta=-1.0, seed=12)
    _check(got, want)


# ------------------------------------------------------------------ recoupling groups of > 4 sources
def test_recoupling_staged_path():
    """SU(2) rank-4 permutes with spins up to 2 have recoupling groups of up to 5 source trees; groups
    of more than 4 sources take the staged-shared-memory recoupling kernel (the rest run in the general
    permute launch). Checked against the dense oracle."""
    from tests.test_gpu_parity import _perm_case
    secs = [((0,), 2), ((1,), 1), ((2,), 2), ((3,), 1), ((4,), 2)]
    for p, q, beta in (([2, 0], [3, 1], 0.0), ([3, 1, 0], [2], 0.5), ([1, 3], [0, 2], 0.0)):
        assert _perm_case("SU2", secs, [0, 0], [0, 0], p, q, alpha=-1.5, beta=beta) <= TOL, (p, q)
    # fZ2 x SU(2) x SU(2): fermionic signs and two recoupled factors
    secs2 = [((0, 0), 1), ((1, 1), 1), ((0, 2), 1), ((2, 0), 1), ((1, 3), 1), ((2, 2), 1)]
    assert _perm_case("fSU2xSU2", secs2, [0, 0], [0, 0], [2, 0], [3, 1]) <= TOL


def test_large_permute_all_job_classes():
    """A 24 M-element permute (>= 2^24: one launch per job class) whose sectors range from degeneracy 1 to
    28, so rows, smem-tiled and packed jobs all occur (TK_PLAN_DEBUG), each pattern against the dense
    oracle (1.9 GB dense arrays on the host)."""
    from tests.test_gpu_parity import _perm_case
    secs = [((-6,), 1), ((-5,), 1), ((-4,), 2), ((-3,), 8), ((-2,), 14), ((-1,), 22), ((0,), 28), ((1,), 22),
            ((2,), 14), ((3,), 8), ((4,), 2), ((5,), 1), ((6,), 1)]
    for p, q in (([0, 2], [1, 3]), ([2, 0], [1, 3]), ([3, 1], [0, 2])):
        assert _perm_case("U1", secs, [0, 0], [0, 0], p, q, beta=0.5) <= TOL, (p, q)


def test_gather_gemm_wide_k():
    """The gathered GEMM's K = 9..16 instance (K and N of 12 / 10): A (V, w ; V) contracted over w with
    B (w' ; w), so every block is skinny and the operand permute is folded into the GEMM."""
    V = W.space("U1", [((q,), d) for q, d in zip(range(-3, 4), [6, 11, 17, 20, 17, 11, 6])])
    w = W.space("U1", [((0,), 12), ((1,), 10)])
    A = {"cod": [V, w], "dom": [V]}
    B = {"cod": [w], "dom": [w]}
    for alpha, beta in ((1.0, 0.0), (-2.0, 0.5)):
        got, want, _ = _run("U1", A, [1, 2, 3], B, [4, 2], [1, 3, 4], 2, alpha=alpha, beta=beta, seed=3)
        _check(got, want)


def test_splitk_alpha_beta():
    """The T3.R step of cfg2 runs split-K (partial tiles + ordered reduction): alpha / beta are applied by
    the reduction kernel; also with an output permute after it."""
    cfg = W.cfg2(chi=512)
    specs = {k: v[0] for k, v in cfg["tensors"].items()}
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"][:3]:
        cod, dom = OC.output_spaces(specs[na]["cod"], specs[na]["dom"], specs[nb]["cod"], specs[nb]["dom"],
                                    la, lb, lc, ncod)
        specs[nc] = {"cod": cod, "dom": dom}
    (na, la, nb, lb, nc, lc, ncod) = cfg["steps"][3]
    for alpha, beta in ((1.0, 0.0), (0.5, -1.25)):
        got, want, _ = _run("U1", specs[na], la, specs[nb], lb, lc, ncod, alpha=alpha, beta=beta, seed=9)
        _check(got, want)
    lc2 = [lc[3], lc[0], lc[2], lc[1]]
    got, want, _ = _run("U1", specs[na], la, specs[nb], lb, lc2, 2, alpha=-1.0, beta=0.5, seed=10)
    _check(got, want)


# ------------------------------------------------------------------ determinism
@pytest.mark.parametrize("cfgfun", [lambda: W.cfg2(chi=512), lambda: W.cfg3(chi=512), lambda: W.cfg7(n_mult=100)],
                         ids=["cfg2", "cfg3", "cfg7"])
def test_bitwise_deterministic(cfgfun):
    """No atomics anywhere on the path (split-K sums its partial tiles in a fixed order): two runs of a
    chain give bit-identical results."""
    from tests import harness as H
    cfg = cfgfun()
    r1 = H.gpu_chain(cfg)
    r2 = H.gpu_chain(cfg)
    for k in r1:
        assert np.array_equal(r1[k][1], r2[k][1]), k


# ------------------------------------------------------------------ large permutes (split launches)
@pytest.mark.parametrize("cplx,alpha,beta", [(False, 1.0, 0.0), (False, -0.5, 0.25), (True, 0.75, -1.0)])
def test_large_permute_cfg4_pattern(cplx, alpha, beta):
    """A permute above 2^24 elements (rows-only launch + tail launch) whose leg 0 stays unit-stride while
    the next legs swap (the cfg4 pattern); alpha / beta and ComplexF64 (tk_permute: interleaved ->
    interleaved)."""
    from paper_2508_10076_b200 import tk
    from oracle import layout as OL, dense as OD, contract as OC
    V = W.space("U1", [((-1,), 26), ((0,), 39), ((1,), 26)])
    cod, dom = [V, V], [V, V]
    p, q = [0, 2], [1, 3]          # A (x1, x2; x3, x4) -> (x1, x3; x2, x4)
    lt = OL.homspace_layout("U1", cod, dom)
    assert lt.nelems >= 1 << 24
    rng = np.random.default_rng(21)
    x = rng.standard_normal(lt.nelems) + (1j * rng.standard_normal(lt.nelems) if cplx else 0.0)
    c2, d2 = OC.permuted_spaces(cod, dom, p, q)
    ls = OL.homspace_layout("U1", c2, d2)
    y0 = rng.standard_normal(ls.nelems) + (1j * rng.standard_normal(ls.nelems) if cplx else 0.0)
    dt = tk.TK_C64 if cplx else tk.TK_F64
    A = tk.tensor_from_spec({"cod": cod, "dom": dom}, dt)
    C = tk.tensor_from_spec({"cod": c2, "dom": d2}, dt)
    a = torch.from_numpy(x).cuda()
    c = torch.from_numpy(y0.copy()).cuda() if beta != 0 else torch.full((ls.nelems,), float("nan"),
                                                                           dtype=a.dtype, device="cuda")
    tk.tk_permute(A, a, p, q, C, c, alpha=alpha, beta=beta)
    torch.cuda.synchronize()
    assert tk.tk_last_launch_count() >= 1
    # the permute is a bijection of subblocks: compare subblock by subblock (no dense embedding needed)
    ref = OD.from_dense(ls, OC.permute_dense(OD.to_dense(lt, x), [OD.parity_vector(s) for s in cod + dom], 2, p, q))
    want = alpha * ref + (beta * y0 if beta != 0 else 0.0)
    got = c.cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
