"""Plan-cache behaviour that needs a device: cold plans inside CUDA-graph capture, per-device keys,
and the binding's buffer checks. Needs a B200."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from workloads import configs as W  # noqa: E402
from tests import harness as H  # noqa: E402
from oracle import dense as OD, contract as OC  # noqa: E402


def test_cold_plan_inside_graph_capture():
    """The first tk_contract of a pattern (plan built and its tables uploaded) may run inside
    torch.cuda.graph capture; the replayed graph gives the oracle's result."""
    from paper_2508_10076_b200 import tk, layout_io
    tk.tk_cache_clear()
    cfg = W.cfg3(chi=64)
    ref = H.oracle_chain_dense(cfg)
    dev = torch.device("cuda")
    T = {}
    for name, (spec, idx) in cfg["tensors"].items():
        t = tk.tensor_from_spec(spec)
        T[name] = (t, torch.from_numpy(layout_io.fill(t, cfg["cfg"], idx)).to(dev))
    steps = []
    for (na, la, nb, lb, nc, lc, ncod) in cfg["steps"]:
        C = tk.tk_contract_output(T[na][0], la, T[nb][0], lb, lc, ncod)
        T[nc] = (C, torch.full((C.nelems,), float("nan"), dtype=torch.float64, device=dev))
        steps.append((na, la, nb, lb, nc, lc))
    # workspaces sized on the host (no plan upload happens on the device before the capture)
    ws = torch.empty(1 << 24, dtype=torch.float64, device=dev)
    assert tk.tk_cache_size() == 0
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for (na, la, nb, lb, nc, lc) in steps:
            tk.tk_contract(T[na][0], T[na][1], la, T[nb][0], T[nb][1], lb, T[nc][0], T[nc][1], lc, ws=ws,
                           ws_bytes=ws.numel() * 8)
    assert tk.tk_cache_size() >= len(steps)
    g.replay()
    torch.cuda.synchronize()
    for name, (lt, D) in ref.items():
        flat = T[name][1].cpu().numpy()
        assert not np.isnan(flat).any()
        assert OC.rel_frobenius(OD.to_dense(lt, flat), D) <= 1e-12


def test_binding_checks_buffers():
    from paper_2508_10076_b200 import tk
    V = W.space("U1", [((-1,), 2), ((0,), 3), ((1,), 2)])
    A = tk.tensor_from_spec({"cod": [V, V], "dom": [V]})
    C = tk.tensor_from_spec({"cod": [V], "dom": [W.dual(V), V]})
    a = torch.zeros(A.nelems, dtype=torch.float64, device="cuda")
    c = torch.zeros(C.nelems, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        tk.tk_permute(A, a.float(), [0], [1, 2], C, c)
    with pytest.raises(ValueError):
        tk.tk_permute(A, a[:-1], [0], [1, 2], C, c)
    with pytest.raises(ValueError):
        tk.tk_permute(A, a.cpu(), [0], [1, 2], C, c)
    with pytest.raises(ValueError):
        tk.tk_permute(A, torch.zeros(2 * A.nelems, dtype=torch.float64, device="cuda")[::2], [0], [1, 2], C, c)
    tk.tk_permute(A, a, [0], [1, 2], C, c)
