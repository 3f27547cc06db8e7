"""Parity at the sizes that are TIMED (bench.py and tools/bench_configs.py run exactly these configs,
so the plans -- job classes, kernel instances, split-K, gathered GEMMs -- are the timed ones).

  * cfg4 (the bench workload): every one of the 6181 output subblocks, Float64 at D_leg 384 and
    ComplexF64 at D_leg 320 (reading C20), against the tier-2 charge-tuple oracle
    (oracle/blocksparse.py; itself equal to the dense oracle at reduced sizes, test_oracle_dense.py).
  * cfg7 (700 multiplets) and cfg8 (270 multiplets): the whole chain against the dense CG oracle
    (every bond sector populated; dense intermediates ~5.4 GB on the host).
Tolerance: relative Frobenius error <= 1e-12 (north_star), outputs start as NaN. Needs a B200 and
~40 GB of host memory.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import dense as OD, contract as OC, blocksparse as BS  # noqa: E402
from workloads import configs as W  # noqa: E402
from tests import harness as H  # noqa: E402

TOL = 1e-12


def _blocks_err(layout, flat, blocks):
    got = BS.to_blocks(layout, flat)
    assert len(got) == len(layout.subblocks)
    num = den = 0.0
    for k, g in got.items():
        r = blocks.get(k)
        if r is None:
            r = np.zeros_like(g)
        num += float(np.sum(np.abs(g - r) ** 2))
        den += float(np.sum(np.abs(r) ** 2))
    return math.sqrt(num / den)


@pytest.mark.parametrize("d_leg,cplx", [(384, False), (320, True)], ids=["f64_d384", "c64_d320"])
def test_cfg4_bench_size_every_subblock(d_leg, cplx):
    cfg = W.cfg4(d_leg=d_leg, complex_=cplx)
    got = H.gpu_chain(cfg, complex_=cplx)
    torch.cuda.empty_cache()
    C, flat = got["C"]
    assert not np.isnan(flat).any(), "unwritten output elements"
    ref = H.oracle_chain_blocks(cfg, complex_=cplx)
    lt, blocks = ref["C"]
    assert C.nelems == lt.nelems
    assert len(lt.subblocks) == 6181
    err = _blocks_err(lt, flat, blocks)
    assert err <= TOL, f"rel Frobenius {err:.3e}"


@pytest.mark.parametrize("cfgfun", [W.cfg7, W.cfg8], ids=["cfg7_m700", "cfg8_m270"])
def test_chain_bench_size_dense(cfgfun):
    cfg = cfgfun()
    got = H.gpu_chain(cfg)
    ref = H.oracle_chain_dense(cfg)
    for name in list(ref):
        lt, D = ref.pop(name)
        C, flat = got[name]
        assert C.nelems == lt.nelems
        assert not np.isnan(flat).any(), f"{name}: unwritten output elements"
        err = OC.rel_frobenius(OD.to_dense(lt, flat), D)
        del D
        assert err <= TOL, f"{name}: rel Frobenius {err:.3e}"
