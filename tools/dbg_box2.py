import sys, numpy as np
sys.path.insert(0, '.')
from workloads import configs as W
from tests import harness as H
from tests.test_gpu_parity import rel_err_blocks
for d in (48, 96, 128):
    cfg = W.cfg4(d_leg=d)
    ref = H.oracle_chain_blocks(cfg)
    got = H.gpu_chain(cfg)
    lt, blocks = ref["C"]
    C, flat = got["C"]
    print(d, "err", rel_err_blocks(lt, flat, blocks), "nan", np.isnan(flat).sum())
