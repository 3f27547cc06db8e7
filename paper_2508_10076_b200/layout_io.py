"""Place seeded subblock values into a flat buffer through the LIBRARY's layout queries.

The values come from `workloads.gen` keyed by tree pair; their position comes from
tk_tensor_subblocks (offset, block rows, extents). If the library's layout were
wrong, the oracle (which places the same keyed values with its own layout) would
disagree with the CUDA result -- that is the point of keying by tree pair.
"""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

from workloads import gen


def decode_keys(t):
    """Subblock keys as (cod_unc, cod_inner, coupled, dom_unc, dom_inner) label tuples."""
    inf = t.info()
    n1, n2, w = inf["n_cod"], inf["n_dom"], inf["width"]
    sb = t.subblocks()
    out = []
    for row in sb["keys"]:
        labs = [tuple(int(x) for x in row[i * w:(i + 1) * w]) for i in range(len(row) // w)]
        i = 0
        su = tuple(labs[i:i + n1]); i += n1
        si = tuple(labs[i:i + max(n1 - 2, 0)]); i += max(n1 - 2, 0)
        c = labs[i]; i += 1
        fu = tuple(labs[i:i + n2]); i += n2
        fi = tuple(labs[i:i + max(n2 - 2, 0)])
        out.append((su, si, c, fu, fi))
    return out


def subblock_geometry(t):
    """Per subblock: (offset, ld, rows_s, cols_s) with rows_s = prod cod extents, cols_s = prod dom extents."""
    inf = t.info()
    n1, n2 = inf["n_cod"], inf["n_dom"]
    _, brows, _, _ = t.blocks()
    sb = t.subblocks()
    ext = sb["extents"]
    rows = np.prod(ext[:, :n1], axis=1) if n1 else np.ones(len(ext), np.int64)
    cols = np.prod(ext[:, n1:n1 + n2], axis=1) if n2 else np.ones(len(ext), np.int64)
    ld = brows[sb["block"]]
    return sb["offset"], ld, rows, cols


def fill(t, cfg, tensor_index, complex_=False, threads=None):
    """Host flat buffer (numpy) of tensor t filled with the seeded values of (cfg, tensor_index)."""
    keys = decode_keys(t)
    off, ld, rows, cols = subblock_geometry(t)
    flat = np.zeros(t.nelems, dtype=np.complex128 if complex_ else np.float64)

    def one(i):
        r, c = int(rows[i]), int(cols[i])
        v = gen.subblock_values(cfg, tensor_index, keys[i], r * c, complex_)
        o, l = int(off[i]), int(ld[i])
        if c == 1 or l == r:
            flat[o:o + r * c] = v
        else:
            view = np.lib.stride_tricks.as_strided(flat[o:], shape=(c, r),
                                                   strides=(l * flat.itemsize, flat.itemsize))
            view[...] = v.reshape(c, r)

    n = len(keys)
    nt = threads or min(32, os.cpu_count() or 1)
    if n > 64 and nt > 1:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, range(n)))
    else:
        for i in range(n):
            one(i)
    return flat
