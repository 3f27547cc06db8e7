"""Thin ctypes binding of libtk_b200.so (include/tk.h). Argument marshalling only.

Every operation runs in the C++ planner / sm_100a kernels of the library; this
module only converts Python values to the C ABI and raises on error. There is
no fallback: if the in-tree library is missing, importing fails loudly.
PyTorch is used by callers only for device memory and streams (raw pointers and
`torch.cuda.current_stream().cuda_stream` are passed through).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TK_LIB_PATH") or os.path.join(_HERE, "libtk_b200.so")  # override: experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2508_10076_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = ["TK_OK", "TK_ERR_INVALID_ARGUMENT", "TK_ERR_UNKNOWN_LABEL", "TK_ERR_SECTOR_MISMATCH",
          "TK_ERR_SPACE_MISMATCH", "TK_ERR_INVALID_PERMUTATION", "TK_ERR_BRAIDING_UNAVAILABLE",
          "TK_ERR_MALFORMED_NETWORK", "TK_ERR_UNSUPPORTED", "TK_ERR_WORKSPACE_TOO_SMALL", "TK_ERR_CUDA"]
TK_F64, TK_C64 = 0, 1

_p = ctypes.c_void_p
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)


class TKError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg}")
        self.code = code
        self.status = STATUS[code] if 0 <= code < len(STATUS) else str(code)


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_lib_tk_last_error = _sig("tk_last_error", [], ctypes.c_char_p)


def _check(code):
    if code != 0:
        raise TKError(code, _lib_tk_last_error().decode())


_space_create = _sig("tk_space_create", [ctypes.c_char_p, ctypes.c_int32, _i32p, _i64p, ctypes.c_int32,
                                         ctypes.POINTER(_p)])
_space_parse = _sig("tk_space_parse", [ctypes.c_char_p, ctypes.POINTER(_p)])
_space_info = _sig("tk_space_info", [_p, _i32p, _i64p, _i32p, _i32p])
_space_sectors = _sig("tk_space_sectors", [_p, _i32p, _i64p])
_space_release = _sig("tk_space_release", [_p], None)
_tensor_create = _sig("tk_tensor_create", [ctypes.c_int, ctypes.c_int32, ctypes.POINTER(_p), ctypes.c_int32,
                                           ctypes.POINTER(_p), ctypes.POINTER(_p)])
_tensor_nelems = _sig("tk_tensor_nelems", [_p, _i64p])
_tensor_info = _sig("tk_tensor_info", [_p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p])
_tensor_blocks = _sig("tk_tensor_blocks", [_p, _i32p, _i64p, _i64p, _i64p])
_tensor_subblocks = _sig("tk_tensor_subblocks", [_p, _i32p, _i32p, _i64p, _i64p, _i64p, _i64p])
_tensor_release = _sig("tk_tensor_release", [_p], None)
_contract_output = _sig("tk_contract_output", [_p, _i32p, _p, _i32p, _i32p, ctypes.c_int32, ctypes.POINTER(_p)])
_permute_workspace = _sig("tk_permute_workspace", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p,
                                                   ctypes.POINTER(ctypes.c_size_t)])
_permute = _sig("tk_permute", [_p, _p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, _p, ctypes.c_double,
                               ctypes.c_double, _p, ctypes.c_size_t, _p])
_permute_transfer = _sig("tk_permute_transfer", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, _dp])
_permute_transfer_planar = _sig("tk_permute_transfer_planar", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p,
                                                               ctypes.c_int32, _dp])
_contract_workspace = _sig("tk_contract_workspace", [_p, _i32p, _p, _i32p, _p, _i32p,
                                                     ctypes.POINTER(ctypes.c_size_t)])
_contract = _sig("tk_contract", [_p, _p, _i32p, ctypes.c_int32, _p, _p, _i32p, ctypes.c_int32, _p, _p, _i32p,
                                 ctypes.c_double, ctypes.c_double, _p, ctypes.c_size_t, _p])
_contract2_workspace = _sig("tk_contract2_workspace", [_p, _i32p, _p, _i32p, _p, _i32p, _p, _i32p, _p, _i32p,
                                                       ctypes.POINTER(ctypes.c_size_t), _i32p])
_contract2 = _sig("tk_contract2", [_p, _p, _i32p, _p, _p, _i32p, _p, _i32p, _p, _p, _i32p, _p, _p, _i32p,
                                   ctypes.c_double, ctypes.c_double, _p, ctypes.c_size_t, _p])
_contract_tuples_output = _sig("tk_contract_tuples_output", [_p, _p, _i32p, _i32p, ctypes.POINTER(_p)])
_contract_tuples_workspace = _sig("tk_contract_tuples_workspace", [_p, _p, _p, _i32p, _i32p,
                                                                   ctypes.POINTER(ctypes.c_size_t)])
_contract_tuples = _sig("tk_contract_tuples", [_p, _p, ctypes.c_int32, _p, _p, ctypes.c_int32, _p, _p, _i32p, _i32p,
                                               ctypes.c_double, ctypes.c_double, _p, ctypes.c_size_t, _p])
_ncon_output = _sig("tk_ncon_output", [ctypes.c_int32, _p, _p, _i32p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(_p)])
_ncon_workspace = _sig("tk_ncon_workspace", [ctypes.c_int32, _p, _p, _i32p, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_size_t)])
_ncon = _sig("tk_ncon", [ctypes.c_int32, _p, _p, _p, _i32p, ctypes.c_int32, ctypes.c_int32, _p, _p, ctypes.c_double,
                         ctypes.c_double, _p, ctypes.c_size_t, _p])
_profile_enable = _sig("tk_profile_enable", [ctypes.c_int32])
_phase_times = _sig("tk_phase_times", [ctypes.POINTER(ctypes.c_float), _dp, _dp])
_last_launch_count = _sig("tk_last_launch_count", [], ctypes.c_int32)
_contract_roofline = _sig("tk_contract_roofline", [_p, _i32p, _p, _i32p, _p, _i32p, ctypes.c_double, ctypes.c_double,
                                                   _dp])
_dmma_probe = _sig("tk_dmma_probe", [ctypes.c_int32, ctypes.c_int64, _p, _dp])
_fsymbol = _sig("tk_fsymbol", [ctypes.c_char_p] + [_i32p] * 6 + [_dp])
_rsymbol = _sig("tk_rsymbol", [ctypes.c_char_p] + [_i32p] * 3 + [_dp])
_svd_workspace = _sig("tk_svd_workspace", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32,
                                           ctypes.POINTER(ctypes.c_size_t)])
_svd = _sig("tk_svd", [_p, _p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, ctypes.c_size_t, _p])
_svd_spectrum = _sig("tk_svd_spectrum", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, _p, _i32p, _i64p,
                                         _dp])
_svd_truncate = _sig("tk_svd_truncate", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, ctypes.c_int64,
                                         ctypes.c_double, _p, ctypes.POINTER(_p), ctypes.POINTER(_p),
                                         ctypes.POINTER(_p), ctypes.POINTER(_p), _dp, _dp])
_svd_extract = _sig("tk_svd_extract", [_p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, _p, _p, _p, _p, _p,
                                       _p, _p])
_trace_output = _sig("tk_trace_output", [_p, _i32p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32,
                                         ctypes.POINTER(_p)])
_trace_workspace = _sig("tk_trace_workspace", [_p, _i32p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _i32p,
                                               ctypes.c_int32, _p, ctypes.POINTER(ctypes.c_size_t)])
_trace = _sig("tk_trace", [_p, _p, _i32p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _p, _p,
                           ctypes.c_double, ctypes.c_double, _p, ctypes.c_size_t, _p])
_trace_transfer = _sig("tk_trace_transfer", [_p, _i32p, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _i32p,
                                             ctypes.c_int32, _p, _dp])
_cache_clear = _sig("tk_cache_clear", [], None)
_cache_size = _sig("tk_cache_size", [], ctypes.c_int64)
_version = _sig("tk_version", [], ctypes.c_char_p)

EXPORTED = ["tk_space_create", "tk_space_parse", "tk_space_info", "tk_space_sectors", "tk_space_dual",
            "tk_space_retain", "tk_space_release", "tk_tensor_create", "tk_tensor_nelems", "tk_tensor_info",
            "tk_tensor_blocks", "tk_tensor_subblocks", "tk_tensor_retain", "tk_tensor_release",
            "tk_contract_output", "tk_permute_workspace", "tk_permute", "tk_contract_workspace", "tk_contract",
            "tk_profile_enable", "tk_phase_times", "tk_last_launch_count", "tk_fsymbol", "tk_rsymbol",
            "tk_permute_transfer", "tk_permute_transfer_planar", "tk_last_error", "tk_cache_clear", "tk_version", "tk_svd_workspace", "tk_svd",
            "tk_svd_spectrum", "tk_svd_truncate", "tk_svd_extract", "tk_trace_output", "tk_trace_workspace",
            "tk_trace", "tk_trace_transfer", "tk_contract_tuples_output", "tk_contract_tuples_workspace",
            "tk_contract_tuples", "tk_ncon_output", "tk_ncon_workspace", "tk_ncon", "tk_cache_size",
            "tk_contract_roofline", "tk_dmma_probe", "tk_contract2_workspace", "tk_contract2"]


def _i32(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int32).ravel())
    return a, a.ctypes.data_as(_i32p)


def _ptr(x):
    """Device pointer of a torch tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


_TORCH_DT = {TK_F64: "torch.float64", TK_C64: "torch.complex128"}


def _data(t, x, what):
    """Pointer to the data of tensor map `t` held in torch tensor `x`, after checking what the C ABI
    cannot: a CUDA tensor, contiguous, of t's element type, with at least t.nelems elements.
    Raw integer pointers are passed through unchecked (C-style callers own that contract)."""
    if x is None or isinstance(x, int):
        return x
    inf = t.info()
    if not x.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if not x.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous tensor")
    if str(x.dtype) != _TORCH_DT[inf["dtype"]]:
        raise TypeError(f"{what}: dtype {x.dtype} does not match the tensor map ({_TORCH_DT[inf['dtype']]})")
    if x.numel() < t.nelems:
        raise ValueError(f"{what}: {x.numel()} elements < the tensor map's {t.nelems}")
    return x.data_ptr()


def _ws(ws, ws_bytes):
    """Workspace pointer; a torch workspace must be CUDA, contiguous and hold ws_bytes."""
    if ws is None or isinstance(ws, int):
        return ws
    if not ws.is_cuda or not ws.is_contiguous():
        raise ValueError("workspace: expected a contiguous CUDA tensor")
    if ws.numel() * ws.element_size() < ws_bytes:
        raise ValueError(f"workspace: {ws.numel() * ws.element_size()} bytes < ws_bytes = {ws_bytes}")
    return ws.data_ptr()


def _labels(t, lab, what):
    n = t.nlegs
    if len(lab) != n:
        raise ValueError(f"{what}: {len(lab)} labels for a tensor map with {n} legs")
    return _i32(lab)


def _stream(stream):
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            return None
    return stream if isinstance(stream, int) else stream.cuda_stream


# ---------------------------------------------------------------------- objects
class Space:
    """tk_space handle (reference counted on the C side)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _space_release is not None:
            _space_release(self.h)
            self.h = None

    def info(self):
        n, dim, dual, w = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _check(_space_info(self.h, ctypes.byref(n), ctypes.byref(dim), ctypes.byref(dual), ctypes.byref(w)))
        return n.value, dim.value, bool(dual.value), w.value

    def sectors(self):
        n, _, _, w = self.info()
        lab = np.zeros(n * w, np.int32)
        deg = np.zeros(n, np.int64)
        _check(_space_sectors(self.h, lab.ctypes.data_as(_i32p), deg.ctypes.data_as(_i64p)))
        return [tuple(int(x) for x in lab[i * w:(i + 1) * w]) for i in range(n)], deg


class Tensor:
    """tk_tensor handle: host-side block layout of a tensor map."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _tensor_release is not None:
            _tensor_release(self.h)
            self.h = None

    @property
    def nelems(self):
        if getattr(self, "_nelems", None) is None:  # tensor maps are immutable: query once
            n = ctypes.c_int64()
            _check(_tensor_nelems(self.h, ctypes.byref(n)))
            self._nelems = n.value
        return self._nelems

    @property
    def nlegs(self):
        inf = self.info()
        return inf["n_cod"] + inf["n_dom"]

    def info(self):
        if getattr(self, "_info", None) is None:
            v = [ctypes.c_int32() for _ in range(7)]
            _check(_tensor_info(self.h, *[ctypes.byref(x) for x in v]))
            keys = ("n_cod", "n_dom", "dtype", "width", "n_blocks", "n_subblocks", "key_len")
            self._info = dict(zip(keys, (x.value for x in v)))
        return dict(self._info)

    def blocks(self):
        inf = self.info()
        nb, w = inf["n_blocks"], inf["width"]
        cp = np.zeros(max(nb * w, 1), np.int32)
        rows, cols, off = (np.zeros(max(nb, 1), np.int64) for _ in range(3))
        _check(_tensor_blocks(self.h, cp.ctypes.data_as(_i32p), rows.ctypes.data_as(_i64p),
                              cols.ctypes.data_as(_i64p), off.ctypes.data_as(_i64p)))
        return cp[:nb * w].reshape(nb, w), rows[:nb], cols[:nb], off[:nb]

    def subblocks(self):
        inf = self.info()
        ns, kl = inf["n_subblocks"], inf["key_len"]
        keys = np.zeros(max(ns * kl, 1), np.int32)
        blk = np.zeros(max(ns, 1), np.int32)
        ro, co, off = (np.zeros(max(ns, 1), np.int64) for _ in range(3))
        ext = np.zeros(max(ns, 1) * 8, np.int64)
        _check(_tensor_subblocks(self.h, keys.ctypes.data_as(_i32p), blk.ctypes.data_as(_i32p),
                                 ro.ctypes.data_as(_i64p), co.ctypes.data_as(_i64p), ext.ctypes.data_as(_i64p),
                                 off.ctypes.data_as(_i64p)))
        return {"keys": keys[:ns * kl].reshape(ns, kl), "block": blk[:ns], "row_off": ro[:ns], "col_off": co[:ns],
                "extents": ext[:ns * 8].reshape(ns, 8), "offset": off[:ns]}


# ---------------------------------------------------------------------- calls
def tk_space_create(kind, labels, degeneracies, is_dual=False):
    labels = np.asarray(labels, dtype=np.int32)
    n = len(degeneracies)
    lab, lp = _i32(labels)
    deg = np.ascontiguousarray(np.asarray(degeneracies, dtype=np.int64))
    h = _p()
    _check(_space_create(kind.encode(), n, lp, deg.ctypes.data_as(_i64p), int(bool(is_dual)), ctypes.byref(h)))
    return Space(h.value)


def tk_space_parse(text):
    h = _p()
    _check(_space_parse(text.encode(), ctypes.byref(h)))
    return Space(h.value)


def tk_tensor_create(dtype, cod, dom):
    cod_arr = (_p * max(len(cod), 1))(*[s.h for s in cod])
    dom_arr = (_p * max(len(dom), 1))(*[s.h for s in dom])
    h = _p()
    _check(_tensor_create(dtype, len(cod), cod_arr, len(dom), dom_arr, ctypes.byref(h)))
    return Tensor(h.value)


def tk_contract_output(A, labA, B, labB, labC, n_cod_C):
    a, ap = _labels(A, labA, "labA")
    b, bp = _labels(B, labB, "labB")
    c, cp = _i32(labC)
    h = _p()
    _check(_contract_output(A.h, ap, B.h, bp, cp, n_cod_C, ctypes.byref(h)))
    return Tensor(h.value)


def tk_permute_workspace(A, p, q, C):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    n = ctypes.c_size_t()
    _check(_permute_workspace(A.h, pp, len(p), qp, len(q), C.h, ctypes.byref(n)))
    return n.value


def tk_permute(A, a, p, q, C, c, alpha=1.0, beta=0.0, ws=None, ws_bytes=0, stream=None):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    _check(_permute(A.h, _data(A, a, "a"), pp, len(p), qp, len(q), C.h, _data(C, c, "c"), float(alpha), float(beta),
                    _ws(ws, ws_bytes), ws_bytes, _stream(stream)))


def tk_permute_transfer(A, p, q, C):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    na, nc = A.info()["n_subblocks"], C.info()["n_subblocks"]
    out = np.zeros((na, nc))
    _check(_permute_transfer(A.h, pp, len(p), qp, len(q), C.h, out.ctypes.data_as(_dp)))
    return out


def tk_permute_transfer_planar(A, p, q, C, kappa_mode=-1):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    na, nc = A.info()["n_subblocks"], C.info()["n_subblocks"]
    out = np.zeros((na, nc))
    _check(_permute_transfer_planar(A.h, pp, len(p), qp, len(q), C.h, int(kappa_mode), out.ctypes.data_as(_dp)))
    return out


def tk_contract_workspace(A, labA, B, labB, C, labC):
    a, ap = _labels(A, labA, "labA")
    b, bp = _labels(B, labB, "labB")
    c, cp = _labels(C, labC, "labC")
    n = ctypes.c_size_t()
    _check(_contract_workspace(A.h, ap, B.h, bp, C.h, cp, ctypes.byref(n)))
    return n.value


def tk_contract(A, a, labA, B, b, labB, C, c, labC, alpha=1.0, beta=0.0, ws=None, ws_bytes=0, conjA=False,
                conjB=False, stream=None):
    la, ap = _labels(A, labA, "labA")
    lb, bp = _labels(B, labB, "labB")
    lc, cp = _labels(C, labC, "labC")
    _check(_contract(A.h, _data(A, a, "a"), ap, int(conjA), B.h, _data(B, b, "b"), bp, int(conjB), C.h,
                     _data(C, c, "c"), cp, float(alpha), float(beta), _ws(ws, ws_bytes), ws_bytes, _stream(stream)))


def tk_contract2_workspace(A, labA, B1, labB1, T, labT, B2, labB2, C, labC, want_fused=False):
    """Workspace bytes of tk_contract2 (and, with want_fused, whether the pair runs as one kernel)."""
    ls = [_labels(x, l, w) for x, l, w in ((A, labA, "labA"), (B1, labB1, "labB1"), (T, labT, "labT"),
                                           (B2, labB2, "labB2"), (C, labC, "labC"))]
    n = ctypes.c_size_t()
    f = ctypes.c_int32(0)
    _check(_contract2_workspace(A.h, ls[0][1], B1.h, ls[1][1], T.h, ls[2][1], B2.h, ls[3][1], C.h, ls[4][1],
                                ctypes.byref(n), ctypes.cast(ctypes.byref(f), _i32p)))
    return (n.value, bool(f.value)) if want_fused else n.value


def tk_contract2(A, a, labA, B1, b1, labB1, T, labT, B2, b2, labB2, C, c, labC, alpha=1.0, beta=0.0, ws=None,
                 ws_bytes=0, stream=None):
    """C = alpha ((A B1 -> T) B2) + beta C: two tk_contract calls, fused into one kernel when both are
    gathered skinny steps (include/tk.h). T is a descriptor only."""
    ls = [_labels(x, l, w) for x, l, w in ((A, labA, "labA"), (B1, labB1, "labB1"), (T, labT, "labT"),
                                           (B2, labB2, "labB2"), (C, labC, "labC"))]
    _check(_contract2(A.h, _data(A, a, "a"), ls[0][1], B1.h, _data(B1, b1, "b1"), ls[1][1], T.h, ls[2][1], B2.h,
                      _data(B2, b2, "b2"), ls[3][1], C.h, _data(C, c, "c"), ls[4][1], float(alpha), float(beta),
                      _ws(ws, ws_bytes), ws_bytes, _stream(stream)))


def _tuples(pA, qA, pB, qB, pAB, qAB):
    parts = [list(map(int, x)) for x in (pA, qA, pB, qB, pAB, qAB)]
    flat = [x for part in parts for x in part]
    t, tp = _i32(flat if flat else [0])
    n, np_ = _i32([len(x) for x in parts])
    return (t, n), tp, np_


def tk_contract_tuples_output(A, pA, qA, B, pB, qB, pAB, qAB):
    keep, tp, np_ = _tuples(pA, qA, pB, qB, pAB, qAB)
    h = _p()
    _check(_contract_tuples_output(A.h, B.h, tp, np_, ctypes.byref(h)))
    return Tensor(h.value)


def tk_contract_tuples_workspace(A, pA, qA, B, pB, qB, C, pAB, qAB):
    keep, tp, np_ = _tuples(pA, qA, pB, qB, pAB, qAB)
    n = ctypes.c_size_t()
    _check(_contract_tuples_workspace(A.h, B.h, C.h, tp, np_, ctypes.byref(n)))
    return n.value


def tk_contract_tuples(A, a, pA, qA, B, b, pB, qB, C, c, pAB, qAB, alpha=1.0, beta=0.0, ws=None, ws_bytes=0,
                       conjA=False, conjB=False, stream=None):
    """Alg. 4 with explicit tuples (include/tk.h): C = alpha permute(permute(A,(pA,qA)) o permute(B,(pB,qB)),
    (pAB,qAB)) + beta C."""
    keep, tp, np_ = _tuples(pA, qA, pB, qB, pAB, qAB)
    _check(_contract_tuples(A.h, _data(A, a, "a"), int(conjA), B.h, _data(B, b, "b"), int(conjB), C.h,
                            _data(C, c, "c"), tp, np_, float(alpha), float(beta), _ws(ws, ws_bytes), ws_bytes,
                            _stream(stream)))


def _ncon_args(tensors, labels, order):
    n = len(tensors)
    th = (_p * n)(*[t.h for t in tensors])
    labs = [_i32(l if len(l) else [0]) for l in labels]
    lp = (_i32p * n)(*[x[1] for x in labs])
    o, op = _i32(order if len(order) else [0])
    return n, th, lp, (labs, o), op, len(order)


def tk_ncon_output(tensors, labels, order, n_cod_out):
    """ncon network output HomSpace (include/tk.h): labels per tensor, > 0 contracted, -1..-m open."""
    n, th, lp, keep, op, no = _ncon_args(tensors, labels, order)
    h = _p()
    _check(_ncon_output(n, ctypes.cast(th, _p), ctypes.cast(lp, _p), op, no, n_cod_out, ctypes.byref(h)))
    return Tensor(h.value)


def tk_ncon_workspace(tensors, labels, order, n_cod_out):
    n, th, lp, keep, op, no = _ncon_args(tensors, labels, order)
    b = ctypes.c_size_t()
    _check(_ncon_workspace(n, ctypes.cast(th, _p), ctypes.cast(lp, _p), op, no, n_cod_out, ctypes.byref(b)))
    return b.value


def tk_ncon(tensors, datas, labels, order, n_cod_out, C, c, alpha=1.0, beta=0.0, ws=None, ws_bytes=0, stream=None):
    for i, (t, l) in enumerate(zip(tensors, labels)):
        _labels(t, l, f"labels[{i}]")
    n, th, lp, keep, op, no = _ncon_args(tensors, labels, order)
    dp = (_p * n)(*[_data(t, x, f"datas[{i}]") for i, (t, x) in enumerate(zip(tensors, datas))])
    _check(_ncon(n, ctypes.cast(th, _p), ctypes.cast(dp, _p), ctypes.cast(lp, _p), op, no, n_cod_out, C.h,
                 _data(C, c, "c"), float(alpha), float(beta), _ws(ws, ws_bytes), ws_bytes, _stream(stream)))


def tk_profile_enable(on=True):
    _check(_profile_enable(int(bool(on))))


def tk_phase_times():
    ms = (ctypes.c_float * 4)()
    by = (ctypes.c_double * 4)()
    fl = ctypes.c_double()
    _check(_phase_times(ms, by, ctypes.byref(fl)))
    return list(ms), list(by), fl.value


def tk_last_launch_count():
    return int(_last_launch_count())


def tk_contract_roofline(A, labA, B, labB, C, labC, peak_flops, peak_bytes_per_s):
    """{flops, gemm_bytes, permute_bytes, seconds} of one tk_contract (include/tk.h)."""
    a, ap = _labels(A, labA, "labA")
    b, bp = _labels(B, labB, "labB")
    c, cp = _labels(C, labC, "labC")
    out = (ctypes.c_double * 4)()
    _check(_contract_roofline(A.h, ap, B.h, bp, C.h, cp, float(peak_flops), float(peak_bytes_per_s), out))
    return {"flops": out[0], "gemm_bytes": out[1], "permute_bytes": out[2], "seconds": out[3]}


def tk_dmma_probe(blocks, iters, stream=None):
    """Launch the FP64 tensor-pipe probe; returns its flop count (time it with CUDA events)."""
    f = ctypes.c_double()
    _check(_dmma_probe(int(blocks), int(iters), _stream(stream), ctypes.byref(f)))
    return f.value


def tk_fsymbol(kind, a, b, c, d, e, f):
    args = [_i32(x) for x in (a, b, c, d, e, f)]
    out = ctypes.c_double()
    _check(_fsymbol(kind.encode(), *[x[1] for x in args], ctypes.byref(out)))
    return out.value


def tk_rsymbol(kind, a, b, c):
    args = [_i32(x) for x in (a, b, c)]
    out = ctypes.c_double()
    _check(_rsymbol(kind.encode(), *[x[1] for x in args], ctypes.byref(out)))
    return out.value


def tk_svd_workspace(A, p, q):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    n = ctypes.c_size_t()
    _check(_svd_workspace(A.h, pp, len(p), qp, len(q), ctypes.byref(n)))
    return n.value


def tk_svd(A, a, p, q, ws, ws_bytes, stream=None):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    _check(_svd(A.h, _data(A, a, "a"), pp, len(p), qp, len(q), _ws(ws, ws_bytes), ws_bytes, _stream(stream)))


def tk_svd_spectrum(A, p, q, ws, stream=None):
    """Per-block singular values (host), blocks in the order of permute(A, (p, q))."""
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    nb = ctypes.c_int32()
    _check(_svd_spectrum(A.h, pp, len(p), qp, len(q), _ptr(ws), _stream(stream), ctypes.byref(nb), None, None))
    counts = np.zeros(max(nb.value, 1), np.int64)
    _check(_svd_spectrum(A.h, pp, len(p), qp, len(q), _ptr(ws), _stream(stream), None,
                         counts.ctypes.data_as(_i64p), None))
    sig = np.zeros(max(int(counts[:nb.value].sum()), 1))
    _check(_svd_spectrum(A.h, pp, len(p), qp, len(q), _ptr(ws), _stream(stream), None, None,
                         sig.ctypes.data_as(_dp)))
    out, o = [], 0
    for k in counts[:nb.value]:
        out.append(sig[o:o + k].copy())
        o += k
    return out


def tk_svd_truncate(A, p, q, ws, max_dim=0, rel_tol=0.0, stream=None):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    w, u, s, vh = _p(), _p(), _p(), _p()
    err, nrm = ctypes.c_double(), ctypes.c_double()
    _check(_svd_truncate(A.h, pp, len(p), qp, len(q), _ptr(ws), int(max_dim), float(rel_tol), _stream(stream),
                         ctypes.byref(w), ctypes.byref(u), ctypes.byref(s), ctypes.byref(vh), ctypes.byref(err),
                         ctypes.byref(nrm)))
    return Space(w.value), Tensor(u.value), Tensor(s.value), Tensor(vh.value), err.value, nrm.value


def tk_svd_extract(A, p, q, ws, U, u, S, s, Vh, vh, stream=None):
    pa, pp = _i32(p)
    qa, qp = _i32(q)
    _check(_svd_extract(A.h, pp, len(p), qp, len(q), _ptr(ws), U.h, _data(U, u, "u"), S.h, _data(S, s, "s"), Vh.h,
                        _data(Vh, vh, "vh"), _stream(stream)))


def _trace_args(pt, qt, p, q):
    a = [_i32(x) for x in (pt, qt, p, q)]
    return a, (a[0][1], a[1][1], len(pt), a[2][1], len(p), a[3][1], len(q))


def tk_trace_output(A, pt, qt, p, q):
    keep, args = _trace_args(pt, qt, p, q)
    h = _p()
    _check(_trace_output(A.h, *args, ctypes.byref(h)))
    return Tensor(h.value)


def tk_trace_workspace(A, pt, qt, p, q, C):
    keep, args = _trace_args(pt, qt, p, q)
    n = ctypes.c_size_t()
    _check(_trace_workspace(A.h, *args, C.h, ctypes.byref(n)))
    return n.value


def tk_trace(A, a, pt, qt, p, q, C, c, alpha=1.0, beta=0.0, ws=None, ws_bytes=0, stream=None):
    keep, args = _trace_args(pt, qt, p, q)
    _check(_trace(A.h, _data(A, a, "a"), *args, C.h, _data(C, c, "c"), float(alpha), float(beta), _ws(ws, ws_bytes),
                  ws_bytes, _stream(stream)))


def tk_trace_transfer(A, pt, qt, p, q, C):
    keep, args = _trace_args(pt, qt, p, q)
    out = np.zeros((A.info()["n_subblocks"], C.info()["n_subblocks"]))
    _check(_trace_transfer(A.h, *args, C.h, out.ctypes.data_as(_dp)))
    return out


def tk_cache_clear():
    _cache_clear()


def tk_cache_size():
    return int(_cache_size())


def tk_version():
    return _version().decode()


def tk_last_error():
    return _lib_tk_last_error().decode()


# ------------------------------------------------------------ marshalling helpers
def space_from_spec(spec):
    """tk_space from a workloads/configs.py space dict (argument marshalling)."""
    labels = [list(l) for l, _ in spec["sectors"]]
    degs = [d for _, d in spec["sectors"]]
    return tk_space_create(spec["kind"], labels, degs, spec["dual"])


def tensor_from_spec(spec, dtype=TK_F64):
    cod = [space_from_spec(s) for s in spec["cod"]]
    dom = [space_from_spec(s) for s in spec["dom"]]
    return tk_tensor_create(dtype, cod, dom)
