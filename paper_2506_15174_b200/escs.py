"""Thin ctypes binding over libescs.so (include/escs.h) -- marshalling only.

Every step of the hot path runs inside the library: the host planner and the
sm_100a kernel.  There is no Python or CPU fallback: if ``libescs.so`` is
missing this module raises at import time.  torch is used only to hand over
device pointers and the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESCS_LIB") or os.path.join(_HERE, "libescs.so")   # ESCS_LIB: A/B experiments

ESCS_OK, ESCS_ERR_ARG, ESCS_ERR_CSR, ESCS_ERR_UNSUPPORTED, ESCS_ERR_OOM, ESCS_ERR_CUDA, \
    ESCS_ERR_INTERNAL = range(7)
HEADER_FIELDS = ("version", "m", "k", "nnz", "bCols", "h", "T", "nP", "NG", "G", "n_items")
PLAN_ARRAYS = ("grp_panel", "grp_mask", "grp_col_ptr", "grp_val_ptr", "gcol", "slot_src",
               "item_panel", "item_group_begin", "item_gcol_ptr")
EXPORTED_SYMBOLS = ("escs_plan", "escs_plan_ex", "escs_spmm", "escs_free", "escs_last_error",
                    "escs_plan_export", "escs_plan_info", "escs_gather_probe", "escs_version",
                    "escs_pack", "escs_spmm_packed", "escs_spmm_scatter", "escs_spmm_group",
                    "escs_gather_probe_packed", "escs_staged_export", "escs_plan_part")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libescs.so not found at {LIB_PATH}: build it with "
                      "`python -m paper_2506_15174_b200.build` (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)


class _Params(ctypes.Structure):
    _fields_ = [("ufi", ctypes.c_int32), ("T", ctypes.c_int32), ("host_only", ctypes.c_int32),
                ("cta_warps", ctypes.c_int32), ("variant", ctypes.c_int32), ("ufk", ctypes.c_int32),
                ("nthreads", ctypes.c_int32), ("autotune", ctypes.c_int32),
                ("colf", ctypes.c_int32), ("tile_order", ctypes.c_int32),
                ("packed", ctypes.c_int32), ("staged", ctypes.c_int32), ("st_warps", ctypes.c_int32),
                ("st_npw", ctypes.c_int32), ("st_nsplit", ctypes.c_int32), ("st_kb", ctypes.c_int32),
                ("hybrid_rows", ctypes.c_int32), ("carveout", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class _StagedView(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n_cta", "n_stage", "n_rec", "hs", "nslot", "max_k",
                                              "max_rec", "max_stages")] + \
               [(n, ctypes.POINTER(ctypes.c_int32)) for n in ("cta", "stage", "hdr", "src")]


class _View(ctypes.Structure):
    _fields_ = [("header", ctypes.c_int32 * 11)] + \
               [(n, ctypes.POINTER(ctypes.c_int32)) for n in PLAN_ARRAYS]


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("h", "T", "bcols", "variant", "cta_warps", "ufk",
                                              "n_tiles", "n_heavy", "n_split_items", "device")] + \
               [(n, ctypes.c_int64) for n in ("nP", "NG", "G", "n_items", "nnz", "device_bytes",
                                              "workspace_bytes")] + \
               [("plan_seconds", ctypes.c_double), ("ctas_per_sm", ctypes.c_int32),
                ("autotuned", ctypes.c_int32), ("colf", ctypes.c_int32),
                ("tile_order", ctypes.c_int32), ("pdl", ctypes.c_int32), ("packed", ctypes.c_int32),
                ("packed_words", ctypes.c_int64)] + \
               [(n, ctypes.c_int32) for n in ("staged", "st_ctas", "st_warps", "st_npw", "st_nsplit",
                                              "st_kb", "st_smem_bytes", "st_launches", "carveout", "hybrid_rows")]


_vp, _i64, _i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
_lib.escs_plan.argtypes = [_i64, _i64, _i64, _vp, _vp, _i32]
_lib.escs_plan.restype = _vp
_lib.escs_plan_ex.argtypes = [_i64, _i64, _i64, _vp, _vp, _i32, ctypes.POINTER(_Params)]
_lib.escs_plan_ex.restype = _vp
_lib.escs_spmm.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.escs_spmm.restype = ctypes.c_int
_lib.escs_spmm_packed.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.escs_spmm_group.restype = _i32
_lib.escs_spmm_group.argtypes = [_i32, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), _vp]
_lib.escs_spmm_packed.restype = ctypes.c_int
_lib.escs_spmm_scatter.argtypes = [_vp, _vp, _vp, ctypes.POINTER(ctypes.c_void_p), _i32, _i64,
                                   ctypes.c_uint32, _vp]
_lib.escs_spmm_scatter.restype = ctypes.c_int
_lib.escs_pack.argtypes = [_vp, _vp, _vp, _vp]
_lib.escs_pack.restype = ctypes.c_int
_lib.escs_gather_probe.argtypes = [_vp, _vp, _vp, _vp]
_lib.escs_gather_probe.restype = ctypes.c_int
_lib.escs_gather_probe_packed.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.escs_gather_probe_packed.restype = ctypes.c_int
_lib.escs_free.argtypes = [_vp]
_lib.escs_free.restype = None
_lib.escs_last_error.argtypes = [ctypes.POINTER(ctypes.c_char_p)]
_lib.escs_last_error.restype = ctypes.c_int
_lib.escs_plan_export.argtypes = [_vp, ctypes.POINTER(_View)]
_lib.escs_plan_export.restype = ctypes.c_int
_lib.escs_plan_info.argtypes = [_vp, ctypes.POINTER(_Stats)]
_lib.escs_plan_info.restype = ctypes.c_int
_lib.escs_plan_part.argtypes = [_vp, _i32]
_lib.escs_plan_part.restype = _vp
_lib.escs_staged_export.argtypes = [_vp, ctypes.POINTER(_StagedView)]
_lib.escs_staged_export.restype = ctypes.c_int
_lib.escs_version.argtypes = []
_lib.escs_version.restype = ctypes.c_char_p


class EscsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"escs error {code}: {msg}")
        self.code = code


def escs_last_error():
    msg = ctypes.c_char_p()
    code = _lib.escs_last_error(ctypes.byref(msg))
    return code, (msg.value or b"").decode()


def _raise_last():
    code, msg = escs_last_error()
    raise EscsError(code, msg)


def escs_version() -> str:
    return _lib.escs_version().decode()


class Plan:
    """Owns an escs_plan_t; freed on close() / garbage collection."""

    def __init__(self, handle, m, k, nnz, bcols, owner=None):
        self.handle = handle
        self.m, self.k, self.nnz, self.bcols = m, k, nnz, bcols
        self._owner = owner   # a hybrid plan's part borrows its container's memory

    def close(self):
        if self.handle:
            if self._owner is None:
                _lib.escs_free(self.handle)
            self.handle = None

    def part(self, i):
        """Part i of a hybrid plan (escs_plan_part), or None."""
        h = _lib.escs_plan_part(self.handle, int(i))
        if not h:
            return None
        s = _Stats()
        _lib.escs_plan_info(h, ctypes.byref(s))
        return Plan(h, 0, self.k, int(s.nnz), self.bcols, owner=self)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def info(self):
        return escs_plan_info(self)

    def export(self):
        return escs_plan_export(self)


def _csr_args(rowptr, colidx):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    return rowptr, colidx


def escs_plan(m, k, nnz, rowptr, colidx, bCols) -> Plan:
    """Enumerate A's pattern and upload the plan (host int32 CSR arrays)."""
    rowptr, colidx = _csr_args(rowptr, colidx)
    h = _lib.escs_plan(int(m), int(k), int(nnz), rowptr.ctypes.data, colidx.ctypes.data,
                       int(bCols))
    if not h:
        _raise_last()
    return Plan(h, int(m), int(k), int(nnz), int(bCols))


def escs_plan_ex(m, k, nnz, rowptr, colidx, bCols, *, ufi=0, T=0, host_only=0, cta_warps=0,
                 variant=0, ufk=0, nthreads=0, autotune=0, colf=0, tile_order=0, packed=0,
                 staged=0, st_warps=0, st_npw=0, st_nsplit=0, st_kb=0, hybrid_rows=0, carveout=0) -> Plan:
    """escs_plan with explicit escs_params (include/escs.h); 0 = auto for every
    field.  autotune: 1 = latency objective (one stream), 2 = concurrent
    throughput objective (independent SpMMs overlapped on several streams).
    packed=1: plan (and tune, including UFi) for escs_pack + escs_spmm_packed.
    staged: 0 auto, 1 L2-gather record walk, 2 staged walk (B rows in shared
    memory); st_*: its tile parameters (0 = auto).  hybrid_rows: 0 auto, -1
    off, X > 0 a hybrid plan of the X longest rows + the rest (escs_plan_part)."""
    rowptr, colidx = _csr_args(rowptr, colidx)
    p = _Params(int(ufi), int(T), int(host_only), int(cta_warps), int(variant), int(ufk),
                int(nthreads), int(autotune), int(colf), int(tile_order), int(packed),
                int(staged), int(st_warps), int(st_npw), int(st_nsplit), int(st_kb), int(hybrid_rows),
                int(carveout), (ctypes.c_int32 * 1)())
    h = _lib.escs_plan_ex(int(m), int(k), int(nnz), rowptr.ctypes.data, colidx.ctypes.data,
                          int(bCols), ctypes.byref(p))
    if not h:
        _raise_last()
    return Plan(h, int(m), int(k), int(nnz), int(bCols))


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def escs_spmm(plan: Plan, vals, B, C, stream=None) -> None:
    """C = A x B on `stream` (default: torch's current stream).  vals/B/C are
    device torch tensors (fp32, contiguous) or raw device pointers (int)."""
    for t in (vals, B, C):
        if t is not None and not isinstance(t, int):
            if not t.is_cuda or t.dtype.itemsize != 4 or not t.is_contiguous():
                raise EscsError(ESCS_ERR_ARG, "vals, B, C must be contiguous fp32 CUDA tensors")
    if not isinstance(B, int) and B.numel() != plan.k * plan.bcols:
        raise EscsError(ESCS_ERR_ARG, f"B must have k*bCols = {plan.k * plan.bcols} elements")
    if not isinstance(C, int) and C.numel() != plan.m * plan.bcols:
        raise EscsError(ESCS_ERR_ARG, f"C must have m*bCols = {plan.m * plan.bcols} elements")
    if vals is not None and not isinstance(vals, int) and vals.numel() < plan.nnz:
        raise EscsError(ESCS_ERR_ARG, f"vals must have at least nnz = {plan.nnz} elements")
    rc = _lib.escs_spmm(plan.handle, _ptr(vals), _ptr(B), _ptr(C), _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()


class Group:
    """Marshalled argument arrays of one escs_spmm_group call (built once,
    reused every call: the C ABI reads them on the host at enqueue time)."""

    def __init__(self, plans, vals, B, C):
        n = len(plans)
        if not (len(vals) == len(B) == len(C) == n):
            raise EscsError(ESCS_ERR_ARG, "plans, vals, B and C must have the same length")
        for pl, v, b, c in zip(plans, vals, B, C):
            for t in (v, b, c):
                if t is not None and not isinstance(t, int):
                    if not t.is_cuda or t.dtype.itemsize != 4 or not t.is_contiguous():
                        raise EscsError(ESCS_ERR_ARG, "vals, B, C must be contiguous fp32 CUDA tensors")
            if not isinstance(b, int) and b.numel() != pl.k * pl.bcols:
                raise EscsError(ESCS_ERR_ARG, f"B must have k*bCols = {pl.k * pl.bcols} elements")
            if not isinstance(c, int) and c.numel() != pl.m * pl.bcols:
                raise EscsError(ESCS_ERR_ARG, f"C must have m*bCols = {pl.m * pl.bcols} elements")
        arr = lambda xs: (ctypes.c_void_p * max(n, 1))(*[_ptr(x) for x in xs])
        self.n = n
        self.keep = (list(plans), list(vals), list(B), list(C))   # keep tensors alive
        self.plans = (ctypes.c_void_p * max(n, 1))(*[pl.handle for pl in plans])
        self.vals, self.B, self.C = arr(vals), arr(B), arr(C)

    def __call__(self, stream=None) -> None:
        rc = _lib.escs_spmm_group(self.n, self.plans, self.vals, self.B, self.C,
                                  _stream_ptr(stream))
        if rc != ESCS_OK:
            _raise_last()


def escs_spmm_group(plans, vals, B, C, stream=None) -> None:
    """C[i] = A_i x B[i] for independent problems, grouped into as few
    launches as possible (bitwise identical to separate escs_spmm calls)."""
    Group(plans, vals, B, C)(stream)


def escs_pack(plan: Plan, vals, packed=None, stream=None):
    """Write the plan's record stream (include/escs.h escs_pack) from the CSR
    values; allocates it (a torch int32 CUDA tensor of
    escs_plan_stats.packed_words) when `packed` is None.  Returns `packed`."""
    if packed is None:
        import torch
        dev = vals.device if not isinstance(vals, int) else torch.device("cuda")
        packed = torch.empty(max(int(plan.info["packed_words"]), 4), dtype=torch.int32, device=dev)
    elif not isinstance(packed, int) and packed.numel() < int(plan.info["packed_words"]):
        raise EscsError(ESCS_ERR_ARG, f"packed needs {plan.info['packed_words']} words")
    rc = _lib.escs_pack(plan.handle, _ptr(vals), _ptr(packed), _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()
    return packed


def escs_spmm_packed(plan: Plan, packed, B, C, stream=None) -> None:
    """C = A x B from the record stream written by escs_pack."""
    rc = _lib.escs_spmm_packed(plan.handle, _ptr(packed), _ptr(B), _ptr(C), _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()


ESCS_SCATTER_MULTICAST = 1


def escs_spmm_scatter(plan: Plan, vals, B, dsts, row_offset: int, stream=None,
                      multicast: bool = False) -> None:
    """Store C = A x B into every buffer of `dsts` (device tensors or raw
    pointers, e.g. the peers' symmetric-memory C) at rows row_offset + i;
    multicast=True: dsts is one NVLS multicast address."""
    arr = (ctypes.c_void_p * len(dsts))(*[_ptr(d) for d in dsts])
    rc = _lib.escs_spmm_scatter(plan.handle, _ptr(vals), _ptr(B), arr, len(dsts), int(row_offset),
                                ESCS_SCATTER_MULTICAST if multicast else 0, _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()


def escs_gather_probe(plan: Plan, B, sink, stream=None) -> None:
    rc = _lib.escs_gather_probe(plan.handle, _ptr(B), _ptr(sink), _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()


def escs_gather_probe_packed(plan: Plan, packed, B, sink, stream=None) -> None:
    rc = _lib.escs_gather_probe_packed(plan.handle, _ptr(packed), _ptr(B), _ptr(sink),
                                       _stream_ptr(stream))
    if rc != ESCS_OK:
        _raise_last()


def escs_free(plan: Plan) -> None:
    plan.close()


def escs_plan_export(plan: Plan) -> dict:
    v = _View()
    if _lib.escs_plan_export(plan.handle, ctypes.byref(v)) != ESCS_OK:
        _raise_last()
    hdr = dict(zip(HEADER_FIELDS, (int(x) for x in v.header)))
    NG, G, NI, nnz = hdr["NG"], hdr["G"], hdr["n_items"], hdr["nnz"]
    sizes = {"grp_panel": NG, "grp_mask": NG, "grp_col_ptr": NG + 1, "grp_val_ptr": NG + 1,
             "gcol": G, "slot_src": nnz, "item_panel": NI, "item_group_begin": NI,
             "item_gcol_ptr": NI + 1}
    out = {"header": hdr}
    for n in PLAN_ARRAYS:
        cnt = sizes[n]
        ptr = getattr(v, n)
        out[n] = np.ctypeslib.as_array(ptr, shape=(cnt,)).copy() if cnt else np.zeros(0, np.int32)
    return out


def escs_staged_export(plan: Plan) -> dict:
    """The staged walk's schedule (include/escs.h escs_staged_export) as numpy
    arrays: cta (n_cta x 4), stage (n_stage x 4), hdr (n_stage x hs), src."""
    v = _StagedView()
    if _lib.escs_staged_export(plan.handle, ctypes.byref(v)) != ESCS_OK:
        _raise_last()
    out = {n: int(getattr(v, n)) for n in ("n_cta", "n_stage", "n_rec", "hs", "nslot", "max_k",
                                           "max_rec", "max_stages")}

    def arr(name, cnt, shape):
        if not cnt:
            return np.zeros(shape if shape[0] == 0 else (0,), np.int32).reshape(shape)
        return np.ctypeslib.as_array(getattr(v, name), shape=(cnt,)).copy().reshape(shape)
    out["cta"] = arr("cta", 4 * out["n_cta"], (out["n_cta"], 4))
    out["stage"] = arr("stage", 4 * out["n_stage"], (out["n_stage"], 4))
    out["hdr"] = arr("hdr", out["hs"] * out["n_stage"], (out["n_stage"], out["hs"]))
    out["src"] = arr("src", out["n_rec"], (out["n_rec"],))
    return out


def escs_plan_info(plan: Plan) -> dict:
    s = _Stats()
    if _lib.escs_plan_info(plan.handle, ctypes.byref(s)) != ESCS_OK:
        _raise_last()
    return {n: getattr(s, n) for n, _ in _Stats._fields_}


def spmm(plan: Plan, vals, B, C=None, stream=None):
    """Convenience: allocate C if needed (torch), run escs_spmm, return C."""
    if C is None:
        import torch
        C = torch.empty((plan.m, plan.bcols), dtype=torch.float32, device=B.device)
    escs_spmm(plan, vals, B, C, stream)
    return C
