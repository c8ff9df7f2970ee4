"""CPU oracle for arXiv 2506.15174 ESC SpMM -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2506_15174_b200``) never imports it, and it never imports
the product path.  See ``escs_oracle.c`` for the definitions and citations.

Parity status: ``spmm`` and ``partition`` are both pinned (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "escs_oracle.c")
# ESCS_ORACLE_LIB: a prebuilt oracle library to load instead (tests/test_oracle_mutants.py
# points it at deliberately broken copies to show the pins catch them)
_LIB_OVERRIDE = os.environ.get("ESCS_ORACLE_LIB")
_LIB = _LIB_OVERRIDE or os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

PLAN_HEADER_FIELDS = ("version", "m", "k", "nnz", "bCols", "h", "T",
                      "nP", "NG", "G", "n_items")


_FLAGS = ["-O3", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O3, no FMA contraction, OpenMP over
    rows only; portable: this library travels to other hosts)."""
    if _LIB_OVERRIDE:
        return _LIB
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc"] + _FLAGS + ["-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def use_native() -> str:
    """bench.py's cpu_baseline: the same source built -O3 -march=native on the
    host that runs it (the oracle timed as a tuned C build) and
    loaded in place of the portable library for this process.  Returns the
    library path.  The arithmetic is unchanged: fp64 sums in CSR order, no FMA
    contraction (and every fp32 x fp32 product is exact in fp64 anyway)."""
    global _lib
    path = os.path.join(_HERE, f"liboracle_native_{os.uname().nodename}.so")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc"] + _FLAGS + ["-march=native", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, path)
    with _lock:
        _lib = None
    os.environ["ESCS_ORACLE_LIB"] = path
    globals()["_LIB"] = path
    return path


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if _LIB == os.path.join(_HERE, "liboracle.so"):
                build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, i32 = ctypes.c_int64, ctypes.c_int32
            lib.oracle_spmm.argtypes = [i64, i64, i32, P, P, P, P, P, i64, P, P, P, i32]
            lib.oracle_spmm.restype = ctypes.c_int
            lib.oracle_partition.argtypes = [i64, i64, i64, P, P, i32, i32, i32, P,
                                             P, P, P, P, P, P, P, P, P, i64, i64]
            lib.oracle_partition.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def spmm(m, k, rowptr, colidx, vals, B, rows=None, with_absum=False, nthreads=0):
    """fp64 CSR x dense in CSR order (Listing 1).

    Returns C (fp64), or (C, absum, nterms) when ``with_absum``.
    ``rows`` selects a subset of output rows (sampled checks at full size)."""
    lib = _load()
    rowptr = _c(rowptr, np.int32)
    colidx = _c(colidx, np.int32)
    vals = _c(vals, np.float32)
    B = _c(B, np.float32)
    ncols = int(B.shape[1]) if B.ndim == 2 else int(B.size // max(k, 1))
    if rows is not None:
        rows = _c(rows, np.int64)
        nout = rows.size
    else:
        nout = m
    C = np.empty((nout, ncols), np.float64)
    absum = np.empty((nout, ncols), np.float64) if with_absum else None
    nterms = np.empty(nout, np.int32) if with_absum else None
    rc = lib.oracle_spmm(m, k, ncols, _ptr(rowptr), _ptr(colidx), _ptr(vals), _ptr(B),
                         _ptr(rows), nout if rows is not None else 0,
                         _ptr(C), _ptr(absum), _ptr(nterms), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_spmm: malformed CSR")
    if with_absum:
        return C, absum, nterms
    return C


def partition(m, k, rowptr, colidx, h, T, bCols=0):
    """Reference enumeration plan (paper's dense-scan dataTransformer).

    Returns a dict with 'header' (dict) and the nine plan arrays as int32."""
    lib = _load()
    rowptr = _c(rowptr, np.int32)
    colidx = _c(colidx, np.int32)
    nnz = int(rowptr[-1])
    nP = (m + h - 1) // h
    cap_groups = min(nP * ((1 << h) - 1), max(nnz, 0)) + 1
    cap_items = nP + nnz + 1
    hdr = np.zeros(11, np.int32)
    a = {
        "grp_panel": np.zeros(cap_groups, np.int32),
        "grp_mask": np.zeros(cap_groups, np.int32),
        "grp_col_ptr": np.zeros(cap_groups + 1, np.int32),
        "grp_val_ptr": np.zeros(cap_groups + 1, np.int32),
        "gcol": np.zeros(max(nnz, 1), np.int32),
        "slot_src": np.zeros(max(nnz, 1), np.int32),
        "item_panel": np.zeros(cap_items, np.int32),
        "item_group_begin": np.zeros(cap_items, np.int32),
        "item_gcol_ptr": np.zeros(cap_items + 1, np.int32),
    }
    rc = lib.oracle_partition(m, k, nnz, _ptr(rowptr), _ptr(colidx), int(bCols), int(h), int(T),
                              _ptr(hdr), *[_ptr(a[n]) for n in a], cap_groups, cap_items)
    if rc != 0:
        raise ValueError(f"oracle_partition failed rc={rc}")
    header = dict(zip(PLAN_HEADER_FIELDS, (int(x) for x in hdr)))
    NG, G, NI = header["NG"], header["G"], header["n_items"]
    out = {
        "header": header,
        "grp_panel": a["grp_panel"][:NG].copy(),
        "grp_mask": a["grp_mask"][:NG].copy(),
        "grp_col_ptr": a["grp_col_ptr"][:NG + 1].copy(),
        "grp_val_ptr": a["grp_val_ptr"][:NG + 1].copy(),
        "gcol": a["gcol"][:G].copy(),
        "slot_src": a["slot_src"][:nnz].copy(),
        "item_panel": a["item_panel"][:NI].copy(),
        "item_group_begin": a["item_group_begin"][:NI].copy(),
        "item_gcol_ptr": a["item_gcol_ptr"][:NI + 1].copy(),
    }
    return out


PLAN_ARRAYS = ("grp_panel", "grp_mask", "grp_col_ptr", "grp_val_ptr", "gcol", "slot_src",
               "item_panel", "item_group_begin", "item_gcol_ptr")
