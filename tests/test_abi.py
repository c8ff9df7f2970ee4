"""The C-ABI library loads, exports every symbol include/escs.h declares, and
reports argument/CSR errors as the header documents (no GPU compute here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2506_15174_b200 import escs, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "escs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(escs_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(escs.LIB_PATH)
    names = declared_functions()
    assert set(names) == set(escs.EXPORTED_SYMBOLS)
    for n in names:
        assert hasattr(lib, n), n


def test_version():
    assert "sm_100a" in escs.escs_version()


def test_kernels_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", escs.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def plan_err(*args, **kw):
    with pytest.raises(escs.EscsError) as e:
        escs.escs_plan_ex(*args, host_only=1, **kw)
    return e.value.code


def test_csr_errors():
    rp = np.array([0, 2, 3], np.int32)
    assert plan_err(2, 4, 3, rp, np.array([0, 1, 5], np.int32), 32) == escs.ESCS_ERR_CSR  # range
    assert plan_err(2, 4, 3, rp, np.array([1, 1, 0], np.int32), 32) == escs.ESCS_ERR_CSR  # dup
    assert plan_err(2, 4, 3, rp, np.array([1, 0, 0], np.int32), 32) == escs.ESCS_ERR_CSR  # unsorted
    assert plan_err(2, 4, 3, np.array([1, 2, 3], np.int32), np.array([0, 1, 2], np.int32), 32) \
        == escs.ESCS_ERR_CSR
    assert plan_err(2, 4, 3, np.array([0, 2, 1], np.int32), np.array([0, 1, 2], np.int32), 32) \
        == escs.ESCS_ERR_CSR
    code, msg = escs.escs_last_error()
    assert code == escs.ESCS_ERR_CSR and "row" in msg


def test_arg_errors():
    rp = np.array([0, 1], np.int32)
    ci = np.array([0], np.int32)
    assert plan_err(0, 1, 0, np.array([0], np.int32), ci, 32) == escs.ESCS_ERR_ARG
    assert plan_err(1, 1, 1, rp, ci, 0) == escs.ESCS_ERR_ARG
    assert plan_err(1, 1, 1, rp, ci, 300) == escs.ESCS_ERR_UNSUPPORTED
    assert plan_err(1, 1, 1, rp, ci, 32, ufi=17) == escs.ESCS_ERR_ARG
    assert plan_err(1, 1, 1, rp, ci, 32, cta_warps=17) == escs.ESCS_ERR_ARG
    assert plan_err(1 << 31, 1, 1, rp, ci, 32) == escs.ESCS_ERR_ARG


def test_host_only_plan_rejects_spmm():
    A = synth.config("c1").A
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 32, host_only=1)
    rc = escs._lib.escs_spmm(pl.handle, 16, 16, 16, None)
    assert rc == escs.ESCS_ERR_ARG
    assert "host-only" in escs.escs_last_error()[1]
    assert escs._lib.escs_spmm(None, 16, 16, 16, None) == escs.ESCS_ERR_ARG
    escs.escs_free(pl)
    escs._lib.escs_free(None)   # NULL is a no-op


def test_plan_info_and_auto_params():
    A = synth.magnitude_pruned(512, 512, 0.9, 5)
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, host_only=1)
    info = pl.info
    assert info["h"] == 1 and info["T"] >= 8 and info["device"] == -1   # 90% sparsity -> UFi 1
    assert info["nnz"] == A.nnz and info["n_tiles"] >= 1 and 1 <= info["cta_warps"] <= 16
    hdr = pl.export()["header"]
    assert hdr["T"] == info["T"] and hdr["bCols"] == 64


def test_env_params(monkeypatch):
    A = synth.config("c1").A
    monkeypatch.setenv("ESCS_PARAMS", "ufi=3,T=9,warps=5")
    info = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 32, host_only=1).info
    assert (info["h"], info["T"], info["cta_warps"]) == (3, 9, 5)


def test_tiles_cover_items():
    """CTA tiles (device-only schedule) cover every item exactly once; a
    panel's items never straddle a non-heavy tile boundary."""
    A = synth.power_law(1024, 1024, 0.98, 3)
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 128, ufi=4, T=16, cta_warps=4,
                           host_only=1)
    info = pl.info
    assert info["n_heavy"] > 0
    assert info["n_tiles"] >= -(-info["n_items"] // 4)


def test_params_out_of_range_rejected():
    """escs_plan_ex rejects out-of-range tuning parameters with ESCS_ERR_ARG
    (host-only plans: no GPU needed)."""
    import pytest
    from paper_2506_15174_b200 import escs, synth
    A = synth.random_csr(20, 30, 100, 1)
    for bad in ({"colf": 5}, {"tile_order": 4}, {"cta_warps": 17}, {"variant": 3},
                {"autotune": 3}, {"autotune": -1}):
        with pytest.raises(escs.EscsError) as e:
            escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 32, host_only=1, **bad)
        assert e.value.code == escs.ESCS_ERR_ARG
    for ok in ({"colf": 8}, {"tile_order": 2}, {"tile_order": 1}, {"tile_order": 3}):
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 32, host_only=1, **ok)
        assert pl.info["tile_order"] == ok.get("tile_order", pl.info["tile_order"]) and pl.info["tile_order"] in (1, 2, 3)
        pl.close()


def test_group_arg_errors_without_gpu():
    lib = ctypes.CDLL(escs.LIB_PATH)
    lib.escs_spmm_group.restype = ctypes.c_int32
    lib.escs_spmm_group.argtypes = [ctypes.c_int32] + [ctypes.c_void_p] * 5
    assert lib.escs_spmm_group(0, None, None, None, None, None) == escs.ESCS_OK
    assert lib.escs_spmm_group(-1, None, None, None, None, None) == escs.ESCS_ERR_ARG
    assert lib.escs_spmm_group(2, None, None, None, None, None) == escs.ESCS_ERR_ARG
    code, msg = escs.escs_last_error()
    assert code == escs.ESCS_ERR_ARG and "NULL" in msg


def test_packed_params_host_only():
    """escs_params.packed: 0/1 accepted (else ESCS_ERR_ARG); the plan reports it
    and the size of escs_pack's record stream (G records of 2/4/8/12 words by
    UFi, include/escs.h); tile widths up to 28 warps for the record walk, 16
    otherwise; host-only plans at UFi 6 and 8 are the canonical plans of the
    oracle partitioner."""
    import oracle
    A = synth.magnitude_pruned(97, 300, 0.8, 5)
    for bad in ({"packed": 2}, {"packed": -1}, {"cta_warps": 29, "packed": 1}, {"cta_warps": 17}):
        with pytest.raises(escs.EscsError) as e:
            escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, host_only=1, **bad)
        assert e.value.code == escs.ESCS_ERR_ARG
    words = {1: 2, 2: 4, 3: 4, 4: 8, 6: 8, 8: 12}
    for h, rw in words.items():
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, ufi=h, T=24, packed=1,
                               cta_warps=28, host_only=1)
        info = pl.info
        assert info["packed"] == 1 and info["h"] == h and info["cta_warps"] == 28
        assert info["packed_words"] == (rw * info["G"] + 3) // 4 * 4   # rounded to 16 bytes
        ref = oracle.partition(A.m, A.k, A.rowptr, A.colidx, h, 24, bCols=64)
        got = pl.export()
        for n in oracle.PLAN_ARRAYS:
            assert np.array_equal(got[n], ref[n]), (h, n)
