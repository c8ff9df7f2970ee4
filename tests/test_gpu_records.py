"""GPU parity of the packed-record walk (escs_pack + escs_spmm_packed, the
paper's data transformation ANNZ §3.3.3 P:455-493 and the enumerated
sparse-coarsened kernel §3.3 on it) against the fp64 oracle.

* The record stream escs_pack writes is checked word by word against a
  record stream rebuilt here from the canonical plan arrays (which are
  themselves byte-checked against the oracle partitioner in
  test_plan_parity.py / below) and the CSR values.
* C: bit-exact on dyadic twins (G1), within G2 on real values, and bitwise
  equal to escs_spmm on the CSR values for finite B (same per-lane FMA order).
"""
import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import synth

from test_gpu_parity import check_exact, check_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


RW = {1: 2, 2: 4, 3: 4, 4: 8, 6: 8, 8: 12}   # int32 words per record (include/escs.h escs_pack)


def expected_records(plan_export, vals, h):
    """Record stream from the canonical plan (include/escs.h escs_pack)."""
    gcol = plan_export["gcol"].astype(np.int64)
    G = len(gcol)
    rw = RW[h]
    shift = 27 if h <= 4 else 24
    out = np.zeros((G, rw), np.int32)
    if h == 1:
        out[:, 0] = gcol
        out[:, 1] = vals[plan_export["slot_src"]].view(np.int32)
        return out.ravel()
    cp, vp, mk = plan_export["grp_col_ptr"], plan_export["grp_val_ptr"], plan_export["grp_mask"]
    slot = plan_export["slot_src"]
    for g in range(len(mk)):
        rows = [r for r in range(h) if mk[g] >> r & 1]
        p = len(rows)
        for c in range(cp[g], cp[g + 1]):
            out[c, 0] = np.array([gcol[c] | (int(mk[g]) << shift)], np.uint32).view(np.int32)[0]
            base = vp[g] + (c - cp[g]) * p
            for q, r in enumerate(rows):
                out[c, 1 + r] = vals[slot[base + q]].view(np.int32)
    return out.ravel()


def run_packed(torch, A, B, **params):
    from paper_2506_15174_b200 import escs
    n = B.shape[1]
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, **params)
    dv = torch.from_numpy(A.vals).cuda() if A.nnz else torch.zeros(1, device="cuda")
    dB = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    pk = escs.escs_pack(pl, dv)
    C = torch.full((A.m, n), float("nan"), device="cuda")
    escs.escs_spmm_packed(pl, pk, dB, C)
    torch.cuda.synchronize()
    return C.cpu().numpy(), pl, pk, dv, dB


@pytest.mark.parametrize("ufi", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("n,colf", [(128, 4), (128, 8), (128, 16), (64, 4), (64, 8), (32, 4), (32, 8),
                                    (16, 4), (8, 4), (4, 4), (256, 8), (256, 16)])
def test_records_and_result(torch_cuda, ufi, n, colf):
    """Every UFi x lane map: the record stream word for word, C bitwise equal
    to the CSR-value walk, and against the oracle (G2 real values; G1 exact
    on the dyadic twin).  Ragged m (m mod UFi != 0), T = 24 (split panels and
    tail batches), 4-warp tiles (heavy panels through the workspace)."""
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    default_colf = {4: 4, 8: 4, 16: 4, 32: 4, 64: 4, 128: 4, 256: 8}[n]
    if ufi > 4 and not (n >= 32 and (colf == default_colf or (n, colf) == (128, 8))):
        pytest.skip("UFi 6/8 are built for the default lane maps of bCols 32..256 and 128/F8")
    A = synth.magnitude_pruned(387, 900, 0.8, 70 + ufi)
    B = synth.dense_b(900, n, 71)
    kw = dict(ufi=ufi, T=24, colf=colf, cta_warps=4, packed=1)
    C, pl, pk, dv, dB = run_packed(torch, A, B, **kw)
    info = pl.info
    assert info["h"] == ufi and info["colf"] == colf and info["packed"] == 1
    assert info["packed_words"] == (info["G"] * RW[ufi] + 3) // 4 * 4   # rounded to 16 bytes
    exp = expected_records(pl.export(), A.vals, ufi)
    assert np.array_equal(pk.cpu().numpy()[:len(exp)], exp)
    C_csr = torch.empty(A.m, n, device="cuda")
    if ufi <= 4:
        escs.escs_spmm(pl, dv, dB, C_csr)
        torch.cuda.synchronize()
    # same lane map -> same per-lane FMA order -> bitwise equal (the CSR walk
    # has the alternative coarsening factors at UFi = 1 only; a record-tuned
    # UFi > 1 plan runs escs_spmm on the default map, a different sum order;
    # the CSR walk stops at UFi 4)
    if ufi > 4:
        with pytest.raises(escs.EscsError):
            escs.escs_spmm(pl, dv, dB, C_csr)
    elif ufi == 1 or colf == default_colf:
        assert np.array_equal(C_csr.cpu().numpy(), C)
    else:
        check_tol(A, B, C_csr.cpu().numpy())
    check_tol(A, B, C)
    Ad, Bd = synth.dyadic_twin(A, n, 72)
    Cd, _, _, _, _ = run_packed(torch, Ad, Bd, **kw)
    check_exact(Ad, Bd, Cd)


@pytest.mark.parametrize("ufi", [1, 2, 3, 4, 6, 8])
def test_records_degenerate(torch_cuda, ufi):
    """Empty rows and panels, dense rows, one-column items (T = 1), nnz = 0
    (C pre-filled with NaN must come back all zero)."""
    cases = [synth.random_csr(301, 700, 9000, 8, empty_rows=(0, 1, 2, 3, 5, 300), dense_rows=(17, 200)),
             synth.random_csr(64, 64, 0, 9),
             synth.random_csr(33, 41, 300, 10)]
    for A0 in cases:
        for T in (1, 0):
            A, B = synth.dyadic_twin(A0, 128, 73)
            C, _, _, _, _ = run_packed(torch_cuda, A, B, ufi=ufi, T=T, packed=1)
            check_exact(A, B, C)


@pytest.mark.parametrize("autotune", [1, 2])
@pytest.mark.parametrize("shape", [(512, 4608, 0.7, 128), (2048, 512, 0.8, 64), (512, 2048, 0.95, 32)])
def test_packed_autotuned_plan_parity(torch_cuda, shape, autotune):
    """A packed-objective autotuned plan (the tuner also searches UFi 1..4,
    P:512-515) is the canonical plan of its (UFi, T) -- byte identical to the
    oracle partitioner given that header -- and exact on the dyadic twin; its
    workspace is clean after tuning (a second call gives the same C)."""
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    m, k, s, n = shape
    A0 = synth.magnitude_pruned(m, k, s, 74)
    A, B = synth.dyadic_twin(A0, n, 75)
    C, pl, pk, dv, dB = run_packed(torch, A, B, autotune=autotune, packed=1)
    info = pl.info
    assert info["autotuned"] in (1, 2) and info["packed"] == 1
    got = pl.export()
    ref = oracle.partition(A.m, A.k, A.rowptr, A.colidx, info["h"], info["T"], bCols=n)
    for nm in oracle.PLAN_ARRAYS:
        assert np.array_equal(got[nm], ref[nm]), nm
    check_exact(A, B, C)
    C2 = torch.empty(A.m, n, device="cuda")
    escs.escs_spmm_packed(pl, pk, dB, C2)
    torch.cuda.synchronize()
    assert np.array_equal(C2.cpu().numpy(), C)


def test_packed_probe_runs(torch_cuda):
    """escs_gather_probe_packed walks the same records and B rows (no FMAs)."""
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    A = synth.magnitude_pruned(512, 1024, 0.7, 76)
    B = synth.dense_b(1024, 128, 77)
    _, pl, pk, dv, dB = run_packed(torch, A, B, ufi=4, packed=1)
    info = pl.info
    sink = torch.zeros(info["n_tiles"] * 32 * info["cta_warps"], device="cuda")
    escs.escs_gather_probe_packed(pl, pk, dB, sink)
    torch.cuda.synchronize()
    assert torch.isfinite(sink).all()


def test_packed_rejects_scalar_and_misaligned(torch_cuda):
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    A = synth.magnitude_pruned(64, 96, 0.8, 78)
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 48, packed=1)   # scalar map
    dv = torch.from_numpy(A.vals).cuda()
    pk = escs.escs_pack(pl, dv)
    dB = torch.zeros(96, 48, device="cuda")
    C = torch.zeros(64, 48, device="cuda")
    with pytest.raises(escs.EscsError) as e:
        escs.escs_spmm_packed(pl, pk, dB, C)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED


@pytest.mark.parametrize("packed", [1, 0])
@pytest.mark.parametrize("n,T,W", [(128, 60, 12), (64, 17, 4), (32, 300, 16), (128, 1000, 8)])
def test_column_window_tiles_exact(torch_cuda, packed, n, T, W):
    """tile_order 3 (column windows: item j of W panels per CTA, split panels
    combined through per-item workspace slots and a per-panel counter): exact
    on the dyadic twin, bitwise stable across repeated calls (counters reset),
    ragged m, empty rows, panels with one item and with many."""
    from paper_2506_15174_b200 import escs
    A = synth.random_csr(333, 2000, 60000, 13, empty_rows=(0, 7, 332), dense_rows=(5,))
    Ad, Bd = synth.dyadic_twin(A, n, 9)
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=1, T=T, cta_warps=W, tile_order=3,
                           packed=packed)
    assert pl.info["tile_order"] == 3
    dv = torch_cuda.from_numpy(Ad.vals).cuda()
    dB = torch_cuda.from_numpy(Bd).cuda()
    pk = escs.escs_pack(pl, dv) if packed else None
    outs = []
    for _ in range(3):
        C = torch_cuda.full((A.m, n), float("nan"), device="cuda")
        if packed:
            escs.escs_spmm_packed(pl, pk, dB, C)
        else:
            escs.escs_spmm(pl, dv, dB, C)
        torch_cuda.cuda.synchronize()
        outs.append(C.cpu().numpy())
    check_exact(Ad, Bd, outs[0])
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
