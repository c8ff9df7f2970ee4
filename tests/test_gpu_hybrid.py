"""GPU parity of hybrid plans (escs_params.hybrid_rows): the X longest rows of
A planned as their own matrix (part 0, rows in descending length order, ties
by row index) and the other rows in row order (part 1), each run by the packed
gather walk writing its rows of C through a row map.

Checked independently of the library's construction: the test derives the two
row sets itself, plans each sub-matrix with the oracle partitioner (the
paper's dense-scan dataTransformer) and compares the parts' canonical plans
byte for byte; C is compared with the fp64 oracle on the whole matrix (G2 on
real values, bit-exact on the dyadic twin).
"""
import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import escs, synth

from test_gpu_parity import check_exact, check_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def split_rows(A, X):
    lens = np.diff(A.rowptr)
    order = np.argsort(-lens, kind="stable")
    return order[:X], np.sort(order[X:])


def sub_csr(A, rows):
    lens = np.diff(A.rowptr)[rows]
    rp = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([A.colidx[A.rowptr[r]:A.rowptr[r + 1]] for r in rows]) if len(rows) else np.zeros(0, np.int32)
    return synth.CSR(len(rows), A.k, rp.astype(np.int32), ci.astype(np.int32), np.ones(len(ci), np.float32))


def run_hybrid(torch, A, B, **params):
    n = B.shape[1]
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, packed=1, **params)
    dv = torch.from_numpy(A.vals).cuda()
    pk = escs.escs_pack(pl, dv)
    C = torch.full((A.m, n), float("nan"), device="cuda")
    escs.escs_spmm_packed(pl, pk, torch.from_numpy(np.ascontiguousarray(B)).cuda(), C)
    torch.cuda.synchronize()
    return C.cpu().numpy(), pl


def check_parts(pl, A, X):
    heavy, light = split_rows(A, X)
    for q, rows in enumerate((heavy, light)):
        part = pl.part(q)
        got = part.export()
        S = sub_csr(A, rows)
        h, T = got["header"]["h"], got["header"]["T"]
        ref = oracle.partition(S.m, S.k, S.rowptr, S.colidx, h, T, bCols=got["header"]["bCols"])
        assert got["header"] == ref["header"], q
        for name in oracle.PLAN_ARRAYS:
            assert np.array_equal(got[name], ref[name]), (q, name)


@pytest.mark.parametrize("X,ufi", [(40, 8), (100, 4), (7, 2), (300, 8)])
def test_hybrid_powerlaw(torch_cuda, X, ufi):
    A = synth.power_law(1000, 1500, 0.97, 61)
    B = synth.dense_b(A.k, 128, 62)
    C, pl = run_hybrid(torch_cuda, A, B, hybrid_rows=X, ufi=ufi)
    info = pl.info
    assert info["hybrid_rows"] == X and info["h"] == ufi and info["nnz"] == A.nnz
    check_tol(A, B, C)
    check_parts(pl, A, X)
    Ad, Bd = synth.dyadic_twin(A, 128, 63)
    Cd, _ = run_hybrid(torch_cuda, Ad, Bd, hybrid_rows=X, ufi=ufi)
    check_exact(Ad, Bd, Cd)


@pytest.mark.parametrize("n", [32, 64])
def test_hybrid_ties_and_empty_rows(torch_cuda, n):
    """Equal-length rows (ties by row index), empty rows in both parts."""
    A = synth.random_csr(200, 300, 4000, 71, empty_rows=(0, 3, 150, 199), dense_rows=(5, 9, 60))
    B = synth.dense_b(A.k, n, 72)
    C, pl = run_hybrid(torch_cuda, A, B, hybrid_rows=3)
    check_tol(A, B, C)
    check_parts(pl, A, 3)


def test_hybrid_c4_full_size(torch_cuda):
    """C4 (16384^2 power law at 99%) with the automatic split (rows of at least
    twice the mean length), every row: G2 and dyadic-exact."""
    p = synth.config("c4")
    A = p.A
    lens = np.diff(A.rowptr)
    X = int(np.sum(lens >= 2.0 * A.nnz / A.m))
    C, pl = run_hybrid(torch_cuda, A, p.B, hybrid_rows=X)
    assert pl.info["h"] == 8 and pl.part(1).info["h"] == 1
    check_tol(A, p.B, C)
    Ad, Bd = synth.dyadic_twin(A, 128, 17)
    Cd, _ = run_hybrid(torch_cuda, Ad, Bd, hybrid_rows=X)
    check_exact(Ad, Bd, Cd)


def test_hybrid_rejections(torch_cuda):
    A = synth.power_law(300, 300, 0.95, 5)
    with pytest.raises(escs.EscsError):   # CSR-value walk
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, hybrid_rows=10)
    with pytest.raises(escs.EscsError):   # X out of range
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, hybrid_rows=300)
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, hybrid_rows=10)
    dv = torch_cuda.from_numpy(A.vals).cuda()
    dB = torch_cuda.zeros(A.k, 64, device="cuda")
    C = torch_cuda.empty(A.m, 64, device="cuda")
    with pytest.raises(escs.EscsError) as e:
        escs.escs_spmm(pl, dv, dB, C)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    with pytest.raises(escs.EscsError):
        pl.export()
    assert pl.part(2) is None
    ordinary = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, hybrid_rows=-1)
    assert ordinary.info["hybrid_rows"] == 0 and ordinary.part(0) is None


def test_hybrid_autotuned_c4(torch_cuda, monkeypatch):
    """The tuner on C4 with the hybrid candidate enabled (ESCS_TUNE_HYBRID=1,
    hybrid_rows = 0): whichever plan it keeps is exact."""
    monkeypatch.setenv("ESCS_TUNE_HYBRID", "1")
    monkeypatch.setenv("ESCS_TUNE_CACHE", "0")
    p = synth.config("c4")
    A = p.A
    Ad, Bd = synth.dyadic_twin(A, 128, 19)
    C, pl = run_hybrid(torch_cuda, Ad, Bd, autotune=1)
    print("C4 tuned plan:", {k: pl.info[k] for k in ("hybrid_rows", "h", "autotuned")})
    check_exact(Ad, Bd, C)
