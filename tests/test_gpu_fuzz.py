"""Seeded randomized parity (GPU): random shapes, densities, forced empty and
dense rows, every bCols class and every plan parameter the ABI exposes (UFi,
T, tile width, UFk, columns per lane, vector/scalar map), dyadic twins so the
comparison with the fp64 oracle is bit-exact whatever the summation order
(SURVEY §8(c) G1).  A failure prints the case so it can be replayed."""
import os

import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import synth

pytestmark = pytest.mark.gpu

BCOLS = (1, 4, 8, 16, 24, 32, 48, 64, 100, 128, 200, 256)


def _case(i):
    rng = np.random.default_rng(9000 + i)
    m = int(rng.integers(1, 700))
    k = int(rng.integers(1, 3000))
    dens = float(rng.choice([0.002, 0.01, 0.05, 0.2, 0.5]))
    nnz = int(min(m * k, max(0, round(dens * m * k))))
    empty = tuple(int(x) for x in rng.choice(m, size=min(m, int(rng.integers(0, 4))), replace=False))
    dense = tuple(int(x) for x in rng.choice(m, size=min(m, int(rng.integers(0, 3))), replace=False)
                  if x not in empty)
    n = int(rng.choice(BCOLS))
    params = {"ufi": int(rng.choice([1, 1, 2, 3, 4])), "T": int(rng.choice([0, 4, 16, 64, 300])),
              "cta_warps": int(rng.choice([0, 1, 4, 8, 16])), "variant": int(rng.choice([0, 0, 2])),
              "ufk": int(rng.choice([0, 2, 4, 8]))}
    if params["ufi"] == 1 and n in (32, 64, 128, 256) and rng.random() < 0.5:
        params["colf"] = int(rng.choice([8, 16]))
    return m, k, nnz, empty, dense, n, params


N_CASES = int(os.environ.get("ESCS_FUZZ_N", "48"))   # a longer sweep: ESCS_FUZZ_N=600


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_case_exact(i):
    import torch
    from paper_2506_15174_b200 import escs
    m, k, nnz, empty, dense, n, params = _case(i)
    A0 = synth.random_csr(m, k, nnz, 100 + i, empty_rows=empty, dense_rows=dense)
    A, B = synth.dyadic_twin(A0, n, 200 + i)
    params = {key: v for key, v in params.items() if v}
    try:
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, **params)
    except escs.EscsError as e:
        # only combinations the library documents as unsupported may be refused
        assert e.code == escs.ESCS_ERR_UNSUPPORTED, (i, params, e)
        pytest.skip(f"unsupported combination {params}: {e}")
    dv = torch.from_numpy(A.vals).cuda() if A.nnz else torch.zeros(1, device="cuda")
    dB = torch.from_numpy(B).cuda()
    dC = torch.full((A.m, n), float("nan"), device="cuda")
    escs.escs_spmm(pl, dv, dB, dC)
    torch.cuda.synchronize()
    ref = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, B)
    got = dC.cpu().numpy().astype(np.float64)
    bad = np.argwhere(got != ref)
    assert bad.size == 0, (i, (m, k, nnz, n), params, pl.info, bad[:3], got[tuple(bad[0])], ref[tuple(bad[0])])


@pytest.mark.parametrize("g", range(max(4, N_CASES // 12)))
def test_random_group_exact(g):
    """escs_spmm_group over a random set of the cases above (mixed bCols,
    UFi, tile widths, lane maps; some launched singly): bit-exact per problem."""
    import torch
    from paper_2506_15174_b200 import escs
    rng = np.random.default_rng(777 + g)
    ids = rng.choice(10 * N_CASES + 500, size=int(rng.integers(3, 41)), replace=False)
    plans, vs, Bs, Cs, refs = [], [], [], [], []
    for i in ids:
        m, k, nnz, empty, dense, n, params = _case(int(i))
        A0 = synth.random_csr(m, k, nnz, 100 + int(i), empty_rows=empty, dense_rows=dense)
        A, B = synth.dyadic_twin(A0, n, 200 + int(i))
        params = {key: v for key, v in params.items() if v}
        try:
            pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, **params)
        except escs.EscsError as e:
            assert e.code == escs.ESCS_ERR_UNSUPPORTED
            continue
        plans.append(pl)
        vs.append(torch.from_numpy(A.vals).cuda() if A.nnz else torch.zeros(1, device="cuda"))
        Bs.append(torch.from_numpy(B).cuda())
        Cs.append(torch.full((A.m, n), float("nan"), device="cuda"))
        refs.append(oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, B))
    escs.escs_spmm_group(plans, vs, Bs, Cs)
    torch.cuda.synchronize()
    for j, (c, r) in enumerate(zip(Cs, refs)):
        got = c.cpu().numpy().astype(np.float64)
        assert np.array_equal(got, r), (g, j, plans[j].info)
