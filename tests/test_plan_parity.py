"""Plan parity: the product planner (libescs.so, UFi-way merge over CSR) must
produce byte-identical plans to the oracle partitioner (dense scan, the
paper's dataTransformer) -- SURVEY §8(c) parity procedure step 3.
Host-only plans (escs_params.host_only = 1): no GPU needed."""
import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import escs, synth
from test_oracle import check_invariants


def assert_same_plan(A, h, T, nthreads=0, bcols=32):
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, bcols, ufi=h, T=T, host_only=1,
                           nthreads=nthreads)
    got = pl.export()
    ref = oracle.partition(A.m, A.k, A.rowptr, A.colidx, h, T, bCols=bcols)
    assert got["header"] == ref["header"]
    for n in oracle.PLAN_ARRAYS:
        assert np.array_equal(got[n], ref[n]), n
    return got


@pytest.mark.parametrize("h,T", [(4, 4), (4, 2), (3, 4), (1, 1), (2, 3)])
def test_golden(h, T):
    import json, os
    with open(os.path.join(os.path.dirname(__file__), "golden", "spec_4x4_plan.json")) as f:
        g = json.load(f)
    A = synth.CSR(4, 4, np.array(g["rowptr"], np.int32), np.array(g["colidx"], np.int32),
                  np.ones(7, np.float32))
    assert_same_plan(A, h, T)


@pytest.mark.parametrize("seed", range(12))
def test_random_small(seed):
    rng = np.random.default_rng(seed)
    m, k = int(rng.integers(1, 60)), int(rng.integers(1, 70))
    nnz = int(rng.integers(0, m * k + 1))
    h = int(rng.integers(1, 9))
    T = int(rng.integers(1, 12))
    A = synth.random_csr(m, k, nnz, seed, empty_rows=(0,) if m > 3 else (),
                         dense_rows=(m - 1,) if m > 5 else ())
    got = assert_same_plan(A, h, T)
    check_invariants(A, got)


@pytest.mark.parametrize("h,T", [(4, 16), (4, 64), (3, 7), (2, 1000), (1, 32), (8, 40)])
def test_c1(h, T):
    A = synth.config("c1").A
    assert_same_plan(A, h, T)


def test_suite_shapes_sampled():
    for (m, k) in synth.TRANSFORMER_SHAPES + synth.RESNET_SHAPES:
        for s in (0.7, 0.98):
            A = synth.magnitude_pruned(m, k, s, 4242)
            assert_same_plan(A, 4, 24)


def test_powerlaw_heavy_panels():
    A = synth.power_law(2048, 2048, 0.99, 9)
    got = assert_same_plan(A, 4, 40)
    check_invariants(A, got)


def test_thread_count_determinism():
    A = synth.magnitude_pruned(2048, 512, 0.7, 11)     # nnz > planner's threading cutoff
    assert A.nnz > 200000
    a = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, ufi=4, T=33, host_only=1,
                          nthreads=1).export()
    b = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, ufi=4, T=33, host_only=1,
                          nthreads=7).export()
    assert a["header"] == b["header"]
    for n in escs.PLAN_ARRAYS:
        assert np.array_equal(a[n], b[n])
    assert_same_plan(A, 4, 33, nthreads=5, bcols=64)


@pytest.mark.slow
def test_c4_full():
    A = synth.config("c4").A
    assert_same_plan(A, 4, 280, bcols=128)
