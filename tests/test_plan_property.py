"""Property-based plan parity (hypothesis): for arbitrary small CSR matrices
(ragged m, empty rows/panels, dense rows, any column set) and any UFi in 1..8
and item size T, the product planner (UFi-way merge over CSR) is byte
identical to the oracle's dense-scan partitioner, and the invariants I1-I6 hold.
Host-only plans: no GPU."""
import numpy as np
from hypothesis import given, settings, strategies as st

import oracle
from paper_2506_15174_b200 import escs, synth
from test_oracle import check_invariants


@st.composite
def csr_matrices(draw):
    m = draw(st.integers(1, 40))
    k = draw(st.integers(1, 48))
    density = draw(st.sampled_from([0.0, 0.02, 0.1, 0.3, 0.7, 1.0]))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    rng = np.random.default_rng(seed)
    D = rng.random((m, k)) < density
    if m > 2 and draw(st.booleans()):
        D[draw(st.integers(0, m - 1)), :] = True          # a dense row
    rows, cols = np.nonzero(D)
    rowptr = np.zeros(m + 1, np.int32)
    np.cumsum(np.bincount(rows, minlength=m), out=rowptr[1:])
    vals = rng.uniform(-1, 1, rows.size).astype(np.float32)
    return synth.CSR(m, k, rowptr, cols.astype(np.int32), vals)


@settings(max_examples=150, deadline=None)
@given(A=csr_matrices(), h=st.integers(1, 8), T=st.integers(1, 20),
       nthreads=st.sampled_from([1, 3]))
def test_planner_matches_oracle(A, h, T, nthreads):
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 32, ufi=h, T=T, host_only=1,
                           nthreads=nthreads)
    got = pl.export()
    ref = oracle.partition(A.m, A.k, A.rowptr, A.colidx, h, T, bCols=32)
    assert got["header"] == ref["header"]
    for n in oracle.PLAN_ARRAYS:
        assert np.array_equal(got[n], ref[n]), n
    check_invariants(A, got)
