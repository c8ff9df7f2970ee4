"""Pins for the CPU oracle (oracle/) against things other than itself.

SpMM (Listing 1): numpy dense fp64 matmul, exact dyadic integer
arithmetic, identity A, identity B, single-nonzero rows, empty A.
Partition: hand-written golden plans
(tests/golden, S:123/S:132/S:501), the exhaustive 15-pattern matrix (P:152,
S:567), 7 patterns for UFi=3, a brute-force enumeration on tiny inputs,
invariants I1-I7, and the closed-form expected gcol count.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense_of(A):
    D = np.zeros((A.m, A.k), np.float64)
    rows = np.repeat(np.arange(A.m), np.diff(A.rowptr))
    D[rows, A.colidx] = A.vals
    return D


# ----------------------------------------------------------------- spmm pins

@pytest.mark.parametrize("m,k,n,nnz,seed", [(1, 1, 1, 1, 0), (7, 5, 3, 11, 1), (33, 65, 32, 400, 2),
                                            (64, 300, 17, 2000, 3)])
def test_spmm_matches_dense_numpy(m, k, n, nnz, seed):
    A = synth.random_csr(m, k, nnz, seed, empty_rows=(0,) if m > 2 else ())
    B = synth.dense_b(k, n, seed + 100)
    C = oracle.spmm(m, k, A.rowptr, A.colidx, A.vals, B)
    ref = dense_of(A) @ B.astype(np.float64)
    np.testing.assert_allclose(C, ref, rtol=1e-12, atol=1e-12)


def test_spmm_c1_matches_dense_numpy():
    p = synth.config("c1")
    A = p.A
    C = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, p.B)
    ref = dense_of(A) @ p.B.astype(np.float64)
    np.testing.assert_allclose(C, ref, rtol=1e-12, atol=1e-12)


def test_spmm_dyadic_exact():
    A0 = synth.magnitude_pruned(96, 200, 0.7, 7)
    A, B = synth.dyadic_twin(A0, 40, 8)
    C = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, B)
    # exact integer arithmetic: 2*A is integral, B is integral
    D2 = np.zeros((A.m, A.k), np.int64)
    rows = np.repeat(np.arange(A.m), np.diff(A.rowptr))
    D2[rows, A.colidx] = (2 * A.vals).astype(np.int64)
    exact = (D2 @ B.astype(np.int64)).astype(np.float64) / 2.0
    assert np.array_equal(C, exact)


def test_spmm_identity_A_gives_B():
    k = 37
    rowptr = np.arange(k + 1, dtype=np.int32)
    colidx = np.arange(k, dtype=np.int32)
    vals = np.ones(k, np.float32)
    B = synth.dense_b(k, 9, 5)
    C = oracle.spmm(k, k, rowptr, colidx, vals, B)
    assert np.array_equal(C, B.astype(np.float64))


def test_spmm_identity_B_gives_dense_A():
    A = synth.random_csr(12, 10, 40, 9)
    B = np.eye(10, dtype=np.float32)
    C = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, B)
    assert np.array_equal(C, dense_of(A))


def test_spmm_single_nonzero_rows_scale():
    rng = np.random.default_rng(3)
    m, k, n = 20, 15, 8
    cols = rng.integers(0, k, m).astype(np.int32)
    vals = rng.uniform(-2, 2, m).astype(np.float32)
    B = synth.dense_b(k, n, 4)
    C = oracle.spmm(m, k, np.arange(m + 1, dtype=np.int32), cols, vals, B)
    assert np.array_equal(C, vals[:, None].astype(np.float64) * B[cols].astype(np.float64))


def test_spmm_empty_and_rows_subset():
    A = synth.random_csr(30, 30, 0, 1)
    C = oracle.spmm(30, 30, A.rowptr, A.colidx, A.vals, synth.dense_b(30, 4, 1))
    assert np.array_equal(C, np.zeros((30, 4)))
    A = synth.random_csr(50, 40, 300, 2)
    B = synth.dense_b(40, 6, 3)
    full, absum, nt = oracle.spmm(50, 40, A.rowptr, A.colidx, A.vals, B, with_absum=True)
    rows = np.array([49, 0, 17, 17], np.int64)
    sub = oracle.spmm(50, 40, A.rowptr, A.colidx, A.vals, B, rows=rows)
    assert np.array_equal(sub, full[rows])
    assert np.all(absum >= np.abs(full))
    assert np.array_equal(nt, np.diff(A.rowptr))
    # absum is the same product with |A| and |B|
    ref = np.abs(dense_of(A)) @ np.abs(B.astype(np.float64))
    np.testing.assert_allclose(absum, ref, rtol=1e-12)


def test_generator_nnz_pin():
    # gen_random(512, 512, 0.7) -> nnz = 78,643 = round(0.3 * 512 * 512)
    A = synth.magnitude_pruned(512, 512, 0.7, 1000)
    assert A.nnz == 78643
    assert np.all(np.diff(A.rowptr) >= 0)
    for i in range(0, 512, 37):
        c = A.colidx[A.rowptr[i]:A.rowptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    # magnitude pruning keeps the largest |w|: every kept |w| >= every dropped one
    rng = np.random.default_rng(1000)
    w = rng.standard_normal((512, 512), dtype=np.float32)
    thr = np.abs(A.vals).min()
    D = dense_of(A)
    assert np.all(np.abs(w[D == 0]) <= thr)


# ------------------------------------------------------------ partition pins

def _golden():
    with open(os.path.join(GOLD, "spec_4x4_plan.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", range(3))
def test_partition_golden(case):
    g = _golden()
    c = g["cases"][case]
    p = oracle.partition(g["m"], g["k"], g["rowptr"], g["colidx"], c["h"], c["T"])
    for key, val in c["header"].items():
        assert p["header"][key] == val, key
    for name in oracle.PLAN_ARRAYS:
        assert p[name].tolist() == c[name], name
    if c["h"] == 4:
        # S:501 reuseFactorB = p_bar = nnz / G = 7/4
        assert p["header"]["nnz"] / p["header"]["G"] == 7 / 4


def test_partition_exhaustive_15_patterns():
    # 4 x 15 matrix, column c has pattern c+1 ("15 possible sparsity patterns")
    rows = [[c for c in range(15) if ((c + 1) >> r) & 1] for r in range(4)]
    rowptr = np.cumsum([0] + [len(r) for r in rows]).astype(np.int32)
    colidx = np.concatenate(rows).astype(np.int32)
    p = oracle.partition(4, 15, rowptr, colidx, 4, 100)
    assert p["header"]["NG"] == 15
    assert p["grp_mask"].tolist() == list(range(1, 16))
    assert p["gcol"].tolist() == list(range(15))
    assert np.all(np.diff(p["grp_col_ptr"]) == 1)
    # UFi=3 over the same rows: panel 0 (rows 0-2) holds all 7 patterns
    p3 = oracle.partition(4, 15, rowptr, colidx, 3, 100)
    assert (p3["grp_panel"] == 0).sum() == 7
    assert p3["grp_mask"][p3["grp_panel"] == 0].tolist() == list(range(1, 8))


def brute_plan(A, h, T):
    """Brute force from the definitions, by a different route than the oracle:
    per panel, for every pattern value mu ascending, scan all columns and keep
    those whose pattern equals mu; CSR positions via a (row, col) dict;
    items by the P7 even-split definition."""
    m, k = A.m, A.k
    where = {}
    for i in range(m):
        for t in range(A.rowptr[i], A.rowptr[i + 1]):
            where[(i, int(A.colidx[t]))] = t
    nP = -(-m // h)
    gp, gm, gcp, gvp, gcol, slots = [], [], [0], [0], [], []
    ip, igb, igp = [], [], [0]
    for P in range(nP):
        pat = [sum(1 << r for r in range(h) if (P * h + r, c) in where) for c in range(k)]
        g0, s0 = len(gp), len(gcol)
        for mu in range(1, 1 << h):
            cols = [c for c in range(k) if pat[c] == mu]
            if not cols:
                continue
            gp.append(P); gm.append(mu)
            gcp.append(gcp[-1] + len(cols))
            prow = [r for r in range(h) if (mu >> r) & 1]
            gvp.append(gvp[-1] + len(cols) * len(prow))
            gcol += cols
            for c in cols:
                for r in prow:
                    slots.append(where[(P * h + r, c)])
        SP = len(gcol) - s0
        n = max(1, -(-SP // T))
        for q in range(n):
            a, b = q * SP // n, (q + 1) * SP // n
            cands = [g for g in range(g0, len(gp)) if gcp[g] - s0 <= a]
            ip.append(P)
            igb.append(cands[-1] if cands else g0)
            igp.append(s0 + b)
    return dict(grp_panel=gp, grp_mask=gm, grp_col_ptr=gcp, grp_val_ptr=gvp, gcol=gcol,
                slot_src=slots, item_panel=ip, item_group_begin=igb, item_gcol_ptr=igp)


@pytest.mark.parametrize("m,k,nnz,h,T,seed", [
    (9, 7, 20, 4, 3, 1), (13, 11, 60, 3, 2, 2), (16, 16, 256, 4, 5, 3),    # dense
    (10, 9, 0, 2, 1, 4), (17, 23, 80, 5, 7, 5), (8, 30, 90, 8, 11, 6),
    (21, 12, 70, 1, 4, 7), (6, 40, 150, 4, 1, 8)])
def test_partition_brute_force(m, k, nnz, h, T, seed):
    A = synth.random_csr(m, k, nnz, seed, empty_rows=(1,) if m > 4 else ())
    p = oracle.partition(m, k, A.rowptr, A.colidx, h, T)
    ref = brute_plan(A, h, T)
    for name in oracle.PLAN_ARRAYS:
        assert p[name].tolist() == ref[name], name


def check_invariants(A, p):
    """I1-I6 of SURVEY §8(c)."""
    hdr = p["header"]
    h, T, nnz = hdr["h"], hdr["T"], A.nnz
    NG, G, NI, nP = hdr["NG"], hdr["G"], hdr["n_items"], hdr["nP"]
    assert nP == -(-A.m // h)
    gm, gp = p["grp_mask"], p["grp_panel"]
    gcp, gvp = p["grp_col_ptr"], p["grp_val_ptr"]
    widths = np.diff(gcp)
    pops = np.array([bin(int(x)).count("1") for x in gm], np.int64)
    # I1: slot_src is a permutation of [0, nnz)
    assert np.array_equal(np.sort(p["slot_src"]), np.arange(nnz))
    # I4: conservation
    assert int((pops * widths).sum()) == nnz
    assert np.array_equal(np.diff(gvp), pops * widths)
    assert G == gcp[-1] == len(p["gcol"])
    # I2: slot -> (row, col) consistency
    rows_of = np.repeat(np.arange(A.m), np.diff(A.rowptr))
    for g in range(NG):
        prow = [r for r in range(h) if (int(gm[g]) >> r) & 1]
        for ci in range(int(widths[g])):
            col = p["gcol"][gcp[g] + ci]
            for rank, r in enumerate(prow):
                t = p["slot_src"][gvp[g] + ci * len(prow) + rank]
                assert rows_of[t] == gp[g] * h + r
                assert A.colidx[t] == col
    # I3 + I5: per panel, masks strictly ascend, <= 2^h - 1 groups, columns unique
    assert np.all(np.diff(gp) >= 0)
    for P in np.unique(gp):
        sel = np.flatnonzero(gp == P)
        assert len(sel) <= (1 << h) - 1
        assert np.all(np.diff(gm[sel]) > 0)
        assert np.all((gm[sel] > 0) & (gm[sel] < (1 << h)))
        cols = np.concatenate([p["gcol"][gcp[g]:gcp[g + 1]] for g in sel])
        assert len(np.unique(cols)) == len(cols)
        for g in sel:
            assert np.all(np.diff(p["gcol"][gcp[g]:gcp[g + 1]]) > 0)
    # I6: items tile each panel's stream, every panel has >= 1 item, sizes <= T, differ by <= 1
    ip, igp = p["item_panel"], p["item_gcol_ptr"]
    assert NI == len(ip) and igp[0] == 0 and igp[-1] == G
    assert np.all(np.diff(ip) >= 0)
    assert np.array_equal(np.unique(ip), np.arange(nP))
    sizes = np.diff(igp)
    assert np.all(sizes >= 0) and np.all(sizes <= T)
    for P in range(nP):
        s = sizes[ip == P]
        assert s.max() - s.min() <= 1
        if len(s) > 1:
            assert s.min() >= 1


@pytest.mark.parametrize("h,T", [(4, 16), (3, 7), (1, 32), (2, 1000)])
def test_partition_invariants_c1(h, T):
    p0 = synth.config("c1")
    A = p0.A
    p = oracle.partition(A.m, A.k, A.rowptr, A.colidx, h, T)
    check_invariants(A, p)


def test_partition_invariants_powerlaw_small():
    A = synth.power_law(512, 512, 0.95, 77)
    p = oracle.partition(A.m, A.k, A.rowptr, A.colidx, 4, 24)
    check_invariants(A, p)


def test_partition_expected_gcol_count():
    # Closed form for a uniform pattern: E[G] = ceil(m/h)*k*(1-s^h),
    # p_bar = h(1-s)/(1-s^h).  Magnitude pruning of iid N(0,1) gives a uniform pattern.
    m, k, s, h = 512, 512, 0.7, 4
    A = synth.magnitude_pruned(m, k, s, 1000)
    p = oracle.partition(m, k, A.rowptr, A.colidx, h, 64)
    EG = -(-m // h) * k * (1 - s ** h)
    assert abs(p["header"]["G"] - EG) / EG < 0.01
    pbar = A.nnz / p["header"]["G"]
    assert abs(pbar - h * (1 - s) / (1 - s ** h)) < 0.02


def test_partition_determinism():
    A = synth.magnitude_pruned(200, 300, 0.8, 4)
    a = oracle.partition(A.m, A.k, A.rowptr, A.colidx, 4, 10)
    b = oracle.partition(A.m, A.k, A.rowptr, A.colidx, 4, 10)
    for name in oracle.PLAN_ARRAYS:
        assert np.array_equal(a[name], b[name])


def test_storage_trend_matches_paper_fig9():
    # P:796-798 / P:823 (Fig. 9): the ESC format (ANNZ + Cols + RPP + NPP) is
    # smaller than CSR for roughly 50-80% sparsity, and CSR is smaller near 99%.
    m = k = 512
    for s, esc_smaller in ((0.5, True), (0.6, True), (0.7, True), (0.8, True),
                           (0.95, False), (0.99, False)):
        A = synth.magnitude_pruned(m, k, s, 77)
        p = oracle.partition(m, k, A.rowptr, A.colidx, 4, 1 << 20)
        hdr = p["header"]
        esc = 4 * hdr["nnz"] + 4 * hdr["G"] + 8 * (hdr["NG"] + 1) + 8 * hdr["NG"]
        csr = 8 * A.nnz + 4 * (m + 1)
        assert (esc < csr) == esc_smaller, (s, esc, csr)


def test_resnet50_shape_list():
    """The extended C3 suite: 21 distinct ResNet-50 GEMM shapes."""
    from paper_2506_15174_b200 import synth
    shapes = synth.RESNET50_ALL_SHAPES
    assert len(shapes) == 21 and len(set(shapes)) == 21
    assert set(synth.RESNET_SHAPES) <= set(shapes)
    suite = synth.resnet50_full_suite(bcols=(32,), sparsities=(0.9,))
    for p, (m, k) in zip(suite, shapes):
        assert (p.A.m, p.A.k) == (m, k)
        assert p.A.nnz == synth.nnz_for(m, k, 0.9)
