"""The staged walk's schedule (escs_params.staged = 2, include/escs.h
escs_staged_export) on host-only plans -- no GPU needed.

The schedule is derived from the canonical plan (whose arrays are byte-checked
against the oracle partitioner in test_plan_parity.py): CTA c = (row block rb,
column range sp) owns panels [rb*nslot, (rb+1)*nslot) and columns
[sp*k/nsplit, (sp+1)*k/nsplit), cut into stages of st_kb columns; its records
are the owned panels' gcols in those columns.  Checked here, independently of
the library's construction:
  * the record stream is a permutation of the canonical gcols (every (panel,
    column, pattern) of the enumeration exactly once) plus padding;
  * each record sits in the CTA, stage and warp slot its panel and column
    select, and a slot's records keep the canonical order (pattern groups
    ascending, columns ascending within a group -- Fig. 4 / Reading R3);
  * headers, stage bounds and 16-byte padding are consistent; the shared
    memory the CTA needs fits the budget.
"""
import numpy as np
import pytest

from paper_2506_15174_b200 import escs, synth


def staged_plan(A, n, **kw):
    return escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, packed=1, staged=2, host_only=1, **kw)


def check_schedule(A, n, h, **kw):
    pl = staged_plan(A, n, ufi=h, **kw)
    info, ex, st = pl.info, escs.escs_plan_export(pl), escs.escs_staged_export(pl)
    hd = ex["header"]
    k, nP, G = hd["k"], hd["nP"], hd["G"]
    W, npw, ns, kb = info["st_warps"], info["st_npw"], info["st_nsplit"], info["st_kb"]
    nslot = W * npw
    assert st["nslot"] == nslot and info["staged"] == 1
    n_rb = -(-nP // nslot)
    assert st["n_cta"] == n_rb * ns == info["st_ctas"]
    # canonical gcol -> (panel, column, canonical index)
    gpanel = np.repeat(ex["grp_panel"], np.diff(ex["grp_col_ptr"]))
    gcol = ex["gcol"]
    src = st["src"]
    assert np.array_equal(np.sort(src[src >= 0]), np.arange(G)), "not a permutation of the gcols"
    rw = {1: 2, 2: 4, 3: 4, 4: 8, 6: 8, 8: 12}[h]
    pad = max(1, 16 // (4 * rw))
    cta, stage, hdr = st["cta"], st["stage"], st["hdr"]
    seen = 0
    for c in range(st["n_cta"]):
        rb, sp, s0, nst = cta[c]
        assert (rb, sp) == (c // ns, c % ns)
        assert s0 == c * st["max_stages"], "stages at a fixed stride per CTA"
        assert np.all(stage[s0 + nst:s0 + st["max_stages"]] == 0) and np.all(hdr[s0 + nst:s0 + st["max_stages"]] == 0)
        k0, k1 = sp * k // ns, (sp + 1) * k // ns
        assert nst == max(0, -(-(k1 - k0) // kb)) and nst <= 16
        rec0 = stage[s0, 2]
        assert rec0 % pad == 0
        for s in range(s0, s0 + nst):
            ks, ke, r0, nr = stage[s]
            assert ks == k0 + (s - s0) * kb and ke == min(k1, ks + kb)
            assert r0 == seen and nr % pad == 0
            hs = hdr[s]
            assert hs[0] == r0 - rec0 and np.all(np.diff(hs[:nslot + 1]) >= 0)
            assert r0 - rec0 + nr - hs[nslot] < pad, "padding beyond one 16-byte unit"
            assert np.all(src[rec0 + hs[nslot]:r0 + nr] == -1)
            for j in range(nslot):
                q = src[rec0 + hs[j]:rec0 + hs[j + 1]]
                assert np.all(q >= 0)
                P = rb * nslot + j
                if P >= nP:
                    assert len(q) == 0
                    continue
                assert np.all(gpanel[q] == P), "record of another panel in the slot"
                assert np.all((gcol[q] >= ks) & (gcol[q] < ke)), "record outside its stage"
                assert np.all(np.diff(q) > 0), "slot does not keep the canonical order"
                # completeness: every gcol of P in [ks, ke) is here
                want = np.nonzero((gpanel == P) & (gcol >= ks) & (gcol < ke))[0]
                assert np.array_equal(q, want)
            seen = r0 + nr
    assert seen == st["n_rec"] == len(src)
    assert st["n_stage"] == st["n_cta"] * st["max_stages"]
    assert info["packed_words"] == (st["n_rec"] * rw + 3) // 4 * 4
    smem = (st["max_k"] * n + st["max_rec"] * rw + st["max_stages"] * st["hdr"].shape[1]) * 4
    assert smem <= 227 * 1024
    return info


@pytest.mark.parametrize("h", [1, 2, 3, 4, 6, 8])
def test_schedule_transformer_layer(h):
    p = synth.transformer_suite(bcols=(128,), sparsities=(0.7,))[0]
    check_schedule(p.A, 128, h)


@pytest.mark.parametrize("h,W,npw,ns", [(1, 8, 4, 3), (3, 16, 2, 2), (4, 5, 1, 7), (8, 16, 1, 37), (2, 3, 2, 64)])
def test_schedule_explicit_tiles(h, W, npw, ns):
    A = synth.magnitude_pruned(300, 700, 0.8, 7)   # ragged: m not a multiple of UFi or of the row block
    info = check_schedule(A, 64, h, st_warps=W, st_npw=npw, st_nsplit=ns)
    assert (info["st_warps"], info["st_npw"], info["st_nsplit"]) == (W, npw, ns)


def test_schedule_kb_and_bcols32():
    A = synth.magnitude_pruned(96, 2048, 0.9, 3)
    check_schedule(A, 32, 4, st_kb=40, st_nsplit=5)


def test_schedule_degenerate():
    # empty matrix, one row, one column, dense row
    for A in (synth.CSR(5, 9, np.zeros(6, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32)),
              synth.magnitude_pruned(1, 50, 0.5, 1), synth.magnitude_pruned(40, 1, 0.5, 2),
              synth.magnitude_pruned(17, 33, 0.0, 3)):
        for h in (1, 3, 8):
            check_schedule(A, 64, h)


def test_schedule_powerlaw_rows():
    A = synth.power_law(600, 900, 0.97, 11)
    for h in (1, 4):
        check_schedule(A, 128, h, st_warps=8)


def test_staged_parameter_errors():
    A = synth.magnitude_pruned(64, 64, 0.7, 1)
    with pytest.raises(escs.EscsError) as e:   # staged needs the packed walk
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, staged=2, host_only=1)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    with pytest.raises(escs.EscsError) as e:   # bCols outside 32/64/128
        staged_plan(A, 256)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    with pytest.raises(escs.EscsError) as e:
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, staged=3, host_only=1)
    assert e.value.code == escs.ESCS_ERR_ARG
    with pytest.raises(escs.EscsError) as e:   # a fixed split that cannot fit shared memory
        staged_plan(synth.magnitude_pruned(16, 60000, 0.5, 1), 128, st_nsplit=1)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    with pytest.raises(escs.EscsError) as e:   # more splits than columns
        staged_plan(A, 64, st_nsplit=65)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    # no staged schedule on an ordinary plan
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, host_only=1)
    assert pl.info["staged"] == 0
    with pytest.raises(escs.EscsError):
        escs.escs_staged_export(pl)


def test_schedule_deterministic():
    p = synth.resnet_suite(bcols=(64,), sparsities=(0.8,))[2]
    a = escs.escs_staged_export(staged_plan(p.A, 64, ufi=4, nthreads=1))
    b = escs.escs_staged_export(staged_plan(p.A, 64, ufi=4, nthreads=8))
    for key in ("cta", "stage", "hdr", "src"):
        assert np.array_equal(a[key], b[key])


def test_hybrid_and_carveout_parameter_errors():
    """Host-side checks of the hybrid_rows and carveout fields (include/escs.h)."""
    A = synth.power_law(200, 300, 0.9, 3)
    with pytest.raises(escs.EscsError) as e:   # hybrid plans are device plans
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, host_only=1, hybrid_rows=10)
    assert e.value.code == escs.ESCS_ERR_UNSUPPORTED
    with pytest.raises(escs.EscsError) as e:
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, host_only=1, hybrid_rows=-5)
    assert e.value.code == escs.ESCS_ERR_ARG
    for cv in (-3, 101):
        with pytest.raises(escs.EscsError) as e:
            escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, host_only=1, carveout=cv)
        assert e.value.code == escs.ESCS_ERR_ARG
    for cv in (-2, -1, 0, 37, 100):   # accepted (host-only plans launch nothing)
        escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, host_only=1, carveout=cv)
