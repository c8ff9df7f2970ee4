"""Small escs_spmm cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): UFi 1 and 4, vector and scalar lane maps, split and
heavy panels, empty panels, ragged last panel, long UFi > 1 items (operand
pipeline), the packed record walk at every UFi with split and heavy panels,
the staged walk (bulk copies, mbarriers, both combines),
a grouped launch, the scatter epilogue.  Exits
non-zero on a mismatch.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import oracle
    from paper_2506_15174_b200 import escs, synth
    cases = []
    A0 = synth.random_csr(203, 150, 3000, 1, empty_rows=(0, 5, 6, 7, 8), dense_rows=(100,))
    for n in (32, 64, 128, 48):
        for ufi in (1, 4):
            cases.append((A0, n, dict(ufi=ufi, T=7, cta_warps=3)))
    P = synth.power_law(1024, 1024, 0.98, 3)
    cases.append((P, 128, dict(ufi=1, T=16, cta_warps=2)))      # heavy panels
    cases.append((P, 64, dict(ufi=4, T=8, cta_warps=4)))
    for n, colf in ((128, 8), (128, 16), (64, 16), (256, 16), (32, 8)):   # columns-per-lane maps
        cases.append((P, n, dict(ufi=1, T=16, cta_warps=2, colf=colf)))
    for n in (4, 8, 16):                                               # narrow-B sub-warp maps
        cases.append((A0, n, dict(ufi=1, T=7, cta_warps=3)))
    W = synth.random_csr(61, 3000, 40000, 2, empty_rows=(4,), dense_rows=(7,))
    for ufi in (2, 3, 4):               # long items: the UFi > 1 three-chunk operand pipeline
        cases.append((W, 128, dict(ufi=ufi, T=300, cta_warps=4)))
        cases.append((W, 32, dict(ufi=ufi, T=130, cta_warps=2)))
    bad = 0
    for A, n, prm in cases:
        Ad, B = synth.dyadic_twin(A, n, 7)
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, **prm)
        C = torch.empty(A.m, n, device="cuda")
        escs.escs_spmm(pl, torch.from_numpy(Ad.vals).cuda(), torch.from_numpy(B).cuda(), C)
        torch.cuda.synchronize()
        ref = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, Ad.vals, B)
        ok = np.array_equal(C.cpu().numpy().astype(np.float64), ref)
        print(n, prm, "ok" if ok else "MISMATCH", flush=True)
        bad += not ok
    # the packed record walk (escs_pack + escs_spmm_packed), UFi 4, long items,
    # heavy panels through the workspace
    Ad, B = synth.dyadic_twin(W, 64, 8)
    pl = escs.escs_plan_ex(W.m, W.k, W.nnz, W.rowptr, W.colidx, 64, ufi=4, T=300, cta_warps=4, packed=1)
    dv = torch.from_numpy(Ad.vals).cuda()
    C = torch.empty(W.m, 64, device="cuda")
    pk = escs.escs_pack(pl, dv)
    escs.escs_spmm_packed(pl, pk, torch.from_numpy(B).cuda(), C)
    torch.cuda.synchronize()
    ok = np.array_equal(C.cpu().numpy().astype(np.float64),
                        oracle.spmm(W.m, W.k, W.rowptr, W.colidx, Ad.vals, B))
    print("packed", "ok" if ok else "MISMATCH", flush=True)
    bad += not ok
    # the packed record walk: every UFi (1-4, 6, 8), split and heavy panels
    # (CTA-parallel workspace combine, named barriers), tails, narrow B
    for A, n, prm in ((A0, 128, dict(T=7, cta_warps=3)), (P, 64, dict(T=8, cta_warps=4)),
                      (W, 128, dict(T=300, cta_warps=4)), (P, 32, dict(T=16, cta_warps=2))):
        for ufi in (1, 2, 3, 4, 6, 8):
            Ad, B = synth.dyadic_twin(A, n, 11)
            pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=ufi, packed=1, **prm)
            pk = escs.escs_pack(pl, torch.from_numpy(Ad.vals).cuda())
            C = torch.empty(A.m, n, device="cuda")
            escs.escs_spmm_packed(pl, pk, torch.from_numpy(B).cuda(), C)
            torch.cuda.synchronize()
            ok = np.array_equal(C.cpu().numpy().astype(np.float64),
                                oracle.spmm(A.m, A.k, A.rowptr, A.colidx, Ad.vals, B))
            print("records", n, ufi, prm, "ok" if ok else "MISMATCH", flush=True)
            bad += not ok
    # the staged walk (TMA bulk copies + mbarriers, in-kernel column-range
    # combine with the cooperative launch, and the two-launch fallback)
    S0 = synth.magnitude_pruned(300, 1100, 0.7, 5)
    S1 = synth.magnitude_pruned(200, 150, 0.7, 6)   # one column range: no combine
    for S, n, prm in ((S0, 128, dict(ufi=8, st_warps=8, st_nsplit=9)), (S0, 64, dict(ufi=4, st_warps=6, st_npw=2, st_nsplit=5)),
                      (S0, 32, dict(ufi=1, st_warps=4, st_npw=4, st_nsplit=3)), (S1, 128, dict(ufi=3, st_warps=16, st_nsplit=1)),
                      (S0, 128, dict(ufi=2, st_warps=2, st_npw=1, st_nsplit=4))):
        Ad, B = synth.dyadic_twin(S, n, 13)
        pl = escs.escs_plan_ex(S.m, S.k, S.nnz, S.rowptr, S.colidx, n, packed=1, staged=2, **prm)
        pk = escs.escs_pack(pl, torch.from_numpy(Ad.vals).cuda())
        C = torch.empty(S.m, n, device="cuda")
        for _ in range(2):   # twice: the combine counters must reset
            escs.escs_spmm_packed(pl, pk, torch.from_numpy(B).cuda(), C)
        torch.cuda.synchronize()
        ok = np.array_equal(C.cpu().numpy().astype(np.float64),
                            oracle.spmm(S.m, S.k, S.rowptr, S.colidx, Ad.vals, B))
        print("staged", n, prm, pl.info["st_ctas"], "launches", pl.info["st_launches"], "ok" if ok else "MISMATCH",
              flush=True)
        bad += not ok
    # grouped launch: mixed tile widths (idle warps), heavy panels, a UFi-4 single
    probs = [(A0, 64, dict(ufi=1, T=7, cta_warps=3)), (P, 64, dict(ufi=1, T=16, cta_warps=2)),
             (A0, 64, dict(ufi=1, T=9, cta_warps=5)), (W, 64, dict(ufi=4, T=300, cta_warps=4)),
             (P, 128, dict(ufi=1, T=16, cta_warps=2))]
    plans, vs, Bs, Cs, refs = [], [], [], [], []
    for j, (A, n, prm) in enumerate(probs):
        Ad, B = synth.dyadic_twin(A, n, 20 + j)
        plans.append(escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, **prm))
        vs.append(torch.from_numpy(Ad.vals).cuda())
        Bs.append(torch.from_numpy(B).cuda())
        Cs.append(torch.empty(A.m, n, device="cuda"))
        refs.append(oracle.spmm(A.m, A.k, A.rowptr, A.colidx, Ad.vals, B))
    escs.escs_spmm_group(plans, vs, Bs, Cs)
    torch.cuda.synchronize()
    ok = all(np.array_equal(c.cpu().numpy().astype(np.float64), r) for c, r in zip(Cs, refs))
    print("group", "ok" if ok else "MISMATCH", flush=True)
    bad += not ok
    # fused all-gather epilogue: two row blocks into two destinations
    A, n = A0, 128
    Ad, B = synth.dyadic_twin(A, n, 9)
    dB = torch.from_numpy(B).cuda()
    dsts = [torch.empty(A.m, n, device="cuda") for _ in range(2)]
    for r in range(2):
        r0, r1 = synth.shard_bounds(A.m, 2, r)
        S = synth.row_block(Ad, r0, r1)
        pl = escs.escs_plan_ex(S.m, S.k, S.nnz, S.rowptr, S.colidx, n, ufi=1, T=7, cta_warps=3)
        escs.escs_spmm_scatter(pl, torch.from_numpy(S.vals).cuda(), dB, dsts, r0)
    torch.cuda.synchronize()
    ref = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, Ad.vals, B)
    ok = all(np.array_equal(d.cpu().numpy().astype(np.float64), ref) for d in dsts)
    print("scatter", "ok" if ok else "MISMATCH", flush=True)
    bad += not ok
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
