"""Small escs_spmm cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): UFi 1 and 4, vector and scalar lane maps, split and
heavy panels, empty panels, ragged last panel.  Exits non-zero on a mismatch.

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
