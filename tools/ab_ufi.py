"""Matched UFi A/B on one layer: UFi 1..4 with the same
tile width (4 warps), the same number of items (~4096 warps -> the same
achieved occupancy), 8 columns per lane and UFk 8; packed record walk.
Prints hot-L2 graph times; under ncu (--nvtx-include ab_ufi/) each plan's
second launch is the captured one.

    python tools/ab_ufi.py [--case 512x4608@70%/b128] [--items 4096]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="512x4608@70%/b128")
    ap.add_argument("--items", type=int, default=4096)
    ap.add_argument("--warps", type=int, default=4)
    ap.add_argument("--ufk", type=int, default=8)
    ap.add_argument("--colf", type=int, default=8)
    ap.add_argument("--ncu", action="store_true", help="two launches per plan inside an NVTX range, no timing")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2506_15174_b200 import escs
    p = [q for wl in ("resnet", "transformer") for q in bench.workload(wl)[0] if q.name == a.case][0]
    A, n = p.A, p.bcols
    dv, dB = torch.from_numpy(A.vals).cuda(), torch.from_numpy(p.B).cuda()
    dC = torch.empty(A.m, n, device="cuda")
    st = torch.cuda.Stream()
    for h in (1, 2, 3, 4):
        host = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=h, T=1 << 20, host_only=1)
        G, nP = host.info["G"], host.info["nP"]
        per = max(1, round(a.items / nP))
        T = max(1, math.ceil(G / nP / per))
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=h, T=T, cta_warps=a.warps,
                               ufk=a.ufk, colf=a.colf, packed=1)
        pk = escs.escs_pack(pl, dv)
        inf = pl.info
        fn = lambda: escs.escs_spmm_packed(pl, pk, dB, dC, st)
        if a.ncu:
            torch.cuda.nvtx.range_push("ab_ufi")
            with torch.cuda.stream(st):
                fn()
                fn()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
            t = float("nan")
        else:
            t = bench.graph_time(torch, fn, st, reps=20)
        print(f"UFi {h}: p = nnz/G {A.nnz / G:.3f}  T {T}  items {inf['n_items']}  tiles {inf['n_tiles']}  "
              f"heavy {inf['n_heavy']}  ctas/SM {inf['ctas_per_sm']}  hot {1e3 * t:.2f} us", flush=True)


if __name__ == "__main__":
    main()
