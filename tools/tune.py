"""Offline tuning sweep (the paper's profiling-based scheduler, §3.5):
for every problem of a workload, time escs_spmm over a grid of (UFi, UFk, T)
with the hot-L2 CUDA-graph protocol and record the best; the parameter table
in csrc/plan.cpp (choose_params) is derived from these results.

    python tools/tune.py [--workload transformer] [--out gpurun_out/tune.json]
"""
import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="transformer")
    ap.add_argument("--out", default="gpurun_out/tune.json")
    ap.add_argument("--ufi", default="1,2,4")
    ap.add_argument("--ufk", default="2,4,8")
    ap.add_argument("--T", default="0,8,16,32,64,128,256")
    ap.add_argument("--warps", default="0")
    ap.add_argument("--colf", default="0", help="B columns per lane of the vector map (0 = default)")
    ap.add_argument("--filter", default="", help="comma-separated substrings of case names")
    ap.add_argument("--packed", action="store_true", help="time escs_spmm_packed (the record walk on escs_pack's stream)")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2506_15174_b200 import escs
    problems, _ = bench.workload(a.workload)
    if a.filter:
        keys = a.filter.split(",")
        problems = [p for p in problems if any(k in p.name for k in keys)]
        seen = set()
        problems = [p for p in problems if not (p.name in seen or seen.add(p.name))]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out = []
    t0 = time.time()
    for p in problems:
        A, n = p.A, p.bcols
        dv = torch.from_numpy(A.vals).cuda()
        dB = torch.from_numpy(p.B).cuda()
        dC = torch.empty(A.m, n, device="cuda")
        auto = escs.escs_plan(A.m, A.k, A.nnz, A.rowptr, A.colidx, n)
        t_auto = bench.graph_time(torch, lambda: escs.escs_spmm(auto, dv, dB, dC, stream), stream,
                                  min_ms=1.0, reps=5)
        rec = {"case": p.name, "auto_us": 1e3 * t_auto,
               "auto": {k: auto.info[k] for k in ("h", "T", "cta_warps", "ufk", "colf", "n_tiles")},
               "grid": []}
        best = (t_auto, rec["auto"])
        grid = itertools.product(*(map(int, v.split(",")) for v in (a.ufi, a.ufk, a.T, a.warps, a.colf)))
        for ufi, ufk, T, w, cf in grid:
            try:
                pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n,
                                       ufi=ufi, ufk=ufk, T=T, cta_warps=w, colf=cf,
                                       packed=1 if a.packed else 0)
            except escs.EscsError:
                continue
            if a.packed:
                pv = escs.escs_pack(pl, dv, None, stream)
                fn = lambda: escs.escs_spmm_packed(pl, pv, dB, dC, stream)
            else:
                fn = lambda: escs.escs_spmm(pl, dv, dB, dC, stream)
            t = bench.graph_time(torch, fn, stream, min_ms=1.0, reps=5)
            inf = pl.info
            cfg = {"h": ufi, "ufk": inf["ufk"], "T": inf["T"], "cta_warps": inf["cta_warps"],
                   "colf": inf["colf"], "n_tiles": inf["n_tiles"], "n_heavy": inf["n_heavy"]}
            rec["grid"].append([1e3 * t, cfg])
            if t < best[0]:
                best = (t, cfg)
            pl.close()
        rec["best_us"] = 1e3 * best[0]
        rec["best"] = best[1]
        out.append(rec)
        print(f"{p.name:28s} auto {rec['auto_us']:7.2f} best {rec['best_us']:7.2f} {best[1]}",
              flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print("tune seconds", time.time() - t0)


if __name__ == "__main__":
    main()
