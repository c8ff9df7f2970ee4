"""Staged-walk parameter sweep on one suite layer (hot L2, bench.py graph_time
protocol) beside the tuned L2-gather record walk; every candidate is checked
against the fp64 oracle (G2) first.

    python tools/staged_sweep.py --case "512x4608@70%/b128" [--quick]
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", default=[])
    ap.add_argument("--hs", default="1,2,3,4,6,8")
    ap.add_argument("--warps", default="8,16")
    ap.add_argument("--npw", default="1,2")
    ap.add_argument("--nsplit-f", default="0.5,1,2")
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", default=None, help="h,W,npw,ns;... explicit staged plans (no sweep)")
    ap.add_argument("--no-gather", action="store_true")
    a = ap.parse_args()
    import torch
    import bench
    import oracle
    from paper_2506_15174_b200 import escs
    probs = {q.name: q for wl in ("transformer", "resnet") for q in bench.workload(wl)[0]}
    stream = torch.cuda.Stream()
    res = []
    for name in a.case or ["512x4608@70%/b128"]:
        p = probs[name]
        A, n = p.A, p.bcols
        ref = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, p.B)
        dv, dB = torch.from_numpy(A.vals).cuda(), torch.from_numpy(p.B).cuda()
        dC = torch.empty(A.m, n, device="cuda")

        def run(pl):
            pk = escs.escs_pack(pl, dv)
            dC.fill_(float("nan"))
            escs.escs_spmm_packed(pl, pk, dB, dC)
            torch.cuda.synchronize()
            C = dC.cpu().numpy().astype(np.float64)
            err = float(np.max(np.abs(C - ref) / np.maximum(np.abs(ref), 1.0)))
            t = bench.graph_time(torch, lambda: escs.escs_spmm_packed(pl, pk, dB, dC, stream=stream), stream)
            return t, err

        tb = float("nan")
        if not a.no_gather:
            base = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, autotune=1, packed=1, staged=1)
            tb, eb = run(base)
            print(f"{name} gather-walk tuned: {tb*1e3:.2f} us err {eb:.1e} {base.info['h']}", flush=True)
            res.append({"case": name, "walk": "gather", "us": tb * 1e3, "err": eb, "h": base.info["h"]})
        best = None
        if a.configs:
            for cfg in a.configs.split(";"):
                v = [int(x) for x in cfg.split(",")]
                h, W, npw, ns = v[:4]
                colf = v[4] if len(v) > 4 else 0
                kb = v[5] if len(v) > 5 else 0
                try:
                    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=h, packed=1, staged=2,
                                           st_warps=W, st_npw=npw, st_nsplit=ns, colf=colf, st_kb=kb)
                except escs.EscsError as ex:
                    print(f"  {name} h{h} W{W} npw{npw} ns{ns}: {ex}", flush=True)
                    continue
                try:
                    t, err = run(pl)
                except escs.EscsError as ex:
                    print(f"  {name} h{h} W{W} npw{npw}: {ex}", flush=True)
                    continue
                print(f"  {name} h{h} W{W} npw{npw} ns{pl.info['st_nsplit']} kb{pl.info['st_kb']} F{pl.info['colf']} ctas {pl.info['st_ctas']} L{pl.info['st_launches']} "
                      f"{t*1e3:7.2f} us err {err:.1e}", flush=True)
                res.append({"case": name, "h": h, "warps": W, "npw": npw, "nsplit": ns, "us": t * 1e3, "err": err})
                pl.close()
            continue
        for h, W, npw in itertools.product(*(list(map(int, x.split(","))) for x in (a.hs, a.warps, a.npw))):
            try:
                auto = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=h, packed=1, staged=2,
                                         st_warps=W, st_npw=npw)
            except escs.EscsError as e:
                continue
            ns0 = auto.info["st_nsplit"]
            auto.close()
            for f in map(float, a.nsplit_f.split(",")):
                ns = max(1, int(round(ns0 * f)))
                try:
                    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, ufi=h, packed=1, staged=2,
                                           st_warps=W, st_npw=npw, st_nsplit=ns)
                except escs.EscsError as e:
                    continue
                t, err = run(pl)
                i = pl.info
                r = {"case": name, "walk": "staged", "h": h, "warps": W, "npw": npw, "nsplit": ns,
                     "ctas": i["st_ctas"], "kb": i["st_kb"], "smem": i["st_smem_bytes"], "launches": i["st_launches"], "us": t * 1e3, "err": err}
                res.append(r)
                ok = err <= 1e-4
                print(f"  h{h} W{W} npw{npw} ns{ns:3d} ctas {i['st_ctas']:4d} smem {i['st_smem_bytes']//1024:3d}K "
                      f"L{i['st_launches']} {t*1e3:7.2f} us err {err:.1e}{'' if ok else ' FAIL'}", flush=True)
                if ok and (best is None or t < best[0]):
                    best = (t, r)
                pl.close()
        if best:
            print(f"BEST {name}: {best[0]*1e3:.2f} us vs gather {tb*1e3:.2f} us  {best[1]}", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
