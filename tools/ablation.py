"""Ablation on B200 (paper Fig. 7: Base / +Enumeration /
+Coarsening, GFLOP/s over random matrices), with this build's knobs:

  base       UFi 1, UFk 2, one item per row (T = inf), 1 warp per CTA
             (Fig. 2a: one C row per block of 32 threads)
  +enum      UFi 4 (enumerated row panels), otherwise as base
  +coarsen   UFi 4, UFk 8, balanced items (T auto), 8-warp tiles
  tuned      the parameter table (escs_plan defaults)

Hot-L2 CUDA-graph timing (bench.graph_time) on 25 magnitude-pruned
matrices (sizes from the Transformer/ResNet suites, sparsity 70-98%),
bCols 64.

    python tools/ablation.py [--out gpurun_out/ablation.json]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "base": dict(ufi=1, ufk=2, T=1 << 20, cta_warps=1),
    "+enum": dict(ufi=4, ufk=2, T=1 << 20, cta_warps=1),
    "+coarsen": dict(ufi=4, ufk=8, cta_warps=8),
    "tuned": None,
}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/ablation.json")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--count", type=int, default=25)
    a = ap.parse_args(argv)
    import numpy as np
    import torch
    import bench
    from paper_2506_15174_b200 import escs, synth
    rng = np.random.default_rng(2506)
    shapes = list(synth.TRANSFORMER_SHAPES + synth.RESNET_SHAPES)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rows = []
    for i in range(a.count):
        m, k = shapes[int(rng.integers(len(shapes)))]
        s = float(rng.choice(synth.SPARSITIES))
        A = synth.magnitude_pruned(m, k, s, 5000 + i)
        B = synth.dense_b(k, a.n, 6000 + i)
        dv, dB = torch.from_numpy(A.vals).cuda(), torch.from_numpy(B).cuda()
        dC = torch.empty(m, a.n, device="cuda")
        rec = {"m": m, "k": k, "s": s, "nnz": A.nnz}
        for name, prm in VARIANTS.items():
            pl = (escs.escs_plan(m, k, A.nnz, A.rowptr, A.colidx, a.n) if prm is None else
                  escs.escs_plan_ex(m, k, A.nnz, A.rowptr, A.colidx, a.n, **prm))
            t = bench.graph_time(torch, lambda: escs.escs_spmm(pl, dv, dB, dC, stream), stream,
                                 min_ms=1.0, reps=5)
            rec[name] = 2 * A.nnz * a.n / (t * 1e-3) / 1e9
            pl.close()
        rows.append(rec)
        print(rec, flush=True)
    geo = {n: math.exp(sum(math.log(r[n]) for r in rows) / len(rows)) for n in VARIANTS}
    out = {"bcols": a.n, "gflops_geomean": geo, "rows": rows,
           "speedup_vs_base": {n: geo[n] / geo["base"] for n in VARIANTS}}
    print(json.dumps(out["gflops_geomean"]), json.dumps(out["speedup_vs_base"]))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
