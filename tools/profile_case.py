"""Run one workload problem's escs_spmm a few times (for ncu / quick timing).

    python tools/profile_case.py --shape 2048x512 --s 0.7 --n 128 [--reps 5] [--c4|--c5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="2048x512")
    ap.add_argument("--s", type=float, default=0.7)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--config", default=None, help="c1/c4/c5 instead of a suite shape")
    ap.add_argument("--probe", action="store_true")
    ap.add_argument("--shard", default=None, help="W/R: profile rank R's row block of W (SURVEY §8(e))")
    ap.add_argument("--case", default=None, help="a problem name from bench.py's workloads")
    ap.add_argument("--no-autotune", dest="autotune", action="store_false",
                    help="plan with the parameter table (default: autotuned, as bench.py)")
    ap.add_argument("--csr", action="store_true",
                    help="the CSR-value walk (escs_spmm) instead of the packed record walk bench.py times")
    ap.add_argument("--ufi", type=int, default=0, help="force UFi (0: tuned)")
    ap.add_argument("--objective", type=int, default=1,
                    help="autotune objective: 1 latency (serial/per-case plans), 2 concurrent "
                         "throughput (the plans bench.py's multi-stream step runs)")
    ap.add_argument("--staged", default=None,
                    help="h,warps,npw,nsplit[,kb]: a staged-walk plan with these parameters")
    a = ap.parse_args()
    import torch
    from paper_2506_15174_b200 import escs, synth
    if a.case:
        import bench
        for wl in ("transformer", "resnet", "resnet50"):
            hit = [q for q in bench.workload(wl)[0] if q.name == a.case]
            if hit:
                A, B = hit[0].A, hit[0].B
                break
        else:
            raise SystemExit(f"no case {a.case}")
    elif a.config:
        p = synth.config(a.config)
        A, B = p.A, p.B
    else:
        m, k = (int(x) for x in a.shape.split("x"))
        A = synth.magnitude_pruned(m, k, a.s, 1234)
        B = synth.dense_b(k, a.n, 99)
    if a.shard:
        world, rank = (int(x) for x in a.shard.split("/"))
        r0, r1 = synth.shard_bounds(A.m, world, rank)
        A = synth.row_block(A, r0, r1)
    if a.staged:
        v = [int(x) for x in a.staged.split(",")] + [0]
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, B.shape[1], packed=1, staged=2,
                               ufi=v[0], st_warps=v[1], st_npw=v[2], st_nsplit=v[3], st_kb=v[4])
    else:
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, B.shape[1],
                               autotune=(a.objective if a.autotune and A.nnz <= 8_000_000 else 0),
                               packed=0 if a.csr else 1, ufi=a.ufi)
    print(pl.info, flush=True)
    dv, dB = torch.from_numpy(A.vals).cuda(), torch.from_numpy(B).cuda()
    pk = None if a.csr else escs.escs_pack(pl, dv)
    dC = torch.empty(A.m, B.shape[1], device="cuda")
    sink = torch.empty(max(1, pl.info["n_tiles"] * 32 * pl.info["cta_warps"]), device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("profile_reps")      # ncu --nvtx-include profile_reps/
    for i in range(a.reps):
        torch.cuda._sleep(2_000_000)   # host runs ahead: events bracket the kernel only
        s.record()
        if a.probe:
            if pk is None:
                escs.escs_gather_probe(pl, dB, sink)
            else:
                escs.escs_gather_probe_packed(pl, pk, dB, sink)
        elif pk is None:
            escs.escs_spmm(pl, dv, dB, dC)
        else:
            escs.escs_spmm_packed(pl, pk, dB, dC)
        e.record()
        torch.cuda.synchronize()
        print(f"rep {i}: {s.elapsed_time(e) * 1e3:.1f} us", flush=True)
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
