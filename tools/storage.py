"""Storage study (paper Fig. 9): bytes of the ESC format
(values in traversal order "ANNZ" + group columns "Cols" + per-group pointers
"RPP"/"NPP" + per-group panel/pattern) vs CSR vs dense, over sparsity, from
the plans escs_plan builds (host-only, no GPU).

    python tools/storage.py [--out profiles/r1_storage.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def esc_bytes(hdr):
    """ANNZ 4*nnz + Cols 4*G + RPP/NPP 4*(NG+1) each + panel/pattern 4*NG each."""
    return 4 * hdr["nnz"] + 4 * hdr["G"] + 8 * (hdr["NG"] + 1) + 8 * hdr["NG"]


def csr_bytes(m, nnz):
    return 4 * nnz + 4 * nnz + 4 * (m + 1)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r1_storage.json")
    ap.add_argument("--shape", default="512x512")
    a = ap.parse_args(argv)
    from paper_2506_15174_b200 import escs, synth
    m, k = (int(x) for x in a.shape.split("x"))
    rows = []
    for s in (0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.98, 0.99, 0.995):
        A = synth.magnitude_pruned(m, k, s, 77)
        rec = {"sparsity": s, "nnz": A.nnz, "csr": csr_bytes(m, A.nnz), "dense": 4 * m * k}
        for h in (2, 3, 4, 8):
            hdr = escs.escs_plan_ex(m, k, A.nnz, A.rowptr, A.colidx, 64, ufi=h, T=1 << 20,
                                    host_only=1).export()["header"]
            rec[f"esc_ufi{h}"] = esc_bytes(hdr)
        rows.append(rec)
        print(s, {kk: v for kk, v in rec.items() if kk != "sparsity"}, flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"shape": a.shape, "rows": rows,
                   "note": "bytes; ESC = ANNZ + Cols + RPP + NPP + group panel/pattern"}, f, indent=1)


if __name__ == "__main__":
    main()
