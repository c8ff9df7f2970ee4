"""Summarise an ncu per-launch DRAM capture (tools/gpu_round.sh *_dram.csv) into
profiles/traffic.json, which bench.py reports as roofline.traffic (DRAM bytes
per escs_spmm launch, averaged over the launches of one bench step)."""
import csv
import json
import sys


def main(src, dst, workload="suite", case=None):
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = {}
    for d in data:
        if not any(x in d["Kernel Name"] for x in ("esc_spmm_kernel", "esc_rec_kernel", "esc_staged_kernel")):
            continue
        per.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    launches = len(per)
    dram = [v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
            for _, v in sorted(per.items(), key=lambda kv: int(kv[0]))]
    out = {"workload": workload, "launches": launches,
           "step_mean_dram_bytes_per_launch": sum(dram) / max(launches, 1),
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one bench step ({src})"}
    if case is not None:
        # the dominant layer's launch: its index in the workload's problem order
        import os
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        names = [p.name for p in bench.workload(workload)[0]]
        idx = names.index(case)
        out.update(case=case, launch_index=idx, dram_bytes_per_launch=dram[idx])
    else:
        out["dram_bytes_per_launch"] = out["step_mean_dram_bytes_per_launch"]
    json.dump(out, open(dst, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
