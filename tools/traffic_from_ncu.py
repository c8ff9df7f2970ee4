"""Summarise an ncu per-launch DRAM capture (tools/gpu_round.sh *_dram.csv) into
profiles/traffic.json, which bench.py reports as roofline.traffic (DRAM bytes
per escs_spmm launch, averaged over the launches of one bench step)."""
import csv
import json
import sys


def main(src, dst, workload="transformer"):
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
        if "esc_spmm_kernel" not in d["Kernel Name"]:
            continue
        per.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    launches = len(per)
    tot = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
    out = {"workload": workload, "launches": launches,
           "dram_bytes_per_launch": tot / max(launches, 1),
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one bench step ({src})"}
    json.dump(out, open(dst, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
