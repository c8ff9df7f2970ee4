"""Summarise an ncu launch list (--csv, metrics gpu__time_duration.sum and
optionally dram__bytes_read.sum / dram__bytes_write.sum) per kernel name:
launches, total ns, share of the captured region, DRAM bytes per launch.

usage: python tools/launch_summary.py launches.csv [header-line ...] > summary.txt
"""
import csv
import io
import re
import sys
from collections import defaultdict


def main(path, *header):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: {"ns": 0.0, "dram": 0.0, "ids": set()})
    for r in rows:
        name = re.sub(r"\(.*$", "", r["Kernel Name"]).replace("std::array<char *, 1>>", "").strip()
        name = name.replace("at::", "").replace("<unnamed>", "<unnamed>")[:80]
        e = per[name]
        e["ids"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            e["ns"] += v * (1000.0 if r["Metric Unit"] == "usecond" else 1.0)
        elif r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
            e["dram"] += v * scale
    total = sum(e["ns"] for e in per.values())
    for h in header:
        print("# " + h)
    print("kernel | launches | total_ns | share_of_region | dram_bytes_per_launch")
    esc_n = esc_ns = esc_dram = 0
    for name, e in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        n = len(e["ids"])
        print(f"{name} | {n} | {e['ns']:.0f} | {e['ns'] / total:.3f} | {e['dram'] / n:.0f}")
        if "esc_spmm" in name:
            esc_n += n; esc_ns += e["ns"]; esc_dram += e["dram"]
    if esc_n:
        print(f"# esc_spmm kernels, all instances: {esc_n} launches, {esc_ns / 1e3:.1f} us total "
              f"({esc_ns / esc_n / 1e3:.2f} us per launch), share {esc_ns / total:.3f}; "
              f"DRAM {esc_dram / esc_n:.0f} B per launch")


if __name__ == "__main__":
    main(*sys.argv[1:])
