"""Register / spill summary of the built kernel instances (ptxas -v logs).

    python tools/regs.py [filter]      e.g. python tools/regs.py "L=16 F=8"
"""
import glob
import os
import re
import sys

BUILD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2506_15174_b200", "build")
MODES = {0: "csr", 1: "probe", 2: "rec", 3: "recprobe"}


def main():
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    for log in sorted(glob.glob(os.path.join(BUILD, "k_*.cu.o.log"))):
        txt = open(log).read()
        for m in re.finditer(r"Compiling entry function '(\w+)'(.*?)Used (\d+) registers", txt, re.S):
            name, spill, regs = m.group(1), m.group(2), m.group(3)
            k = re.search(r"esc_(?:spmm|rec)_kernelILi(\d)ENS0_(\d+)(VecMap|ScalarMap)ILi(\d+)E(?:Li(\d+)E)?EELi(\d)ELi(\d)E", name)
            if not k:
                continue
            h, mp, L, F, U, md = k.group(1), k.group(3), k.group(4), k.group(5), k.group(6), int(k.group(7))
            sp = re.search(r"(\d+) bytes spill stores", spill)
            line = f"h={h} {mp} L={L} F={F} U={U} {MODES[md]:8s} regs={regs} spill={sp.group(1) if sp else '?'}"
            if flt in line:
                try:
                    print(line)
                except BrokenPipeError:
                    return


if __name__ == "__main__":
    main()
