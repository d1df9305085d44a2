"""Registers and spills per kernel from the ptxas -v build log
(paper_2404_16990_b200/build.log).  python tools/ptxas_summary.py [filter]"""
import re
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else "k_win"
log = open("paper_2404_16990_b200/build.log").read().splitlines()
name = None
for ln in log:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        name = m.group(1)
        continue
    if name and flt in name:
        t = re.search(r"(k_\w+?)I(.*?)EEv", name)
        label = f"{t.group(1)}<{','.join(re.findall(r'L[ib](\d+)E', t.group(2)))}>" if t else name[:60]
        s = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if s:
            spill = f"spill st/ld {s.group(1)}/{s.group(2)}"
        r = re.search(r"Used (\d+) registers", ln)
        if r:
            print(f"{label:40s} regs {r.group(1):>3s}  {spill}")
            name = None
