"""Registers / spills per kernel from paper_1511_03296_b200/ptxas_info.txt: python scripts/regs.py [regex]"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
txt = open("paper_1511_03296_b200/ptxas_info.txt").read().splitlines()
cur = None
for i, l in enumerate(txt):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", l)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", l)
    if m and cur and pat.search(cur):
        print(f"{int(m.group(1)):4d} regs {spill:16s} {cur[:110]}")
