"""Registers and spills per kernel from `nvcc -Xptxas -v` output on stdin (profiling helper).
usage: nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_regs.py [substring]"""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", ln)
    if m and cur:
        spill = int(m.group(1))
        continue
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        name = subprocess.run(["c++filt"], input=cur, capture_output=True, text=True).stdout.strip()
        if pat in name:
            print(f"{int(m.group(1)):4d} regs {spill:4d} B spill  {name[:150]}")
        cur = None
