"""Summarise an `ncu --page source --print-source sass --csv` dump: instructions executed
per opcode and the top stall-sampled instructions (profiling helper, not product code)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
ops, stall = Counter(), []
tot = 0
for r in body:
    try:
        n = int(float(r[ix["Instructions Executed"]] or 0))
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    tot += n
    s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    stall.append((s, r[ix["Address"]], src, n))
print("total warp instructions", tot)
for op, n in ops.most_common(40):
    print(f"{op:12s} {n:12d} {100.0 * n / tot:6.2f}%")
stall.sort(reverse=True)
ts = sum(s for s, *_ in stall)
print("\ntop stall-sampled instructions (of", ts, "samples)")
for s, a, src, n in stall[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100.0 * s / ts:5.1f}% {a} {src[:90]}  x{n}")

# per-reason top instructions
if len(sys.argv) > 3:
    for reason in sys.argv[3].split(","):
        col = ix.get(reason)
        if col is None:
            continue
        lst = []
        for r in body:
            try:
                s = int(float(r[col] or 0))
            except ValueError:
                continue
            lst.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()))
        lst.sort(reverse=True)
        tot_r = sum(s for s, *_ in lst)
        print(f"\n== {reason}: {tot_r} samples")
        for s, a, src in lst[:12]:
            print(f"{100.0 * s / max(tot_r, 1):5.1f}% {a} {src[:100]}")
