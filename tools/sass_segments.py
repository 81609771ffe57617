"""Split an ncu SASS source dump at LDTM/UTCHMMA/BAR/LDG/STG/SYNCS markers and print the
per-segment instruction count normalised by a unit count (profiling helper)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
unit = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seq = []
for r in rows[2:]:
    try:
        n = int(float(r[ix["Instructions Executed"]] or 0))
    except ValueError:
        continue
    seq.append((r[ix["Address"]][-5:], n, r[ix["Source"]].strip()))
keys = ("LDTM", "UTCHMMA", "BAR.", "LDG", "STG", "SYNCS.PHASECHK", "STS")
prev = 0
for i, (a, n, s) in enumerate(seq):
    if any(k in s for k in keys):
        seg = seq[prev:i]
        cnt = sum(x[1] for x in seg)
        if cnt / unit >= 0.5:
            print(f"{seq[prev][0]}..{a} n={len(seg):4d} exec={cnt / unit:7.1f}  -> {s[:70]}")
        prev = i
