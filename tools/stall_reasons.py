"""Per-stall-reason top instructions from an `ncu --page source --print-source sass --csv`
dump (profiling helper, not product code).  usage: stall_reasons.py CSV [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
per = {r: [] for r in reasons}
for k, row in enumerate(body):
    for r in reasons:
        try:
            v = int(float(row[ix[r]] or 0))
        except ValueError:
            v = 0
        tot[r] += v
        if v:
            per[r].append((v, k, row[ix["Address"]][-5:], row[ix["Source"]].strip()[:70]))
allt = sum(tot.values())
for r in sorted(reasons, key=lambda r: -tot[r]):
    if tot[r] * 50 < allt:
        continue
    print(f"== {r}: {tot[r]} ({100.0 * tot[r] / allt:.1f}%)")
    for v, k, a, s in sorted(per[r], reverse=True)[:top]:
        print(f"   {v:6d} #{k:5d} {a} {s}")
