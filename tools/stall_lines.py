"""Stall samples per CUDA source line, split by reason (profiling helper, not product code).
usage: stall_lines.py SASS.csv CUBIN FUNCTION_MANGLED [topN]"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_lines import line_map  # noqa: E402


def main():
    csvp, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    lm = line_map(cubin, fn)
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    per = {r: collections.Counter() for r in reasons}
    for k, r in enumerate(body[: len(lm)]):
        key = lm[k] or ("?", 0)
        for rs in reasons:
            per[rs][key] += int(float(r[ix[rs]] or 0))
    tot = sum(sum(c.values()) for c in per.values()) or 1
    for rs in sorted(reasons, key=lambda x: -sum(per[x].values())):
        s = sum(per[rs].values())
        if s < 0.02 * tot:
            continue
        print(f"== {rs}: {100.0 * s / tot:.1f}%")
        for (f, l), n in per[rs].most_common(top):
            print(f"   {100.0 * n / tot:5.1f}%  {f}:{l}")


if __name__ == "__main__":
    main()
