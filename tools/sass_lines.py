"""Instructions executed and stall samples per CUDA source line (profiling helper, not product
code).  Joins an `ncu --page source --print-source sass --csv` dump (per-instruction counts)
with `nvdisasm --print-line-info` of the same cubin (instruction -> file:line), by order.

usage: sass_lines.py SASS.csv CUBIN FUNCTION_MANGLED [per_unit_divisor] [topN]"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn):
    txt = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    cur, out, inside = None, [], False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = ln.strip() == f".text.{fn}:"
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", ln):
            out.append(cur)
    return out


def main():
    csvp, cubin, fn = sys.argv[1:4]
    div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    lm = line_map(cubin, fn)
    if len(lm) != len(body):
        print(f"warning: {len(lm)} disassembled vs {len(body)} profiled instructions", file=sys.stderr)
    cnt, smp = collections.Counter(), collections.Counter()
    for k, r in enumerate(body):
        if k >= len(lm):
            break
        key = lm[k] or ("?", 0)
        cnt[key] += int(float(r[ix["Instructions Executed"]] or 0))
        smp[key] += int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    srcs = {}
    tot, tots = sum(cnt.values()), sum(smp.values()) or 1
    print(f"total {tot / div:.1f} instructions per unit, {tots} stall samples")
    for (f, l), n in cnt.most_common(top):
        if (f, l) not in srcs:
            try:
                path = next(p for p in (f"paper_2305_17105_b200/csrc/{f}",) if p)
                srcs[(f, l)] = open(path).read().splitlines()[l - 1].strip()[:80]
            except Exception:
                srcs[(f, l)] = ""
        print(f"{n / div:8.1f} {100.0 * smp[(f, l)] / tots:5.1f}%  {f}:{l:<5d} {srcs[(f, l)]}")


if __name__ == "__main__":
    main()
