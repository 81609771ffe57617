"""Instructions executed and stall samples per source REGION of a kernel (profiling helper, not
product code).  Like sass_lines.py, but every instruction is attributed to the OUTERMOST line of
the given source file in its inline chain (`nvdisasm -gi`), so inlined helpers and lambdas count
at their call site in the kernel body.

usage: sass_regions.py SASS.csv CUBIN FUNCTION_MANGLED FILE 'name:lo-hi,name:lo-hi,...' [--innermost]
(--innermost: attribute to the innermost line of FILE instead, for kernels built of lambdas)"""
import collections
import csv
import re
import subprocess
import sys

LINE = re.compile(r'//## File "([^"]+)", line (\d+)(.*)')
INL = re.compile(r'inlined at "([^"]+)", line (\d+)')


def outer_map(cubin, fn, fname, innermost=False):
    """instruction index -> line of `fname` (outermost, or innermost) of the longest inline
    chain among the line comments nvdisasm prints before that instruction"""
    txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    out, inside, best, last = [], False, None, None
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = ln.strip() == f".text.{fn}:"
            best = None
            continue
        if not inside:
            continue
        m = LINE.search(ln)
        if m:
            chain = [(m.group(1), int(m.group(2)))] + [(f, int(l)) for f, l in INL.findall(m.group(3))]
            if best is None or len(chain) > len(best):
                best = chain
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[^.]", ln) and "/*" in ln:
            if best is not None:  # line entries are sticky: no comment = the previous line
                last = best
            hits = [l for f, l in (last or []) if f.endswith(fname)]
            out.append((hits[0] if innermost else hits[-1]) if hits else None)
            best = None
    return out


def main():
    csvp, cubin, fn, fname, spec = sys.argv[1:6]
    innermost = "--innermost" in sys.argv
    regions = []
    for item in spec.split(","):
        nm, rng = item.split(":")
        lo, hi = rng.split("-")
        regions.append((nm, int(lo), int(hi)))
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    lm = outer_map(cubin, fn, fname, innermost)
    if len(lm) != len(body):
        print(f"warning: {len(lm)} disassembled vs {len(body)} profiled instructions", file=sys.stderr)
    samp, inst = collections.Counter(), collections.Counter()
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    rs = collections.defaultdict(collections.Counter)
    for k, r in enumerate(body[: len(lm)]):
        l = lm[k]
        name = "other"
        if l is not None:
            for nm, lo, hi in regions:
                if lo <= l <= hi:
                    name = nm
        samp[name] += int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
        inst[name] += int(float(r[ix["Instructions Executed"]] or 0))
        for x in reasons:
            rs[name][x] += int(float(r[ix[x]] or 0))
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    for nm in sorted(samp, key=lambda x: -samp[x]):
        top = ", ".join(f"{k[6:]}={v * 100 / ts:.1f}" for k, v in rs[nm].most_common(3) if v)
        print(f"{nm:10s} samples {100 * samp[nm] / ts:5.1f}%  inst {100 * inst[nm] / ti:5.1f}%  ({top})")


if __name__ == "__main__":
    main()
