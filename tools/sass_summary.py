"""Per-kernel SASS instruction-class counts of the built library (profiling helper, not product
code): static counts of the Blackwell-native instructions that prove the path runs on tcgen05 /
TMEM / TMA (UTCHMMA, LDTM / STTM, UBLKCP / UTMALDG / UTMASTG, SYNCS), plus shared / global memory
and total instructions, for each kernel of each object file.
usage: python tools/sass_summary.py OUT.json [objects...]   (default: paper_2305_17105_b200/build/*.o)"""
import glob
import json
import os
import re
import subprocess
import sys

CLASSES = {
    "UTCHMMA": r"^UTC\w*MMA", "LDTM": r"^LDTM", "STTM": r"^STTM", "UBLKCP": r"^UBLKCP", "UTMALDG": r"^UTMALDG",
    "UTMASTG": r"^UTMASTG", "SYNCS": r"^SYNCS", "STS": r"^STS", "LDS": r"^LDS", "STG": r"^STG", "LDG": r"^LDG",
    "RED": r"^RED", "SHFL": r"^SHFL", "HFMA2": r"^HFMA2", "FFMA": r"^FFMA", "FMUL2": r"^FMUL2",
}


def kernels(obj):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    out, cur = {}, None
    for ln in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            out[cur] = {k: 0 for k in CLASSES} | {"total": 0}
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if cur and m:
            op = m.group(2)
            out[cur]["total"] += 1
            for k, pat in CLASSES.items():
                if re.match(pat, op):
                    out[cur][k] += 1
    return out


def main():
    dst = sys.argv[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    objs = sys.argv[2:] or sorted(glob.glob(os.path.join(root, "paper_2305_17105_b200", "build", "*.o")))
    res = {}
    for o in objs:
        for k, v in kernels(o).items():
            res[f"{os.path.basename(o)}:{k}"] = v
    with open(dst, "w") as f:
        json.dump({"tool": "cuobjdump -sass (static instruction counts per kernel)", "kernels": res}, f, indent=1)
    # a short table of the hot kernels
    for k, v in res.items():
        if any(s in k for s in ("decode_kernel", "train_kernel", "decode_multi")) and "Li9E" in k or "Li16ELb1" in k:
            print(f"{k[:90]:90s} UTCHMMA {v['UTCHMMA']:4d} LDTM {v['LDTM']:4d} UBLKCP {v['UBLKCP']:2d} "
                  f"STS {v['STS']:4d} total {v['total']}")


if __name__ == "__main__":
    main()
