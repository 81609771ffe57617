"""Build a variant of libntc.so for A/B timing (profiling helper, not product code):
  python tools/build_variant.py OUT.so FILE.cu [-DNAME=VALUE ...]
recompiles FILE.cu (csrc/) with the extra defines and links it with the other objects of the
in-tree build (paper_2305_17105_b200/build/*.o, built by build.py)."""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17105_b200 import build as B  # noqa: E402


def main():
    out, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    if "--no-base" not in defs:
        B.build()
    defs = [d for d in defs if d != "--no-base"]
    srcp = os.path.join(B.HERE, "csrc", src)
    stem = os.path.splitext(src)[0]
    tag = os.path.splitext(os.path.basename(out))[0]
    vdir = os.path.join(B.OBJDIR, "variants")
    os.makedirs(vdir, exist_ok=True)
    obj = os.path.join(vdir, f"{stem}.{tag}.o")
    subprocess.check_call([B.NVCC, *B.FLAGS, *defs, "-c", "-o", obj, srcp])
    objs = [o for o in glob.glob(os.path.join(B.OBJDIR, "*.o")) if os.path.basename(o) != f"{stem}.o"]
    subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, obj, *objs])


if __name__ == "__main__":
    main()
