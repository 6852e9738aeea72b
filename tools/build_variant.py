"""Build a variant of libgvom.so for A/B timing (GVOM_LIBRARY=<path> selects it).

  python tools/build_variant.py NAME [--rev GIT_REV | --src DIR] [-DMACRO ...]

Sources come from the working tree, or from GIT_REV (git show) when given.
The library lands in paper_2109_13176_b200/lib/variants/NAME.so (git-ignored,
travels to the GPU box with the snapshot).
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_13176_b200 import build_ext as B  # noqa: E402


def main():
    name = sys.argv[1]
    rev = None
    srcdir = None
    defs = []
    args = sys.argv[2:]
    while args:
        a = args.pop(0)
        if a == "--rev":
            rev = args.pop(0)
        elif a == "--src":
            srcdir = args.pop(0)
        elif a.startswith("-D"):
            defs.append(a)
    src = srcdir or B.CSRC
    tmpd = tempfile.mkdtemp()
    if rev:
        src = tmpd
        for f in B.SOURCES + B.HEADERS:
            rel = os.path.relpath(os.path.join(B.CSRC, f), ROOT)
            with open(os.path.join(tmpd, f), "wb") as fh:
                fh.write(subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:{rel}"]))
    outdir = os.path.join(B.LIBDIR, "variants")
    os.makedirs(outdir, exist_ok=True)
    objs = []
    for f in B.SOURCES:
        o = os.path.join(tmpd, f.replace(".cu", ".o"))
        subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, *defs, "-I", src, "-c",
                               os.path.join(src, f), "-o", o])
        objs.append(o)
    out = os.path.join(outdir, name + ".so")
    subprocess.check_call([B.nvcc(), "-shared", "-cudart", "static", "-gencode",
                           "arch=compute_100a,code=sm_100a", *objs, "-o", out])
    print(out)


if __name__ == "__main__":
    main()
