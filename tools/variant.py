#!/usr/bin/env python
"""Build libwfpg_b200.so from the working tree with source edits applied to a
copy (A/B experiments; the tree itself is untouched):
    python tools/variant.py out.so 'wavefront.cu|||old text|||new text' [...]
      [--flags '-DSOMETHING']
then  tools/ab.sh "<bench args>" paper_2405_06997_b200/libwfpg_b200.so out.so"""
import argparse
import os
import shutil
import subprocess
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("edits", nargs="*")
    ap.add_argument("--flags", default="")
    a = ap.parse_args()
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "paper_2405_06997_b200", "csrc")
    shutil.copytree(os.path.join(REPO, "paper_2405_06997_b200", "csrc"), src,
                    ignore=shutil.ignore_patterns("build"))
    os.makedirs(os.path.join(tmp, "include"))
    shutil.copy(os.path.join(REPO, "include", "wfpg_b200.h"), os.path.join(tmp, "include"))
    for e in a.edits:
        fname, old, new = e.split("|||")
        p = os.path.join(src, fname)
        s = open(p).read()
        if old not in s:
            raise SystemExit(f"edit not found in {fname}: {old[:60]!r}")
        open(p, "w").write(s.replace(old, new))
    flags = ("-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a "
             "-Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -warn-spills " + a.flags)
    subprocess.run(["make", "-s", "-j16", "-C", src, f"OUT={os.path.abspath(a.out)}",
                    f"NVFLAGS={flags}"], check=True)
    shutil.rmtree(tmp)
    print("built", a.out)


if __name__ == "__main__":
    main()
