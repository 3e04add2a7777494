"""Import the reference package (/root/reference/pkg) for golden-vector
generation IN THIS CONTAINER ONLY.  The reference is read-only, so it is
copied to /tmp and its Cython extension compiled there with the system gcc
(the default toolchain cannot link -fopenmp).  Nothing under
tests/ imports this module at test time; only make_golden.py does."""

import os
import shutil
import subprocess
import sys

REF = "/root/reference/pkg"
SCRATCH = "/tmp/wfpg_ref"


def import_reference():
    if not os.path.isdir(REF):
        raise RuntimeError("the reference is not available on this machine")
    so_dir = os.path.join(SCRATCH, "src", "wfpg")
    have = os.path.isdir(so_dir) and any(f.startswith("_kernels") and f.endswith(".so")
                                         for f in os.listdir(so_dir))
    if not have:
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree(REF, SCRATCH)
        env = dict(os.environ, CC="/usr/bin/gcc", LDSHARED="/usr/bin/gcc -shared")
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       env=env, check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    os.environ.setdefault("WFPG_THREADS", "1")
    import wfpg  # noqa: F401

    return wfpg
