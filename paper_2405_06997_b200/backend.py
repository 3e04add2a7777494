"""Backend selection with the reference's API (backend.py:1-49).

The B200 build has exactly one backend: the CUDA kernels (backend_cuda).
``set_backend`` exists for API compatibility (tests swap modules); there is
no pure-Python fallback, so WFPG_PURE_PYTHON is rejected loudly.
"""

import os

from . import backend_cuda

if os.environ.get("WFPG_PURE_PYTHON", "") == "1":
    raise RuntimeError("WFPG_PURE_PYTHON=1: the B200 build has no CPU fallback")

_active = backend_cuda


def get():
    return _active


def set_backend(module):
    global _active
    _active = module


def compiled_available():
    return True


def workers():
    """Kept for API parity; device kernels ignore host worker counts."""
    env = os.environ.get("WFPG_THREADS")
    return max(1, int(env)) if env else 1
