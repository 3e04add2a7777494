"""B200-native guided wavefront path tracer with sparse-voxel-octree path
guiding (arXiv 2405.06997) — drop-in for the reference package ``wfpg``'s
render path.  Hot path: hand-written sm_100a CUDA kernels behind the C ABI in
include/wfpg_b200.h (libwfpg_b200.so); torch tensors are device buffers only.
"""

__version__ = "0.1.0"

__all__ = ["accumulation", "backend", "backend_cuda", "core", "guiding", "imageio", "scene",
           "svo", "wavefront"]
