"""ctypes binding of libwfpg_b200.so (the C ABI declared in include/wfpg_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2405_06997_b200/csrc``).  There is no CPU fallback: loading
fails loudly when the library is missing, and every call that returns a
non-zero status raises.
"""

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# WFPG_LIB overrides the library path (A/B measurements of alternative builds)
LIB_PATH = os.environ.get("WFPG_LIB") or os.path.join(_HERE, "libwfpg_b200.so")

c_i32 = C.c_int32
c_i64 = C.c_int64
c_u64 = C.c_uint64
c_dbl = C.c_double
c_vp = C.c_void_p
c_size = C.c_size_t


class Scene(C.Structure):
    _fields_ = [
        ("n_tris", c_i32),
        ("v0", c_vp), ("v1", c_vp), ("v2", c_vp), ("e1", c_vp), ("e2", c_vp),
        ("normals", c_vp), ("tri_mat", c_vp), ("mat_kind", c_vp), ("mat_rgb", c_vp),
        ("n_mats", c_i32), ("n_emit", c_i32),
        ("emitter_cdf", c_vp), ("emitter_tris", c_vp),
        ("emitter_area", c_dbl), ("ray_eps", c_dbl),
        ("bbox_lo", c_dbl * 3), ("bbox_hi", c_dbl * 3),
        ("bvh_nodes", c_i32),
        ("bvh_lo", c_vp), ("bvh_hi", c_vp), ("bvh_left", c_vp), ("bvh_right", c_vp),
        ("bvh_count", c_vp), ("bvh_order", c_vp),
        ("brute", c_i32), ("bvh_box_f32", c_vp),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("position", c_dbl * 3), ("forward", c_dbl * 3), ("right", c_dbl * 3),
        ("up", c_dbl * 3), ("tan_half", c_dbl), ("width", c_i32), ("height", c_i32),
    ]


class Svo(C.Structure):
    _fields_ = [
        ("depth", c_i32), ("resolution", c_i32), ("n_nodes", c_i64),
        ("lo", c_dbl * 3), ("size", c_dbl), ("level_off", c_i64 * 32),
        ("codes", c_vp), ("child_base", c_vp), ("child_mask", c_vp), ("parent", c_vp),
        ("node_desc", c_vp), ("normal", c_vp), ("sum_a", c_vp), ("sum_b", c_vp),
        ("weight_a", c_vp), ("weight_b", c_vp), ("mean_a", c_vp), ("mean_b", c_vp),
        ("counter", c_vp), ("top_index", c_vp), ("top_level", c_i32),
    ]


class Paths(C.Structure):
    _fields_ = [
        ("n", c_i64), ("max_depth", c_i32),
        ("ray_o", c_vp), ("ray_d", c_vp), ("beta", c_vp), ("radiance", c_vp),
        ("key", c_vp), ("ctr", c_vp), ("alive", c_vp), ("prev_pdf", c_vp),
        ("rec_pos", c_vp), ("rec_T", c_vp), ("emit_le", c_vp), ("emit_depth", c_vp),
        ("n_rec", c_vp), ("rec_depth_major", c_i32),
    ]


class Guide(C.Structure):
    _fields_ = [
        ("mode", c_i32), ("n", c_i32), ("capacity", c_i32), ("eps", c_dbl),
        ("vals", c_vp), ("row_sum", c_vp), ("marg", c_vp), ("total", c_vp),
        ("block_sums", c_vp), ("n_bins", c_vp), ("upper_dirs", c_vp), ("cum", c_vp),
        ("block_rows", c_vp),
    ]


class PassConfig(C.Structure):
    _fields_ = [
        ("l_min", c_i32), ("c_ray", c_i32), ("field_res", c_i32), ("guided_depths", c_i32),
        ("max_depth", c_i32), ("product", c_i32), ("jitter", c_i32),
        ("blur_sigma", c_dbl), ("epsilon", c_dbl),
        ("russian_roulette", c_i32), ("rr_depth", c_i32),
        ("seed", c_u64), ("sample_index", c_i64), ("n_samples", c_i32),
        ("deterministic", c_i32),
        ("blur_radius", c_i32), ("blur_w", c_dbl * 33), ("upper_dirs", c_vp),
        ("pixel_offset", c_i64), ("n_pixels", c_i64), ("leaf_acc", c_vp),
        ("use_graph", c_i32),
        ("bin_image", c_vp),
        ("dep_leaf", c_vp),
        ("dep_dir", c_vp),
        ("dep_rad", c_vp),
        ("dep_count", c_vp),
        ("dep_capacity", c_i64),
        ("comm", c_vp),
        ("dep_wire_capacity", c_i64),
        ("sample_list", c_vp),
        ("own_bins", c_i32 * 32),
        ("ev_wait_counters", c_vp), ("ev_wait_svo", c_vp),
        ("ev_rec_counters", c_vp), ("ev_rec_svo", c_vp), ("skip_unguided_bins", c_i32),
    ]


# host exchange callback (include/wfpg_b200.h wfpg_exchange_fn)
EXCHANGE_FN = C.CFUNCTYPE(c_i32, c_vp, c_i32, c_vp, c_vp, c_i64, c_i32, c_vp)

# struct ids of wfpg_abi_sizeof / wfpg_abi_offsetof
ABI_STRUCTS = {0: "Scene", 1: "Camera", 2: "Svo", 3: "Paths", 4: "Guide", 5: "PassConfig",
               6: "PassStats"}


class PassStats(C.Structure):
    _fields_ = [
        ("depths_run", c_i32),
        ("bins_per_depth", c_i32 * 32),
        ("rays_per_depth", c_i32 * 32),
        ("live_per_depth", c_i32 * 32),
        ("deposits", c_i32),
        ("mat_groups", (c_i32 * 64) * 32),
    ]


P = C.POINTER
_SIGS = {
    "wfpg_abi_version": (c_i32, []),
    "wfpg_last_error": (C.c_char_p, []),
    "wfpg_launch_count": (c_u64, []),
    "wfpg_abi_sizeof": (c_i64, [c_i32]),
    "wfpg_abi_offsetof": (c_i64, [c_i32, C.c_char_p]),
    "wfpg_memcpy": (c_i32, [c_vp, c_vp, c_size, c_vp]),
    "wfpg_event_create": (c_i32, [P(c_vp)]),
    "wfpg_event_destroy": (c_i32, [c_vp]),
    "wfpg_comm_nccl_available": (c_i32, []),
    "wfpg_comm_nccl_unique_id": (c_i32, [c_vp]),
    "wfpg_comm_init_nccl": (c_i32, [c_i32, c_i32, c_vp, P(c_vp)]),
    "wfpg_comm_init_host": (c_i32, [c_i32, c_i32, c_vp, c_vp, P(c_vp)]),
    "wfpg_comm_settle": (c_i32, [c_vp]),
    "wfpg_comm_destroy": (c_i32, [c_vp]),
    "wfpg_scan_workspace_bytes": (c_size, [c_i64]),
    "wfpg_scan_u32": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_size, c_vp]),
    "wfpg_sort_workspace_bytes": (c_size, [c_i64]),
    "wfpg_sort_pairs_u64": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_size, c_vp]),
    "wfpg_voxelize_workspace_bytes": (c_size, [c_i32, c_i64]),
    "wfpg_voxelize_count": (c_i32, [P(Scene), c_vp, c_dbl, c_i32, P(c_i64), c_vp, c_size, c_vp]),
    "wfpg_voxelize_emit": (c_i32, [P(Scene), c_vp, c_dbl, c_i32, c_i64, c_vp, c_vp, c_i64,
                                   P(c_i64), c_vp, c_size, c_vp]),
    "wfpg_svo_build_workspace_bytes": (c_size, [c_i64, c_i32]),
    "wfpg_svo_build_structure": (c_i32, [P(Svo), c_vp, c_i64, c_vp, c_size, c_vp]),
    "wfpg_svo_build_structure_points": (c_i32, [P(Svo), c_vp, c_i64, c_vp, c_size, c_vp]),
    "wfpg_svo_build_fill": (c_i32, [P(Svo), c_vp, c_vp, c_i64, c_u64, c_vp, c_size, c_vp]),
    "wfpg_svo_build_sorted": (c_i32, [c_vp, c_i64, P(c_vp), P(c_vp)]),
    "wfpg_descend": (c_i32, [P(Svo), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "wfpg_bvh_build_host": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_vp]),
    "wfpg_bvh_build_workspace_bytes": (c_size, [c_i64]),
    "wfpg_bvh_build_device": (c_i32, [P(Scene), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_size, c_vp]),
    "wfpg_svo_top_index_bytes": (c_size, [c_i32]),
    "wfpg_svo_build_top_index": (c_i32, [P(Svo), c_vp]),
    "wfpg_svo_refresh_leaves": (c_i32, [P(Svo), c_vp, c_i64, c_vp, c_vp]),
    "wfpg_graph_release": (c_i32, [c_vp]),
    "wfpg_frame_accumulate": (c_i32, [c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "wfpg_quantise_points": (c_i32, [c_vp, c_dbl, c_i32, c_vp, c_i64, c_vp, c_vp]),
    "wfpg_accumulate_workspace_bytes": (c_size, [c_i64]),
    "wfpg_svo_accumulate": (c_i32, [P(Svo), c_vp, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_size,
                                    c_vp]),
    "wfpg_svo_propagate": (c_i32, [P(Svo), c_vp]),
    "wfpg_svo_apply_leaf_acc": (c_i32, [P(Svo), c_vp, c_vp]),
    "wfpg_update_exitance_workspace_bytes": (c_size, [c_i64, c_i32]),
    "wfpg_update_exitance": (c_i32, [P(Svo), P(Paths), c_i32, c_vp, c_vp, c_size, c_vp]),
    "wfpg_trace_cones": (c_i32, [P(Scene), P(Svo), c_vp, c_i32, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "wfpg_generate_fields": (c_i32, [P(Scene), P(Svo), c_vp, c_vp, c_i64, c_vp, c_i32,
                                     c_i32, P(c_dbl), P(Guide), c_vp]),
    "wfpg_guide_fill": (c_i32, [P(Guide), c_i64, c_vp]),
    "wfpg_guide_expand": (c_i32, [P(Guide), c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "wfpg_camera_rays": (c_i32, [P(Camera), c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "wfpg_intersect": (c_i32, [P(Scene), c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp]),
    "wfpg_occluded": (c_i32, [P(Scene), c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp]),
    "wfpg_shade_depth": (c_i32, [P(Scene), P(Paths), c_i32, c_vp, c_i64, c_vp, c_vp, c_vp,
                                 P(Guide), c_vp, c_i32, c_i32, c_vp]),
    "wfpg_partition_workspace_bytes": (c_size, [c_i64, c_i64]),
    "wfpg_partition_spatial": (c_i32, [P(Svo), c_vp, c_vp, c_i64, c_vp, c_i32, c_i32, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_i64, c_vp, c_size, c_vp]),
    "wfpg_render_workspace_bytes": (c_size, [P(Scene), P(Svo), P(Camera), P(PassConfig)]),
    "wfpg_render_pass": (c_i32, [P(Scene), P(Svo), P(Camera), P(PassConfig), P(Paths), c_vp,
                                 P(PassStats), c_vp, c_size, c_vp]),
    "wfpg_profile_enable": (c_i32, [c_i32]),
    "wfpg_profile_read": (c_i32, [P(c_dbl), P(c_dbl), P(c_i64), c_i32]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class WfpgError(RuntimeError):
    pass


def load():
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise WfpgError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            MISSING.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


MISSING = []


def check(status, what=""):
    if status != 0:
        msg = load().wfpg_last_error().decode(errors="replace")
        if status == 1:
            raise ValueError(f"{what}: {msg}")
        raise WfpgError(f"{what} failed ({status}): {msg}")


def call(name, *args):
    status = getattr(load(), name)(*args)
    check(status, name)
    return status


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def launch_count():
    return int(load().wfpg_launch_count())
