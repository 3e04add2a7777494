"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the development container (the reference tree exists only here):

    python tests/golden/make_golden.py [svo] [cones] [fields] [render] ...

Each fixture records the numpy / OpenBLAS versions it was produced with.
The GPU tests compare the CUDA path against these files; they never import
the reference.
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from _refimport import import_reference  # noqa: E402

wfpg = import_reference()
from wfpg import core, guiding, svo as rsvo, wavefront  # noqa: E402
from wfpg import scene as rscene  # noqa: E402

SCENES = "/root/reference/pkg/scenes"


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def meta():
    try:
        blas = np.show_config(mode="dicts")["Build Dependencies"]["blas"]["version"]
    except Exception:  # pragma: no cover
        blas = "unknown"
    return {"numpy": np.__version__, "blas": str(blas)}


def save(name, **arrays):
    path = os.path.join(HERE, name)
    m = meta()
    np.savez_compressed(path, _numpy=m["numpy"], _blas=m["blas"], **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def load_scene(name, w=None, h=None):
    sc = rscene.load_scene(os.path.join(SCENES, name))
    if w is not None:
        c = sc.camera
        sc.camera = rscene.Camera(c.position, c.target, c.up, c.vfov_deg, w, h)
    return sc


# ---------------------------------------------------------------------------
def gen_svo():
    """Full arrays of small builds; digests of the C1-size builds."""
    out = {}
    for tag, scene_name, res, seed in (("c64s1", "cornell.scene", 64, 1),
                                       ("e32s3", "cornell_enclosed.scene", 32, 3)):
        sc = load_scene(scene_name)
        frags = rsvo.voxelize(sc, res)
        lo, side = rsvo.scene_cube(sc)
        tree = rsvo.build_octree(frags, lo, side, res, seed)
        codes = core.morton_encode(frags.coords[:, 0], frags.coords[:, 1], frags.coords[:, 2])
        order = np.argsort(codes, kind="stable")
        out.update({
            f"{tag}_frag_coords": frags.coords.astype(np.int32),
            f"{tag}_frag_tris": frags.tris.astype(np.int32),
            f"{tag}_sorted_codes": codes[order],
            f"{tag}_sort_perm": order.astype(np.int32),
            f"{tag}_level_off": tree.level_off,
            f"{tag}_codes": tree.codes,
            f"{tag}_child_base": tree.child_base.astype(np.int32),
            f"{tag}_child_mask": tree.child_mask,
            f"{tag}_parent": tree.parent.astype(np.int32),
            f"{tag}_normal": tree.normal,
            f"{tag}_cube": np.array([*lo, side]),
        })
    # digests of the bigger builds (arrays too large to commit)
    dig = []
    for scene_name, res, seed in (("cornell.scene", 256, 0), ("cornell_enclosed.scene", 256, 0),
                                  ("cornell_enclosed.scene", 128, 3)):
        sc = load_scene(scene_name)
        frags = rsvo.voxelize(sc, res)
        lo, side = rsvo.scene_cube(sc)
        tree = rsvo.build_octree(frags, lo, side, res, seed)
        codes = core.morton_encode(frags.coords[:, 0], frags.coords[:, 1], frags.coords[:, 2])
        order = np.argsort(codes, kind="stable")
        row = [scene_name, str(res), str(seed), str(len(frags)), str(tree.node_count),
               digest(frags.coords.astype(np.int64)), digest(frags.tris.astype(np.int64)),
               digest(codes[order]), digest(order.astype(np.int64)),
               digest(tree.level_off.astype(np.int64)), digest(tree.codes),
               digest(tree.child_base.astype(np.int64)), digest(tree.child_mask),
               digest(tree.parent.astype(np.int64)), digest(tree.normal)]
        dig.append(",".join(row))
        print(row)
    out["digests"] = np.array(dig)
    out["digest_fields"] = np.array(
        "scene,res,seed,frags,nodes,frag_coords,frag_tris,sorted_codes,sort_perm,level_off,"
        "codes,child_base,child_mask,parent,normal")
    save("svo_golden.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["svo"]
    for w in which:
        globals()["gen_" + w]()
