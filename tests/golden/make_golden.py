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


# ---------------------------------------------------------------------------
RENDER_CFG = dict(W=32, H=32, R=64, svo_seed=0, max_depth=4, field_res=32, l_min=3, c_ray=16,
                  seed=7)


def _capture_pass(scene, tree, cfg, sample):
    """Run the reference render_pass and capture PathState, guide tables and bins."""
    cap = {"tables": {}, "bins": {}}
    orig_update = wavefront.update_exitance
    orig_build = wavefront._build_guide_tables
    orig_part = wavefront.partition_spatial

    def upd(state, svo):
        cap["state"] = {k: getattr(state, k).copy() for k in
                        ("radiance", "rec_pos", "rec_T", "emit_le", "emit_depth", "ray_o",
                         "ray_d", "beta", "ctr", "alive", "prev_pdf")}
        return orig_update(state, svo)

    depth_box = [0]

    def part(svo, positions, path_idx, l_min, c_ray):
        depth_box[0] += 1
        bins = orig_part(svo, positions, path_idx, l_min, c_ray)
        cap["bins"][depth_box[0]] = (np.array([b.node for b in bins], dtype=np.int64),
                                     [b.members.copy() for b in bins],
                                     positions.copy(), path_idx.copy())
        return bins

    def build(svo, scene_, cfg_, bins, pos, sample_index, depth, n_paths):
        tables, slot = orig_build(svo, scene_, cfg_, bins, pos, sample_index, depth, n_paths)
        keys = core.stream_key(np.uint64(cfg_.seed), np.array(
            [wavefront.bin_stream_id(sample_index, depth, b.node) for b in bins], dtype=np.uint64))
        origins = np.array([pos[b.members[min(int(core.u01_at(k, np.uint64(0)) * len(b.members)),
                                              len(b.members) - 1)]] for k, b in zip(keys, bins)])
        jit = np.stack([core.u01_at(keys, np.uint64(1)), core.u01_at(keys, np.uint64(2))], axis=1)
        cap["tables"][depth] = (tables, slot.copy(), origins, jit)
        return tables, slot

    wavefront.update_exitance = upd
    wavefront._build_guide_tables = build
    wavefront.partition_spatial = part
    try:
        frame, stats = wavefront.render_pass(scene, tree, cfg, [sample])
    finally:
        wavefront.update_exitance = orig_update
        wavefront._build_guide_tables = orig_build
        wavefront.partition_spatial = orig_part
    return frame, stats, cap


def _svo_state(tree):
    return {k: getattr(tree, k).copy() for k in ("sum_a", "sum_b", "weight_a", "weight_b",
                                                  "mean_a", "mean_b")}


def gen_render():
    c = RENDER_CFG
    sc = load_scene("cornell.scene", c["W"], c["H"])
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    out = {"cfg_keys": np.array(list(c)), "cfg_vals": np.array(list(c.values()))}
    pt_cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                     field_res=c["field_res"], l_min=c["l_min"],
                                     c_ray=c["c_ray"], seed=c["seed"])
    f0, st0, cap0 = _capture_pass(sc, tree, pt_cfg, 0)
    out["p0_frame"] = f0
    for k, v in cap0["state"].items():
        out["p0_" + k] = v
    for k, v in _svo_state(tree).items():
        out["p0_svo_" + k] = v
    out["p0_bins_per_depth"] = np.array(st0.bins_per_depth)
    out["p0_rays_per_depth"] = np.array(st0.rays_per_depth)
    for d, (nodes, members, pos, pidx) in cap0["bins"].items():
        out[f"p0_d{d}_bin_nodes"] = nodes
        out[f"p0_d{d}_bin_sizes"] = np.array([len(m) for m in members])
        out[f"p0_d{d}_bin_members"] = (np.concatenate(members) if members
                                       else np.zeros(0, dtype=np.int64))
        out[f"p0_d{d}_positions"] = pos
        out[f"p0_d{d}_path_idx"] = pidx
    base_state = _svo_state(tree)
    for tag, product in (("p1", False), ("p1x", True)):
        for k, v in base_state.items():
            setattr(tree, k, v.copy())
        g_cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                        field_res=c["field_res"], l_min=c["l_min"],
                                        c_ray=c["c_ray"], seed=c["seed"], product=product)
        f1, st1, cap1 = _capture_pass(sc, tree, g_cfg, 1)
        out[tag + "_frame"] = f1
        for k, v in cap1["state"].items():
            out[f"{tag}_{k}"] = v
        for k, v in _svo_state(tree).items():
            out[f"{tag}_svo_" + k] = v
        out[tag + "_bins_per_depth"] = np.array(st1.bins_per_depth)
        out[tag + "_rays_per_depth"] = np.array(st1.rays_per_depth)
        for d, (tables, slot, origins, jit) in cap1["tables"].items():
            out[f"{tag}_d{d}_origins"] = origins
            out[f"{tag}_d{d}_jitters"] = jit
            out[f"{tag}_d{d}_bin_slot"] = slot
            for k in ("marg", "cond", "pdftab", "vals", "block_sums", "blk_marg", "blk_cond"):
                out[f"{tag}_d{d}_{k}"] = getattr(tables, k)
        print(tag, "bins", st1.bins_per_depth, "rays", st1.rays_per_depth)
    # cone queries against the PT-first exitance state
    for k, v in base_state.items():
        setattr(tree, k, v.copy())
    rng = np.random.default_rng(11)
    m = 4096
    lo, hi = sc.bbox_lo, sc.bbox_hi
    org = lo + (hi - lo) * (0.05 + 0.9 * rng.random((m, 3)))
    dirs = rng.standard_normal((m, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    for omega in (4 * np.pi / 32 ** 2, 4 * np.pi / 128 ** 2):
        tag = f"cone_{int(round(np.sqrt(4 * np.pi / omega)))}"
        out[tag + "_rgb"] = wfpg.backend.get().trace_cones_multi(tree, sc, org, dirs, omega)
        out[tag + "_omega"] = np.array(omega)
    out["cone_origins"] = org
    out["cone_dirs"] = dirs
    # intersection queries
    t, tri = sc.intersect_batch(org, dirs)
    out["isect_t"] = t
    out["isect_tri"] = tri
    occ = sc.occluded_batch(org, dirs, 0.5 * np.where(np.isfinite(t), t, 1e3))
    out["occ_half"] = occ
    save("render_golden.npz", **out)


def gen_fields():
    """Field generation at every resolution from fixed origins (PT-first SVO state)."""
    c = RENDER_CFG
    sc = load_scene("cornell.scene", c["W"], c["H"])
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0, seed=c["seed"])
    wavefront.render_pass(sc, tree, cfg, [0])
    wavefront.render_pass(sc, tree, cfg, [1])
    out = {}
    for k, v in _svo_state(tree).items():
        out["svo_" + k] = v
    rng = np.random.default_rng(5)
    lo, hi = sc.bbox_lo, sc.bbox_hi
    b = 6
    org = lo + (hi - lo) * (0.1 + 0.8 * rng.random((b, 3)))
    jit = rng.random((b, 2))
    out["origins"] = org
    out["jitters"] = jit
    for n in (8, 16, 32, 64, 128):
        vals = guiding.generate_fields_batch(tree, sc, org, n, jit, blur_sigma=1.0)
        out[f"vals_{n}"] = vals
        t = guiding.GuideTables(2, n, b)
        t.fill_batch(vals)
        for k in ("marg", "cond", "pdftab", "block_sums", "blk_marg", "blk_cond"):
            out[f"tab_{n}_{k}"] = getattr(t, k)
    vals = guiding.generate_fields_batch(tree, sc, org, 16, jit, blur_sigma=2.5)
    out["vals_16_s25"] = vals
    vals = guiding.generate_fields_batch(tree, sc, org, 16, jit, blur_sigma=0.0)
    out["vals_16_s0"] = vals
    save("fields_golden.npz", **out)


# ---------------------------------------------------------------------------
C3_CFG = dict(W=64, H=36, R=128, svo_seed=2, max_depth=5, field_res=32, l_min=3, c_ray=16,
              seed=3)
C3_SCENE = os.path.join(HERE, "..", "..", "scenes", "c3_two_rooms.scene")


def gen_c3():
    """C3 (procedural occluded-light interior, paper_2405_06997_b200/scenegen.py):
    SVO arrays + digests, a PT-first pass and two guided passes (plain, then
    product) learning from it, per-path records, bins and SVO state."""
    c = C3_CFG
    sc = rscene.load_scene(C3_SCENE)
    cam = sc.camera
    sc.camera = rscene.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    out = {"cfg_keys": np.array(list(c)), "cfg_vals": np.array(list(c.values()))}
    dig = []
    for res, seed in ((64, 1), (256, 0), (512, 0)):
        frags = rsvo.voxelize(sc, res)
        lo, side = rsvo.scene_cube(sc)
        tree = rsvo.build_octree(frags, lo, side, res, seed)
        row = [str(res), str(seed), str(len(frags)), str(tree.node_count),
               digest(tree.level_off.astype(np.int64)), digest(tree.codes),
               digest(tree.child_base.astype(np.int64)), digest(tree.child_mask),
               digest(tree.parent.astype(np.int64)), digest(tree.normal)]
        dig.append(",".join(row))
        print(row)
    out["svo_digests"] = np.array(dig)
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    out["svo_level_off"] = tree.level_off
    out["svo_codes"] = tree.codes
    out["svo_normal"] = tree.normal
    passes = (("p0", 0, 0, False), ("p1", 1, c["max_depth"], False),
              ("p2", 2, c["max_depth"], True))
    for tag, sample, g, product in passes:
        cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=g,
                                      field_res=c["field_res"], l_min=c["l_min"],
                                      c_ray=c["c_ray"], seed=c["seed"], product=product)
        f, st, cap = _capture_pass(sc, tree, cfg, sample)
        out[tag + "_frame"] = f
        for k in ("radiance", "rec_pos", "emit_depth"):
            out[f"{tag}_{k}"] = cap["state"][k]
        for k, v in _svo_state(tree).items():
            out[f"{tag}_svo_" + k] = v
        out[tag + "_bins_per_depth"] = np.array(st.bins_per_depth)
        out[tag + "_rays_per_depth"] = np.array(st.rays_per_depth)
        print(tag, "bins", st.bins_per_depth, "rays", st.rays_per_depth,
              "deposits", int(tree.weight_a.sum() + tree.weight_b.sum()))
    save("c3_golden.npz", **out)


# ---------------------------------------------------------------------------
def gen_cli():
    """collect_bin_image of render_pass (1- and 2-sample PT passes) and whole
    CLI runs (cli.run) on the scene file's own 64x64 camera."""
    import tempfile

    from wfpg import cli

    c = RENDER_CFG
    out = {}
    sc = load_scene("cornell.scene", c["W"], c["H"])
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    for tag, samples in (("bins1", [0]), ("bins2", [0, 1])):
        frame, st, img = wavefront.render_pass(sc, tree, cfg, samples, collect_bin_image=True)
        out[tag + "_image"] = img
        out[tag + "_frame"] = frame
        out[tag + "_bins_per_depth"] = np.array(st.bins_per_depth)
    # a guided pass over two consecutive samples (bins pool both samples'
    # paths; bin streams use the first sample index, wavefront.py:249)
    gcfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                   field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                   seed=c["seed"])
    wavefront.render_pass(sc, tree, cfg, [5])  # some exitance state first
    for k, v in _svo_state(tree).items():
        out["multi_pre_" + k] = v
    cap = {}
    orig_update = wavefront.update_exitance

    def upd(state, svo):
        cap["state"] = {k: getattr(state, k).copy() for k in ("radiance", "rec_pos",
                                                               "emit_depth")}
        return orig_update(state, svo)

    wavefront.update_exitance = upd
    try:
        fm, stm = wavefront.render_pass(sc, tree, gcfg, [1, 2])
    finally:
        wavefront.update_exitance = orig_update
    out["multi_frame"] = fm
    out["multi_bins_per_depth"] = np.array(stm.bins_per_depth)
    for k, v in cap["state"].items():
        out["multi_" + k] = v
    tmp = tempfile.mkdtemp()
    runs = (("pt", dict(mode="pt", spp=2)),
            ("wfpg", dict(mode="wfpg", spp=3, depth=4, svo_res=64, field_res=32, lmin=3,
                          cray=16, seed=5)),
            ("prod", dict(mode="wfpg-product", spp=2, depth=3, guided_depths=3, svo_res=32, field_res=16,
                          lmin=2, cray=8, seed=1, heuristic="linear")))
    for tag, kw in runs:
        conf = cli.RunConfig(scene=os.path.join(SCENES, "cornell.scene"),
                             out=os.path.join(tmp, tag + ".pfm"), **kw)
        logs = []
        status, frame = cli.run(conf, log=logs.append)
        assert status == 0
        out[f"cli_{tag}_frame"] = frame
        out[f"cli_{tag}_log"] = np.array([ln for ln in logs if ln.startswith("sample ")])
        out[f"cli_{tag}_config"] = np.array(conf.to_json())
        print(tag, frame.mean(), logs[-3:])
    save("cli_golden.npz", **out)


# ---------------------------------------------------------------------------
def gen_dump():
    """WFPGSVO1 dumps written by the reference (svo.py:344-362): a fresh
    Cornell build at R=16 (seed 0) and the same tree after a 16x16 PT-first
    pass (exitance state)."""
    sc = load_scene("cornell.scene", 16, 16)
    tree = rsvo.build_from_scene(sc, 16, seed=0)
    tree.dump(os.path.join(HERE, "svo_cornell_r16_fresh.wfpgsvo"))
    cfg = wavefront.GuidingConfig(max_depth=4, guided_depths=0, l_min=2, c_ray=8, seed=3)
    wavefront.render_pass(sc, tree, cfg, [0])
    tree.dump(os.path.join(HERE, "svo_cornell_r16_pt.wfpgsvo"))
    print("nodes", tree.node_count, "weights", tree.weight_a.sum() + tree.weight_b.sum())


# ---------------------------------------------------------------------------
TESS_CFG = dict(W=32, H=32, R=64, svo_seed=0, max_depth=4, field_res=32, l_min=3, c_ray=16,
                seed=7)


def gen_tess():
    """BVH-path scene (scenegen.write_tessellated_cornell, 2,304 triangles):
    SVO digests, intersection queries, a PT-first and a guided pass."""
    c = TESS_CFG
    sc = rscene.load_scene(os.path.join(HERE, "..", "..", "scenes", "cornell_tess.scene"))
    cam = sc.camera
    sc.camera = rscene.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    out = {"cfg_keys": np.array(list(c)), "cfg_vals": np.array(list(c.values()))}
    dig = []
    for res, seed in ((64, 0), (128, 1)):
        frags = rsvo.voxelize(sc, res)
        lo, side = rsvo.scene_cube(sc)
        tree = rsvo.build_octree(frags, lo, side, res, seed)
        dig.append(",".join([str(res), str(seed), str(len(frags)), str(tree.node_count),
                             digest(tree.level_off.astype(np.int64)), digest(tree.codes),
                             digest(tree.child_base.astype(np.int64)), digest(tree.child_mask),
                             digest(tree.parent.astype(np.int64)), digest(tree.normal)]))
    out["svo_digests"] = np.array(dig)
    rng = np.random.default_rng(13)
    lo, hi = sc.bbox_lo, sc.bbox_hi
    org = lo + (hi - lo) * (0.05 + 0.9 * rng.random((4096, 3)))
    dirs = rng.standard_normal((4096, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    t, tri = sc.intersect_batch(org, dirs)
    out.update(isect_o=org, isect_d=dirs, isect_t=t, isect_tri=tri)
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    for tag, sample, g in (("p0", 0, 0), ("p1", 1, c["max_depth"])):
        cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=g,
                                      field_res=c["field_res"], l_min=c["l_min"],
                                      c_ray=c["c_ray"], seed=c["seed"])
        f, st, cap = _capture_pass(sc, tree, cfg, sample)
        out[tag + "_frame"] = f
        for k in ("radiance", "rec_pos", "emit_depth"):
            out[f"{tag}_{k}"] = cap["state"][k]
        for k, v in _svo_state(tree).items():
            out[f"{tag}_svo_" + k] = v
        out[tag + "_bins_per_depth"] = np.array(st.bins_per_depth)
        print(tag, "bins", st.bins_per_depth)
    save("tess_golden.npz", **out)


# ---------------------------------------------------------------------------
RELMSE_RUNS = dict(spp=32, depth=5, svo_res=64, field_res=32, lmin=3, cray=16)


def gen_relmse():
    """Equal-spp relMSE protocol of SURVEY.md 8(d) at reduced size: the
    reference CLI renders cornell_enclosed (64x64) with 32 spp guided (wfpg,
    pt-first) and unguided (pt) for seeds 1..3; the GPU tests render the same
    runs and compare both against a high-spp reference."""
    import tempfile

    from wfpg import cli

    tmp = tempfile.mkdtemp()
    out = {"cfg_keys": np.array(list(RELMSE_RUNS)),
           "cfg_vals": np.array(list(RELMSE_RUNS.values()))}
    scene_file = os.path.join(HERE, "..", "..", "scenes", "cornell_enclosed.scene")
    for mode in ("wfpg", "pt"):
        for seed in (1, 2, 3):
            conf = cli.RunConfig(scene=scene_file, mode=mode, seed=seed,
                                 out=os.path.join(tmp, f"{mode}{seed}.pfm"), **RELMSE_RUNS)
            status, frame = cli.run(conf, log=lambda *_: None)
            assert status == 0
            out[f"{mode}_{seed}"] = frame
            print(mode, seed, frame.mean())
    save("relmse_golden.npz", **out)


# ---------------------------------------------------------------------------
C1_CFG = dict(W=256, H=256, R=256, svo_seed=0, max_depth=4, field_res=128, l_min=5, c_ray=512,
              seed=0)


def _path_record(cap, stats):
    st = cap["state"]
    return {"emit_depth": st["emit_depth"].astype(np.int8),
            "rec_pos": st["rec_pos"][:, 1:].astype(np.float32),
            "radiance": st["radiance"].astype(np.float32),
            "bins": np.array(stats.bins_per_depth), "rays": np.array(stats.rays_per_depth),
            "mat_groups": _mat_groups(stats)}


def _mat_groups(stats):
    """material_groups per depth as a dense (depths, n_mats) int64 table."""
    n = max([max(g) + 1 for g in stats.material_groups if g] + [1])
    out = np.zeros((len(stats.material_groups), n), dtype=np.int64)
    for d, g in enumerate(stats.material_groups):
        for m, k in g.items():
            out[d, m] = k
    return out


def gen_c1():
    """the primary per-path equivalence configuration:
    Cornell 256x256, SVO R=256 (depth 8), D=4, N0=128, l_min 5, c_ray 512,
    seed 0; pass 0 PT-first (SVO updated), then sample 1 guided plain and,
    from the same PT-first SVO state, sample 1 guided product.  Per path:
    emit depth, vertices 1..4 and radiance (float32), plus bins / rays /
    material groups per depth.  ~5 min of reference time."""
    import time

    c = C1_CFG
    sc = load_scene("cornell.scene", c["W"], c["H"])
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    out = {"cfg_keys": np.array(list(c)), "cfg_vals": np.array(list(c.values()))}
    base = dict(max_depth=c["max_depth"], field_res=c["field_res"], l_min=c["l_min"],
                c_ray=c["c_ray"], seed=c["seed"])
    _, st0, cap0 = _capture_pass(sc, tree, wavefront.GuidingConfig(guided_depths=0, **base), 0)
    for k, v in _path_record(cap0, st0).items():
        out["p0_" + k] = v
    state = _svo_state(tree)
    for k, v in state.items():
        out["p0_svo_" + k] = v.astype(np.float32) if k.startswith("mean") else v
    for tag, product in (("p1", False), ("p1x", True)):
        for k, v in state.items():
            setattr(tree, k, v.copy())
        t0 = time.time()
        _, st1, cap1 = _capture_pass(
            sc, tree, wavefront.GuidingConfig(guided_depths=c["max_depth"], product=product,
                                              **base), 1)
        print(tag, "pass", time.time() - t0, "s, bins", st1.bins_per_depth, flush=True)
        for k, v in _path_record(cap1, st1).items():
            out[f"{tag}_" + k] = v
        out[f"{tag}_svo_weight_a"] = tree.weight_a.copy()
        out[f"{tag}_svo_weight_b"] = tree.weight_b.copy()
    save("c1_golden.npz", **out)


def gen_queries():
    """Direct parity anchors for helpers the render loop uses implicitly:
    descend_tracked (node, present, deepest; _kernelshim.py:60-71 ->
    _kernels.pyx:591-658), SvoCache.ancestor_chain (svo.py:326-340) and
    PassStats.material_groups (wavefront.py:88-95,250-253)."""
    c = RENDER_CFG
    sc = load_scene("cornell.scene", c["W"], c["H"])
    tree = rsvo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    rng = np.random.default_rng(21)
    m = 4096
    lo, size = tree.cube_lo, tree.cube_size
    pts = lo + size * rng.random((m, 3))
    # plus exact voxel corners (boundary quantisation)
    corners = lo + size * (rng.integers(0, tree.resolution, (256, 3)) / tree.resolution)
    pts = np.concatenate([pts, corners])
    node, present, deepest = wfpg.backend.get().descend_tracked(tree, pts)
    out = {"desc_points": pts, "desc_node": node, "desc_present": present,
           "desc_deepest": deepest}
    coords = rng.integers(0, tree.resolution, (600, 3))
    # plus the leaf coordinates of materialised leaves (full-depth chains)
    leaf_codes = tree.codes[tree.level_off[tree.depth]:tree.level_off[tree.depth + 1]]
    pick = rng.choice(len(leaf_codes), 200, replace=False)
    coords = np.concatenate([coords, np.stack(core.morton_decode(leaf_codes[pick]), axis=1)])
    chains = [tree.ancestor_chain(cc) for cc in coords]
    out["chain_coords"] = coords
    out["chain_len"] = np.array([len(ch) for ch in chains])
    out["chain_flat"] = np.concatenate([np.array(ch, dtype=np.int64) for ch in chains])
    base = dict(max_depth=c["max_depth"], field_res=c["field_res"], l_min=c["l_min"],
                c_ray=c["c_ray"], seed=c["seed"])
    for tag, g, sample in (("p0", 0, 0), ("p1", c["max_depth"], 1)):
        _, st = wavefront.render_pass(sc, tree, wavefront.GuidingConfig(guided_depths=g, **base),
                                      [sample])
        out[tag + "_mat_groups"] = _mat_groups(st)
    # a mirror scene: every material kind (lambert, mirror, emitter) appears
    sc2 = load_scene("cornell.scene", 48, 40)
    tree2 = rsvo.build_from_scene(sc2, 64, seed=0)
    _, st = wavefront.render_pass(sc2, tree2, wavefront.GuidingConfig(guided_depths=0, **base), [0])
    out["w48_mat_groups"] = _mat_groups(st)
    save("queries_golden.npz", **out)


def gen_r1024():
    """Reference digests of the C2 SVO (cornell.scene, R=1024, seed 0), the
    headline depth (~4-5 min in the reference)."""
    import time

    sc = load_scene("cornell.scene")
    t0 = time.time()
    frags = rsvo.voxelize(sc, 1024)
    lo, side = rsvo.scene_cube(sc)
    tree = rsvo.build_octree(frags, lo, side, 1024, seed=0)
    print("R=1024 build", time.time() - t0, "s", flush=True)
    out = {"frags": np.array(len(frags.tris)), "nodes": np.array(tree.node_count),
           "level_off": np.asarray(tree.level_off)}
    for k in ("codes", "child_base", "child_mask", "parent", "normal"):
        out[k] = np.array(digest(getattr(tree, k)))
    out["frag_coords"] = np.array(digest(frags.coords))
    out["frag_tris"] = np.array(digest(frags.tris))
    save("r1024_golden.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["svo"]
    for w in which:
        globals()["gen_" + w]()
