"""``wfpg``-compatible command line (reference cli.py:21-343) on the device
render path.

Same flags, defaults, validation messages, log lines and outputs (PFM + PNG,
``--dump-bins`` false-colour bin image, ``--dump-field`` guided vs
path-traced field at a pixel, ``--ref`` metrics).  What changes is how the
samples flow: every pass runs through one cached ``wavefront.PassRunner``
(CUDA-graph replay after the second pass) and is folded into a
device-resident Eq. 7 buffer (``accumulation.AccumulationBuffer``), so a
many-spp render moves only the final frame to the host.

Deliberate superset: ``--svo-res`` accepts powers of two up to 4096 (the
reference stops at 256, a CPU memory limit), so the C2 / C3 configurations
(R = 1024 / 2048) run from the command line.

    python -m paper_2405_06997_b200.cli --scene scenes/cornell.scene --spp 64
"""

import argparse
import json
import os
import sys
import time

import numpy as np

from . import _dev, accumulation, backend, core, guiding, imageio
from . import scene as scene_mod
from . import svo as svo_mod
from . import wavefront

MODES = ("pt", "wfpg", "wfpg-product")
SVO_RES = tuple(1 << k for k in range(4, 13))
FIELD_RES = (16, 32, 64, 128)


class RunConfig:
    """Validated run parameters (cli.py:21-89)."""

    FIELDS = ("scene", "mode", "spp", "depth", "guided_depths", "field_res", "lmin", "cray",
              "svo_res", "heuristic", "seed", "deterministic", "out", "ref", "dump_bins",
              "dump_field", "workers", "rr")
    DEFAULTS = dict(mode="wfpg", spp=8, depth=5, guided_depths=4, field_res=128, lmin=5,
                    cray=512, svo_res=256, heuristic="pt-first", seed=0, deterministic=False,
                    out="out.pfm", ref=None, dump_bins=False, dump_field=None, workers=None,
                    rr=False)
    _INT = ("spp", "depth", "guided_depths", "field_res", "lmin", "cray", "svo_res", "seed")
    _BOOL = ("deterministic", "dump_bins", "rr")

    def __init__(self, scene, *args, **kw):
        if len(args) > len(self.FIELDS) - 1:
            raise TypeError("too many positional run parameters")
        for k, v in zip(self.FIELDS[1:], args):  # positional order as the reference
            if k in kw:
                raise TypeError(f"duplicate run parameter '{k}'")
            kw[k] = v
        unknown = set(kw) - set(self.DEFAULTS)
        if unknown:
            raise TypeError(f"unknown run parameters: {sorted(unknown)}")
        vals = dict(self.DEFAULTS, **kw)
        self.scene = scene
        for k, v in vals.items():
            if k in self._INT:
                v = int(v)
            elif k in self._BOOL:
                v = bool(v)
            elif k == "dump_field" and v is not None:
                v = tuple(v)
            setattr(self, k, v)
        self.validate()

    def validate(self):
        checks = (
            (self.mode in MODES, f"mode must be one of {MODES}"),
            (self.spp >= 1, "spp must be >= 1"),
            (self.depth >= 1, "depth must be >= 1"),
            (0 <= self.guided_depths <= self.depth, "guided-depths must be within [0, depth]"),
            (self.svo_res in SVO_RES, "svo-res must be a power of two in [16, 4096]"),
            (self.field_res in FIELD_RES, "field-res must be one of 16, 32, 64, 128"),
            (self.heuristic in accumulation.HEURISTICS, f"unknown heuristic '{self.heuristic}'"),
            (self.cray >= 1, "cray must be >= 1"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    def effective_lmin(self, svo_depth):
        """l_min scaled down for shallow trees (cli.py:73-75)."""
        return min(self.lmin, svo_depth - 1)

    def as_dict(self):
        return {k: getattr(self, k) for k in self.FIELDS}

    def to_json(self):
        return json.dumps(self.as_dict(), sort_keys=True)

    @classmethod
    def from_json(cls, text):
        d = json.loads(text)
        return cls(d.pop("scene"), **d)

    def __eq__(self, other):
        return isinstance(other, RunConfig) and self.as_dict() == other.as_dict()


def _bin_false_color(bin_image):
    """Stable pseudo-random colour per bin node id (cli.py:92-107); -1 black."""
    ids = np.asarray(bin_image, dtype=np.int64)
    rgb = np.zeros(ids.shape + (3,))
    on = ids >= 0
    key = core.stream_key(np.uint64(0xB1C0108), ids[on].astype(np.uint64))
    for c in range(3):
        rgb[..., c][on] = 0.15 + 0.85 * core.u01_at(key, np.uint64(c))
    return rgb


def _trace_radiance(scene, origin, dirs, cfg):
    """Radiance arriving at ``origin`` along ``dirs``: unguided paths through
    the device wavefront kernels (cli.py:139-164), keys on stream i*4+3."""
    n = len(dirs)
    st = wavefront.PathState(n, cfg.max_depth, np.asarray(origin))
    key = core.stream_key(np.uint64(cfg.seed),
                          np.arange(n, dtype=np.uint64) * np.uint64(4) + np.uint64(3))
    st.dev["key"].copy_(_dev.upload(key))
    st.dev["ctr"].zero_()
    st.dev["ray_o"].copy_(_dev.upload(np.broadcast_to(np.asarray(origin, float), (n, 3))))
    st.dev["ray_d"].copy_(_dev.upload(np.asarray(dirs, dtype=np.float64)))
    impl = backend.get()
    hit_t = np.zeros(n)
    hit_tri = np.zeros(n, dtype=np.int64)
    for depth in range(1, cfg.max_depth + 1):
        live = np.flatnonzero(st.alive)
        if live.size == 0:
            break
        t, tri = scene.intersect_batch(st.ray_o[live], st.ray_d[live])
        hit_t[live], hit_tri[live] = t, tri
        impl.shade_depth(st, scene, depth, hit_t, hit_tri, None, None,
                         rr_enabled=cfg.russian_roulette, rr_depth=cfg.rr_depth)
    return st.radiance


def estimate_incident_field(scene, origin, n, spp_per_cell, max_depth, seed):
    """Path-traced n x n incident-luminance field at ``origin`` (cli.py:110-136):
    spp_per_cell random directions per octahedral cell, RngStream(seed, 0xF1E1D)."""
    rs = core.RngStream(seed, 0xF1E1D)
    jit = rs.next_n(n * n * spp_per_cell * 2).reshape(-1, 2)
    col = np.repeat(np.tile(np.arange(n), n), spp_per_cell)
    row = np.repeat(np.repeat(np.arange(n), n), spp_per_cell)
    dirs = core.octa_uv_to_dir((col + jit[:, 0]) / n, (row + jit[:, 1]) / n)
    cfg = wavefront.GuidingConfig(max_depth=max_depth, guided_depths=0, seed=seed)
    lum = core.luminance(_trace_radiance(scene, origin, dirs, cfg))
    return lum.reshape(n * n, spp_per_cell).mean(axis=1).reshape(n, n)


def dump_field(config, scene, svo, pixel, out_prefix, log=print):
    """Guided field at the primary hit of ``pixel``, its pdf, and a
    path-traced reference, each normalised to max 1 (cli.py:167-196)."""
    px, py = pixel
    cam = scene.camera
    if not (0 <= px < cam.width and 0 <= py < cam.height):
        raise ValueError("pixel out of range")
    d = cam.ray_directions(np.array([px]), np.array([py]), 0.5, 0.5)[0]
    hit = scene_mod.intersect(scene, cam.position, d)
    if hit is None:
        raise ValueError("pixel ray misses the scene")
    n = config.field_res
    fld = guiding.generate_field(svo, scene, hit.position, n, rng=core.RngStream(config.seed, 0xD0F1),
                                 jitter=False, blur_sigma=1.0)
    pdf = guiding.build_distribution(fld).pdf_table
    ref = np.maximum(estimate_incident_field(scene, hit.position, n, 64, config.depth,
                                             config.seed), 0.0)
    for name, grid in (("field", fld.values), ("field-ref", ref), ("field-pdf", pdf)):
        peak = grid.max()
        g = grid / peak if peak > 0 else grid
        imageio.write_pfm(f"{out_prefix}.{name}.pfm", np.repeat(g[..., None], 3, axis=2))
    log(f"dump-field: origin={hit.position.tolist()} res={n}")
    return fld, ref


def _pass_cfg(config, guided_depths):
    return wavefront.GuidingConfig(
        l_min=config.lmin, c_ray=config.cray, field_res=config.field_res,
        guided_depths=guided_depths, max_depth=config.depth,
        product=config.mode == "wfpg-product", seed=config.seed, russian_roulette=config.rr)


def render(config, scene, svo, log=print, stats_every=1):
    """Accumulate config.spp passes on the device; returns (frame, timings).
    Sample i (1-based) renders pass index i-1; with "pt-first" and a guided
    mode sample 1 is unguided (cli.py:224-230)."""
    cam = scene.camera
    guided = config.guided_depths if config.mode != "pt" else 0
    cfg = _pass_cfg(config, guided)
    if svo is not None:
        cfg.l_min = config.effective_lmin(svo.depth)
    cfg.validate(svo.depth if svo is not None else None)
    buf = accumulation.AccumulationBuffer(cam.height, cam.width, config.heuristic)
    pt_first = config.heuristic == "pt-first" and config.mode != "pt"
    runners = {}

    def runner(g, want_bins):
        key = (g, want_bins)
        if key not in runners:
            c = _pass_cfg(config, g)
            c.l_min = cfg.l_min
            runners[key] = wavefront.PassRunner(scene, svo, c, 1,
                                                deterministic=True,
                                                collect_bin_image=want_bins)
        return runners[key]

    bin_image = None
    t0 = time.perf_counter()
    for i in range(1, config.spp + 1):
        g = 0 if (pt_first and i == 1) else guided
        want_bins = config.dump_bins and i == 1 and svo is not None
        r = runner(g, want_bins)
        log_now = svo is not None and stats_every and (i - 1) % stats_every == 0
        r.launch(i - 1, want_stats=bool(log_now or want_bins))
        buf.add_sample(r.frame, i)
        if want_bins:
            bin_image = _dev.download(r.bin_image).astype(np.int64).reshape(cam.height, cam.width)
        if log_now:
            st = r.pass_stats()
            pairs = [f"{b}/{(n / b if b else 0):.1f}"
                     for b, n in zip(st.bins_per_depth, st.rays_per_depth)]
            log(f"sample {i}: bins/avg-rays per depth: " + " ".join(pairs))
    frame = buf.resolve()
    return frame, bin_image, time.perf_counter() - t0


def run(config, log=print):
    """Execute a configured render; returns (exit status, resolved frame)."""
    try:
        scene = scene_mod.load_scene(config.scene)
    except scene_mod.SceneError as e:
        log(f"error: {e}")
        return 1, None
    if config.workers is not None:
        os.environ["WFPG_THREADS"] = str(config.workers)
    log(f"config: {config.to_json()}")
    log(f"backend: {backend.get().NAME}")
    svo = None
    if config.mode != "pt":
        svo = svo_mod.build_from_scene(scene, config.svo_res, seed=config.seed)
        log(f"svo: resolution={config.svo_res}^3 nodes={svo.node_count} "
            f"leaves={svo.leaf_count} memory_bytes={svo.memory_bytes()} "
            f"(record={svo_mod.NODE_RECORD_BYTES} B/node)")
        log(f"effective l_min: {config.effective_lmin(svo.depth)}")
    frame, bin_image, secs = render(config, scene, svo, log=log)
    log(f"rendered {config.spp} spp in {secs:.3f} s")
    imageio.write_pfm(config.out, frame)
    png = os.path.splitext(config.out)[0] + ".png"
    imageio.write_png(png, frame)
    log(f"wrote {config.out} and {png}")
    if bin_image is not None:
        bout = os.path.splitext(config.out)[0] + ".bins.png"
        imageio.write_png(bout, _bin_false_color(bin_image), tonemap=False)
        log(f"dump-bins: wrote {bout} regions={len(np.unique(bin_image[bin_image >= 0]))}")
    if config.dump_field is not None and svo is not None:
        dump_field(config, scene, svo, config.dump_field, os.path.splitext(config.out)[0],
                   log=log)
    if config.ref:
        ref = imageio.read_pfm(config.ref)
        log(f"mse: {accumulation.mse(frame, ref):.6g}")
        log(f"mean-abs-diff: {accumulation.mean_abs_diff(frame, ref):.6g}")
    return 0, frame


def build_parser():
    p = argparse.ArgumentParser(prog="wfpg",
                                description="Wavefront path tracer with sparse-voxel path guiding")
    d = RunConfig.DEFAULTS
    p.add_argument("--scene", required=True, help="wfpg-scene v1 file")
    p.add_argument("--mode", default=d["mode"], choices=MODES)
    for flag, key, hlp in (("--spp", "spp", None), ("--depth", "depth", "maximum path depth"),
                           ("--guided-depths", "guided_depths", None),
                           ("--field-res", "field_res",
                            "base radiance-field resolution (halves per depth)"),
                           ("--lmin", "lmin", None), ("--cray", "cray", None),
                           ("--svo-res", "svo_res", None), ("--seed", "seed", None)):
        p.add_argument(flag, type=int, default=d[key], help=hlp)
    p.add_argument("--heuristic", default=d["heuristic"],
                   choices=sorted(accumulation.HEURISTICS))
    p.add_argument("--deterministic", action="store_true",
                   help="force single-worker execution")
    p.add_argument("--out", default=d["out"])
    p.add_argument("--ref", default=None, help="PFM reference for metrics")
    p.add_argument("--dump-bins", action="store_true",
                   help="write a false-color image of the depth-1 bins")
    p.add_argument("--dump-field", default=None, metavar="X,Y",
                   help="dump the guided + reference field at a pixel")
    p.add_argument("--workers", type=int, default=None,
                   help="kernel worker threads (WFPG_THREADS fallback)")
    p.add_argument("--rr", action="store_true", help="enable russian roulette")
    return p


def config_from_args(argv):
    a = build_parser().parse_args(argv)
    px = None
    if a.dump_field:
        parts = a.dump_field.split(",")
        try:
            if len(parts) != 2:
                raise ValueError
            px = (int(parts[0]), int(parts[1]))
        except ValueError as e:
            raise ValueError("--dump-field expects X,Y") from e
    return RunConfig(a.scene, mode=a.mode, spp=a.spp, depth=a.depth,
                     guided_depths=min(a.guided_depths, a.depth), field_res=a.field_res,
                     lmin=a.lmin, cray=a.cray, svo_res=a.svo_res, heuristic=a.heuristic,
                     seed=a.seed, deterministic=a.deterministic, out=a.out, ref=a.ref,
                     dump_bins=a.dump_bins, dump_field=px, workers=a.workers, rr=a.rr)


def main(argv=None):
    try:
        config = config_from_args(sys.argv[1:] if argv is None else argv)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    return run(config)[0]


if __name__ == "__main__":
    sys.exit(main())
