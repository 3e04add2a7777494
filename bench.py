#!/usr/bin/env python
"""Guided wavefront path tracing throughput on B200 (path samples / s).

Workload (BASELINE.json configs[1], "C2"): Cornell box 1920x1080, SVO depth 10
(R = 1024), max path depth 4, all 4 depths guided, N0 = 128, l_min 5,
c_ray 512, plain guiding, fp64.  A step is one guided render pass over the
whole image (1 sample per pixel = 2,073,600 path samples), including Alg. 2
binning, per-bin field + table generation, shading, the Eq. 5 exitance update
and the SVO refresh.  Setup renders the PT-first pass (sample 0); warm-up and
timed passes are guided samples 1, 2, ... so the SVO keeps learning.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun (N > 1) the 1920x1080 image is split into N pixel bands
(strong scaling; --weak: every rank renders its own 1920x1080 band).  Each
rank's pass bins the guided depths globally (start nodes all-gathered),
generates the fields of only the bins its own paths belong to, and splats
every rank's exitance deposits in global path order — NCCL collectives issued
by the native library inside the pass's CUDA graph (multigpu.py).  The image
is the 1-GPU image path for path.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

HBM_PEAK_FALLBACK = 6650.0
SCENES = {"c2": ("cornell.scene", 1024, "C2: Cornell"),
          "c3": ("c3_two_rooms.scene", 2048, "C3: occluded-light two-room interior"),
          "tess": ("cornell_tess.scene", 1024, "Cornell tessellated to 2,304 triangles (BVH)")}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--scene", default="c2", choices=list(SCENES),
                   help="c2: Cornell box (the headline); c3: occluded-light two-room "
                        "interior; tess: Cornell with 2,304 triangles (BVH paths)")
    p.add_argument("--svo-res", type=int, default=None,
                   help="SVO resolution (default 1024 for c2, 2048 for c3)")
    p.add_argument("--depth", type=int, default=4)
    p.add_argument("--field-res", type=int, default=128)
    p.add_argument("--product", action="store_true")
    p.add_argument("--tiled", action="store_true",
                   help="(default) --width x --height is the whole image, split into one band "
                        "per GPU (strong scaling); C4 = --tiled --width 3840 --height 2160")
    p.add_argument("--weak", action="store_true",
                   help="every GPU renders its own width x height band of a taller image")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-overlap", action="store_true",
                   help="one GPU: run the passes back to back on one stream (no PassPipeline)")
    p.add_argument("--no-own", action="store_true",
                   help="N > 1: every rank generates the fields of the bins its paths use at "
                        "every depth (no bin ownership for depths >= 2)")
    a = p.parse_args()
    if a.svo_res is None:
        a.svo_res = SCENES[a.scene][1]
    return a


METRIC = "path samples/sec (guided wavefront pass)"
DATA = "synthetic: scenes/{scene}, path samples from the counter RNG"


def scaling(args):
    return "weak" if args.weak else "strong"


def image_height(args, world):
    return args.height * world if args.weak else args.height


def workload_config(args, svo_depth, world):
    """The config dict both arms print (identical for the same arguments)."""
    H = image_height(args, world)
    lmin = min(5, svo_depth - 1)
    return {"workload": f"{SCENES[args.scene][2]} {args.width}x{H}, 1 spp guided pass per step, "
                        f"SVO depth {svo_depth}, D={args.depth}, G={args.depth}, "
                        f"N0={args.field_res}, l_min {lmin}, c_ray 512, "
                        f"{'product' if args.product else 'plain'} guiding",
            "scene": SCENES[args.scene][0], "image": [args.width, H], "svo_depth": svo_depth,
            "max_depth": args.depth, "guided_depths": args.depth, "field_res": args.field_res,
            "l_min": lmin, "c_ray": 512, "product": bool(args.product), "seed": args.seed,
            "l2": "inputs larger than L2 (path state + guide tables > 126 MB)",
            "parallelism": "single GPU" if world == 1 else (
                f"image bands x{world} ({'weak: one band per GPU' if args.weak else 'strong: one image split'}), "
                "global Alg. 2 binning, depth-1 fields of the rank's own bins, bin ownership "
                "for depths >= 2, per-pass deposit exchange (NCCL, in the pass graph)")}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:  # in-process NVML sampling (nvidia_ml_py), 20 ms period
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.stop = threading.Event()

            def loop():
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                while not self.stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = ["Active" if rs & b else "Not Active" for b in (
                        0x8, 0x40, 0x20, 0x4)]  # hw_slowdown, hw_thermal, sw_thermal, sw_power
                    self.rows.append([str(sm), str(mx), hex(rs)] + flags)
                    self.stop.wait(0.02)

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            self.nvml = True
            return self
        except Exception:
            self.nvml = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if getattr(self, "nvml", False):
            self.stop.set()
            self.t.join(timeout=2)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def build_workload(args, world=1):
    import torch

    from paper_2405_06997_b200 import scene as S, svo, wavefront

    sc = S.load_scene(os.path.join(REPO, "scenes", SCENES[args.scene][0]))
    cam = sc.camera
    # strong scaling (default): the width x height image is split into world
    # bands; --weak: every rank renders its own width x height band
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, args.width,
                         image_height(args, world))
    t0 = time.perf_counter()
    tree = svo.build_from_scene(sc, args.svo_res, seed=args.seed)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    lmin = min(5, tree.depth - 1)
    mk = lambda g: wavefront.GuidingConfig(  # noqa: E731
        l_min=lmin, c_ray=512, field_res=args.field_res, guided_depths=g, max_depth=args.depth,
        product=args.product, seed=args.seed)
    return sc, tree, mk(0), mk(args.depth), build_ms


def _traffic_entry(args):
    key = f"{args.scene}:{args.width}x{args.height}:R{args.svo_res}:D{args.depth}:N{args.field_res}"
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(key)
    except (OSError, ValueError):
        return None


def traffic(args):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture of this workload (profiles/traffic.json), else None."""
    t = _traffic_entry(args)
    try:
        return None if t is None else t["dram_read_bytes"] + t["dram_write_bytes"]
    except KeyError:
        return None


def algorithmic_bytes_per_cone(svo_depth):
    # descent mask 1 + child_base 4 per level, normal 12 +
    # side mean 12, output 4 -> 5 d + 28 bytes per cone
    return 5 * svo_depth + 28


def run_b200(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2405_06997_b200 import _lib, multigpu, wavefront

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; WFPG_DIST_BACKEND=gloo + a shared device lets the
    # multi-rank path be exercised on a 1-GPU box (functional check only:
    # host-exchange communicator over gloo, eager passes)
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    backend = os.environ.get("WFPG_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    sc, tree, pt_cfg, g_cfg, build_ms = build_workload(args, world)
    lib = _lib.load()
    comm = None
    if world > 1:
        # the pass's own collectives: NCCL captured in the pass graph, or the
        # host-exchange protocol over gloo
        comm = (multigpu.Communicator.nccl() if backend == "nccl"
                else multigpu.Communicator.torch_distributed())
    total_pix = args.width * image_height(args, world)
    off, npx = multigpu.band(total_pix, rank, world)
    pt = wavefront.PassRunner(sc, tree, pt_cfg, pixel_offset=off, n_pixels=npx, comm=comm)
    gr = wavefront.PassRunner(sc, tree, g_cfg, pixel_offset=off, n_pixels=npx, comm=comm)

    # field-kernel timing stamps are part of the captured pass, so switch them
    # on before the warm-up (which also captures the pass's CUDA graph)
    lib.wfpg_profile_enable(1)
    pt.launch(0, want_stats=True)
    sample = 1
    gr.launch(sample, want_stats=True)  # first guided pass: stats (bins per depth)
    sample += 1
    stats = gr.pass_stats()
    if comm is not None and not args.no_own:
        # bin ownership for depths >= 2 sized from this pass's global bins
        gr.set_ownership(stats.bins_per_depth)
    # one GPU: consecutive passes on two streams, pass i+1's ray generation,
    # intersection and first binning overlapping pass i's last depth and
    # exitance update (wavefront.PassPipeline; same results as sequential
    # passes).  Multi-GPU passes run back to back on one runner.
    pipe = (wavefront.PassPipeline(sc, tree, g_cfg, runners=[gr, wavefront.PassRunner(
        sc, tree, g_cfg, pixel_offset=off, n_pixels=npx)]) if world == 1 and not args.no_overlap
        else None)
    launch = (lambda s_: pipe.launch(s_)) if pipe else (lambda s_: gr.launch(s_, want_stats=False))
    warmup = max(args.warmup, 5)  # >= 2 per pipeline runner: eager, then graph capture
    for _ in range(warmup - 1):
        launch(sample)
        sample += 1
    if pipe:
        pipe.join()
    if comm is not None:
        comm.settle()
    torch.cuda.synchronize()

    lib.wfpg_profile_enable(1)  # zero the accumulators; timed passes replay the graph
    launches0 = _lib.launch_count()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    with ClockSampler(dev) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            launch(sample)
            sample += 1
        if pipe:
            pipe.join()
        if comm is not None:
            comm.settle()  # the last pass's deposit exchange is part of the work
        end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = start.elapsed_time(end)
    launches = _lib.launch_count() - launches0
    D = args.depth
    fms = (C.c_double * (D + 1))()
    cones = (C.c_double * (D + 1))()
    nl = (C.c_int64 * (D + 1))()
    lib.wfpg_profile_read(fms, cones, nl, D)
    lib.wfpg_profile_enable(0)
    per_rank = {"rank": rank, "paths_per_pass": npx, "ms": ms,
                "cones_per_pass": sum(cones[d] for d in range(1, D + 1)) / args.steps,
                "field_bins_per_pass": [cones[d] / max(nl[d], 1) / max(8, args.field_res >> (d - 1)) ** 2
                                        for d in range(1, D + 1)]}
    if world > 1:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        ranks = [None] * world
        dist.all_gather_object(ranks, per_rank)
    else:
        ranks = [per_rank]

    ms_step = ms / args.steps
    value = total_pix * args.steps / (ms / 1e3)  # whole job

    # roofline of the dominant kernel (depth-1 field generation, n = N0)
    bpc = algorithmic_bytes_per_cone(tree.depth)
    d1_ms = fms[1] / max(nl[1], 1)
    d1_bytes = cones[1] / max(nl[1], 1) * bpc
    peak, peak_kind = peaks()
    achieved = d1_bytes / (d1_ms / 1e3) / 1e9 if d1_ms > 0 else 0.0
    field_ms_step = sum(fms[d] for d in range(1, D + 1)) / args.steps
    roof = {"bound": "hbm", "kernel": f"k_fields<{args.field_res}> (depth-1 fields)",
            "timer": "%globaltimer stamp kernels on the pass stream around each field launch, "
                     "inside the timed CUDA-graph replays (host events cannot sit between "
                     "graph nodes)",
            "achieved": achieved,
            "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / peak if peak else None, "traffic": traffic(args),
            "launch_ms": d1_ms, "bytes_per_launch": d1_bytes,
            "cones_per_launch": cones[1] / max(nl[1], 1), "bytes_per_cone": bpc,
            "gcones_per_s": (cones[1] / max(nl[1], 1)) / (d1_ms / 1e3) / 1e9 if d1_ms else None,
            "field_share_of_step": field_ms_step / ms_step,
            "limiter": (_traffic_entry(args) or {}).get("limiter")}

    # e2e through the public API with every pass's frame in pinned host memory
    e2e = None
    if world == 1 and not args.no_e2e:
        frame_bytes = npx * 3 * 8
        fpipe = wavefront.FramePipeline(sc, tree, g_cfg)
        # API warm-up: two passes per pipeline runner (eager, graph capture)
        for _ in fpipe.run(range(sample, sample + 4)):
            pass
        sample += 4
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        checksum = 0.0
        for _, f, _ in fpipe.run(range(sample, sample + args.steps)):
            checksum += float(f[0, 0, 0])  # the host frame is read every step
        e2e_s = time.perf_counter() - t0
        sample += args.steps
        e2e = {"value": npx * args.steps / e2e_s, "unit": "path samples/s",
               "h2d_bytes_per_step": C.sizeof(_lib.PassConfig) + C.sizeof(_lib.Camera),
               "d2h_bytes_per_step": frame_bytes,
               "api": "paper_2405_06997_b200.wavefront.FramePipeline.run -> pinned host "
                      "frame per pass (copy of pass i overlapped with pass i+1)"}
    elif world > 1 and not args.no_e2e:
        # per rank: pass (with its in-graph exchange) + its band of the frame
        # to pinned host memory; whole-job time = max over ranks
        host = torch.empty((npx, 3), dtype=torch.float64, pin_memory=True)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            gr.launch(sample, want_stats=False)
            sample += 1
            host.copy_(gr.frame, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            float(host[0, 0])
        comm.settle()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                             device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": total_pix * args.steps / float(e2e_s.item()),
               "unit": "path samples/s",
               "h2d_bytes_per_step": C.sizeof(_lib.PassConfig) + C.sizeof(_lib.Camera),
               "d2h_bytes_per_step": npx * 3 * 8,
               "api": "wavefront.PassRunner.launch(comm=multigpu.Communicator) per rank, band "
                      "frame -> pinned host; max over ranks"}

    out = {
        "metric": METRIC,
        "value": value, "unit": "path samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "warmup_passes": {"guided": warmup, "pt_first": 1,
                          "note": "untimed passes actually run before the timed region: at "
                                  "least --warmup, and at least two per pipeline runner "
                                  "(eager + CUDA-graph capture)"},
        "scaling": scaling(args), "vs_baseline": None, "dtype": "f64",
        "data": DATA.format(scene=SCENES[args.scene][0]),
        "config": workload_config(args, tree.depth, world),
        "svo_nodes": tree.node_count,
        "bins_per_depth": stats.bins_per_depth, "rays_per_depth": stats.rays_per_depth,
        "per_rank": ranks,
        "svo_build_ms": build_ms,
        "gpu_launches": int(launches),
        "roofline": roof,
        "e2e": e2e,
        "clocks": clocks.summary(),
    }
    if world > 1:
        out["comm"] = {"backend": backend, "kind": comm.kind,
                       "bin_ownership_depths": [d for d in range(32) if gr.pc.own_bins[d]]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, sc, tree, g_cfg, sample)
    if rank == 0:
        print(json.dumps(out))
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args, sc, tree, cfg, next_sample):
    """The CPU oracle (port of the reference's guided pass) on a bounded
    sample of the same workload: ONE full guided pass of the next sample,
    continuing from the device run's SVO state (structure + exitance, bit-exact
    with the oracle's), timed on this host's cores."""
    try:
        from oracle import render as OR
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "path samples/s", "cores": 0, "kind": "port",
                "sample": f"oracle unavailable: {e}"}
    wl = OR.CpuWorkload.from_device(sc, tree, cfg, next_sample)
    return OR.time_guided_passes(wl, args.width * args.height, passes=1)


def run_reference(args):
    """--impl reference: the CPU port of the reference's guided pass (oracle/:
    C + OpenMP field generation on every host thread, numpy bookkeeping; the
    reference itself is Python/Cython and does not travel to the GPU box).  No
    CUDA and no product library on this arm: the scene is parsed by the
    package's pure-Python loader and its BVH comes from the numpy restatement
    (oracle/render.py _oracle_bvh).  Setup builds the SVO and renders the
    PT-first pass with the oracle; every warm-up and timed step then renders
    the next guided sample IN FULL (wavefront.render_pass semantics, SVO
    learning between passes).  Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from types import SimpleNamespace

    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S

    sc = S.load_scene(os.path.join(REPO, "scenes", SCENES[args.scene][0]))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, args.width, args.height)
    depth = args.svo_res.bit_length() - 1
    cfg = SimpleNamespace(l_min=min(5, depth - 1), c_ray=512, field_res=args.field_res,
                          guided_depths=args.depth, max_depth=args.depth, product=args.product,
                          seed=args.seed)
    wl = OR.CpuWorkload(sc, args.svo_res, cfg, seed=args.seed)
    n_paths = args.width * args.height
    secs = []
    for step in range(args.warmup + args.steps):
        dt, st = wl.run_pass()
        secs.append(dt)
    timed = secs[args.warmup:]
    v = n_paths * len(timed) / sum(timed)
    cb = {"value": v, "unit": "path samples/s", "cores": OR._threads(), "kind": "port",
          "sample": f"every step is one full guided pass of the workload ({n_paths} paths) by "
                    f"the CPU oracle; {wl.describe()}; bins per depth of the last pass "
                    f"{st.get('bins')}",
          "pass_seconds": timed}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v,
        "unit": "path samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(timed) / len(timed) * 1e3, "higher_is_better": True,
        "scaling": scaling(args), "vs_baseline": None, "dtype": "f64", "data": DATA.format(
            scene=SCENES[args.scene][0]),
        "config": workload_config(args, depth, world),
        "host": "CPU only (rank 0's host threads); n_gpus mirrors the B200 arm this line is "
                "paired with",
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "path samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
