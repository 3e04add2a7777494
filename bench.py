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

Under torchrun (N > 1) each rank renders its own 1920x1080 band of a
1920 x (1080 N) image (weak scaling); after every pass the leaf exitance
deposits are summed across ranks with an NCCL all-reduce.
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
                   help="C4: --width x --height is the whole image, split into one band per "
                        "GPU (strong scaling); default: every GPU renders its own "
                        "width x height band of a taller image (weak scaling)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-seconds", type=float, default=20.0,
                   help="budget of the CPU-baseline sample")
    p.add_argument("--ref-seconds", type=float, default=None,
                   help="--impl reference: CPU sample per step (default min(10, 150 / (W + K)) s)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    a = p.parse_args()
    if a.svo_res is None:
        a.svo_res = SCENES[a.scene][1]
    return a


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


def image_height(args, world):
    return args.height if args.tiled else args.height * world


def build_workload(args, rank=0, world=1):
    import torch

    from paper_2405_06997_b200 import scene as S, svo, wavefront

    sc = S.load_scene(os.path.join(REPO, "scenes", SCENES[args.scene][0]))
    cam = sc.camera
    # weak scaling: rank r renders band r of a width x (height * world) image;
    # --tiled (C4): the width x height image is split into world bands
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
    import torch
    import torch.distributed as dist

    from paper_2405_06997_b200 import _lib, wavefront

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; WFPG_DIST_BACKEND=gloo + a shared device lets the
    # multi-rank path be exercised on a 1-GPU box (functional check only)
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    backend = os.environ.get("WFPG_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    sc, tree, pt_cfg, g_cfg, build_ms = build_workload(args, rank, world)
    lib = _lib.load()

    from paper_2405_06997_b200 import multigpu

    # per-pass SVO sync: every rank exports its deposits, all-gathers the
    # lists and splats them in global path order (multigpu.DepositExchange)
    sync_svo = multigpu.DepositExchange(tree) if world > 1 else None
    total_pix = args.width * image_height(args, world)
    off, npx = multigpu.band(total_pix, rank, world)
    pt = wavefront.PassRunner(sc, tree, pt_cfg, pixel_offset=off, n_pixels=npx,
                              deposit_sink=sync_svo)
    gr = wavefront.PassRunner(sc, tree, g_cfg, pixel_offset=off, n_pixels=npx,
                              deposit_sink=sync_svo)

    def one_pass(runner, sample, stats=False):
        runner.launch(sample, want_stats=stats)
        if sync_svo is not None:
            sync_svo.reduce_and_apply(runner)

    # field-kernel timing stamps are part of the captured pass, so switch them
    # on before the warm-up (which also captures the pass's CUDA graph)
    lib.wfpg_profile_enable(1)
    one_pass(pt, 0, True)
    sample = 1
    for _ in range(max(args.warmup, 3)):
        one_pass(gr, sample, True)
        sample += 1
    stats = gr.pass_stats()
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
            one_pass(gr, sample)
            sample += 1
        end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = start.elapsed_time(end)
    launches = _lib.launch_count() - launches0
    import ctypes as C

    D = args.depth
    fms = (C.c_double * (D + 1))()
    cones = (C.c_double * (D + 1))()
    nl = (C.c_int64 * (D + 1))()
    lib.wfpg_profile_read(fms, cones, nl, D)
    lib.wfpg_profile_enable(0)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    n_paths = npx  # this rank's paths per pass
    ms_step = ms / args.steps
    value = total_pix * args.steps / (ms / 1e3)  # whole job

    # roofline of the dominant kernel (depth-1 field generation, n = N0)
    bpc = algorithmic_bytes_per_cone(tree.depth)
    d1_ms = fms[1] / max(nl[1], 1)
    d1_bytes = cones[1] / max(nl[1], 1) * bpc
    peak, peak_kind = peaks()
    achieved = d1_bytes / (d1_ms / 1e3) / 1e9 if d1_ms > 0 else 0.0
    field_ms_step = sum(fms[d] for d in range(1, D + 1)) / args.steps
    roof = {"bound": "hbm", "kernel": "k_fields<128> (depth-1 fields)",
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

    # e2e through the public API: every pass's frame delivered to pinned host
    # memory by wavefront.FramePipeline (D2H of pass i overlapped with pass i+1)
    e2e = None
    if world == 1 and not args.no_e2e:
        frame_bytes = n_paths * 3 * 8
        pipe = wavefront.FramePipeline(sc, tree, g_cfg)
        for _ in pipe.run(range(sample, sample + 3)):  # API warm-up (captures both graphs)
            pass
        sample += 3
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        checksum = 0.0
        for _, f, _ in pipe.run(range(sample, sample + args.steps)):
            checksum += float(f[0, 0, 0])  # the host frame is read every step
        e2e_s = time.perf_counter() - t0
        sample += args.steps
        e2e = {"value": n_paths * args.steps / e2e_s, "unit": "path samples/s",
               "h2d_bytes_per_step": C.sizeof(_lib.PassConfig) + C.sizeof(_lib.Camera),
               "d2h_bytes_per_step": frame_bytes,
               "api": "paper_2405_06997_b200.wavefront.FramePipeline.run -> pinned host "
                      "frame per pass (copy of pass i overlapped with pass i+1)"}
    elif world > 1 and not args.no_e2e:
        # per rank: pass + deposit exchange + its band of the frame to pinned
        # host memory; whole-job time = max over ranks
        host = torch.empty((npx, 3), dtype=torch.float64, pin_memory=True)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_pass(gr, sample)
            sample += 1
            host.copy_(gr.frame, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                             device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": total_pix * args.steps / float(e2e_s.item()),
               "unit": "path samples/s",
               "h2d_bytes_per_step": C.sizeof(_lib.PassConfig) + C.sizeof(_lib.Camera),
               "d2h_bytes_per_step": npx * 3 * 8 + 4,
               "api": "wavefront.PassRunner.launch + multigpu.DepositExchange per rank, "
                      "band frame -> pinned host; max over ranks"}

    out = {
        "metric": "path samples/sec (guided wavefront pass)",
        "value": value, "unit": "path samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.tiled else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: "
        f"scenes/{SCENES[args.scene][0]}, path samples from the counter RNG",
        "config": {"workload": f"{SCENES[args.scene][2]} {args.width}x{args.height} "
                               + ("image tiled over the GPUs, " if args.tiled else "per GPU, ")
                               + 
                               f"1 spp guided pass, SVO depth {tree.depth}, D={D}, G={D}, N0={args.field_res}, "
                               f"l_min {g_cfg.l_min}, c_ray 512, "
                               f"{'product' if args.product else 'plain'} guiding",
                   "image": [args.width, image_height(args, world)],
                   "svo_nodes": tree.node_count,
                   "l2": "inputs larger than L2 (path state + guide tables > 126 MB)",
                   "parallelism": f"image bands x{world}" + (
                       f", per-pass deposit all-gather ({backend})" if world > 1 else "")},
        "bins_per_depth": stats.bins_per_depth, "rays_per_depth": stats.rays_per_depth,
        "svo_build_ms": build_ms,
        "gpu_launches": int(launches),
        "roofline": roof,
        "e2e": e2e,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, sc, tree, g_cfg, stats)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args, sc, tree, cfg, stats, seconds=None):
    """Time the CPU oracle (port of the reference's guided pass) on a bounded
    sample of the same workload: the guided field generation of a subset of
    the depth-1 bins plus the shading of their paths, scaled to path samples/s
    by the fraction of the pass's field work the sample covers."""
    try:
        from oracle import render as OR
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "path samples/s", "cores": 0, "kind": "port",
                "sample": f"oracle unavailable: {e}"}
    seconds = seconds or args.cpu_seconds
    return OR.time_guided_pass_sample(sc, tree, cfg, stats, args.width * args.height, seconds)


def run_reference(args):
    """--impl reference: the CPU port of the reference's guided pass (oracle/,
    C + OpenMP on every host core; the reference itself is Python/Cython and
    does not travel to the GPU box).  No CUDA anywhere on this arm.  Setup
    builds the SVO and runs the PT-first pass with the oracle; each step then
    times a bounded sample of the guided pass's field generation, scaled to the
    full pass by its bin counts.  Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
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
                          seed=args.seed, blur_sigma=1.0, epsilon=1e-2)
    wl = OR.CpuWorkload(sc, args.svo_res, cfg, seed=args.seed)
    n_paths = args.width * args.height
    budget = args.ref_seconds or min(10.0, 150.0 / max(1, args.warmup + args.steps))
    vals, ms = [], []
    for step in range(args.warmup + args.steps):
        r = wl.time_pass(n_paths, budget, seed=step)
        vals.append(r)
    timed = vals[args.warmup:]
    v = statistics.mean(x["value"] for x in timed)
    cb = dict(timed[-1])
    cb["value"] = v
    cb["sample"] += f"; {budget:.1f} s sample per step; " + cb.pop("setup")
    cb.pop("pass_seconds", None)
    print(json.dumps({
        "impl": "reference", "metric": "path samples/sec (guided wavefront pass)", "value": v,
        "unit": "path samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_paths / v * 1e3 if v else None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{SCENES[args.scene][2]} {args.width}x{args.height}, 1 spp guided pass, "
                               f"SVO depth {depth}, D={args.depth}",
                   "host": "CPU only, rank 0's host cores; n_gpus mirrors the B200 arm "
                           "this line is paired with"},
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
