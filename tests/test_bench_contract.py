"""bench.py's JSON-line contract on both arms, at a tiny workload: the
reference arm (CPU port, no CUDA) runs here; the B200 arm on the GPU box."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    env = dict(os.environ, PYTHONPATH=REPO)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                         env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


REF_ARGS = ["--width", "48", "--height", "32", "--svo-res", "64", "--steps", "1", "--warmup", "1"]


def _ref_config():
    sys.path.insert(0, REPO)
    import bench

    old = sys.argv
    sys.argv = ["bench.py"] + REF_ARGS
    try:
        args = bench.parse()
    finally:
        sys.argv = old
    return bench.workload_config(args, 6, 1)


def test_reference_arm_line():
    d = _run("--impl", "reference", *REF_ARGS)
    assert BASE <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "path samples/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["value"] == d["value"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    assert "full guided pass" in cb["sample"] and len(cb["pass_seconds"]) == 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # both arms print the same config for the same arguments
    assert d["config"] == _ref_config()


def test_reference_arm_maps_no_product_library():
    """The CPU arm runs the oracle only: the product library (and CUDA) is
    never mapped into its process."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference'] + %r; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('MAPS', 'libwfpg_b200' in maps, 'libcudart' in maps or 'libcuda.so' in maps)"
            % (REF_ARGS,))
    env = dict(os.environ, PYTHONPATH=REPO)
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("MAPS")][0]
    assert line == "MAPS False False", line


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run("--width", "96", "--height", "64", "--svo-res", "64", "--steps", "3", "--warmup", "3")
    assert BASE <= set(d) and d.get("impl", "b200") != "reference"
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and r["peak"] > 0 and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["kind"] in ("port", "reference")
    assert d["per_rank"][0]["paths_per_pass"] == 96 * 64


@pytest.mark.gpu
def test_b200_arm_two_ranks_gloo():
    """The N>1 launch path (torchrun, one process per rank, per-pass deposit
    exchange, max-over-ranks timing) on the one visible GPU over gloo."""
    env = dict(os.environ, PYTHONPATH=REPO, WFPG_DIST_BACKEND="gloo")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(REPO, "bench.py"),
         "--gpus", "2", "--width", "96", "--height", "64", "--svo-res", "64", "--steps", "3",
         "--warmup", "3", "--no-cpu-baseline"],
        cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["image"] == [96, 64] and d["e2e"]["value"] > 0
    assert [r["paths_per_pass"] for r in d["per_rank"]] == [3072, 3072]
    assert d["comm"]["backend"] == "gloo" and d["comm"]["kind"] == "host"
    assert d["comm"]["bin_ownership_depths"] == [2, 3, 4]
