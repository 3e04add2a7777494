#!/usr/bin/env python
"""Kernel timeline of pipelined guided passes (torch.profiler / CUPTI, graph
replays included): per pass the wall span, the summed kernel time, the time
covered by at least one kernel, and the idle gaps on the GPU — how much of a
pass is launch / dependency latency rather than kernel work.
    python tools/kernel_timeline.py [--scene c2] [--passes 6]"""
import argparse
import collections
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default="c2")
    ap.add_argument("--passes", type=int, default=6)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2405_06997_b200 import wavefront

    saved = sys.argv
    sys.argv = ["bench.py", f"--scene={a.scene}"]
    args = bench.parse()
    sys.argv = saved
    sc, tree, pt_cfg, g_cfg, _ = bench.build_workload(args)
    wavefront.render_pass(sc, tree, pt_cfg, [0])
    pipe = wavefront.PassPipeline(sc, tree, g_cfg)
    s = 1
    for _ in range(6):
        pipe.launch(s)
        s += 1
    pipe.join()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.passes):
            pipe.launch(s)
            s += 1
        pipe.join()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and "wfpg" in e.name]
    ev.sort(key=lambda e: e.time_range.start)
    if not ev:
        print("no kernel events (CUPTI did not report graph kernels)")
        return
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:
        st, en = e.time_range.start, e.time_range.end
        if cur_e is None or st > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = st, en
        else:
            cur_e = max(cur_e, en)
    busy += cur_e - cur_s
    ksum = sum(e.time_range.end - e.time_range.start for e in ev)
    span = t1 - t0
    print(f"{a.passes} passes: span {span / 1e3:.3f} ms ({span / 1e3 / a.passes:.3f} ms/pass), "
          f"kernels {len(ev)} ({len(ev) / a.passes:.0f}/pass), summed kernel time "
          f"{ksum / 1e3:.3f} ms, covered {busy / 1e3:.3f} ms = {100 * busy / span:.1f}% of the span, "
          f"idle {100 * (span - busy) / span:.1f}%")
    per = collections.Counter()
    for e in ev:
        per[e.name.split("(")[0]] += e.time_range.end - e.time_range.start
    for k, v in per.most_common(12):
        print(f"  {k[:60]:60s} {v / 1e3 / a.passes:.3f} ms/pass")


if __name__ == "__main__":
    main()
