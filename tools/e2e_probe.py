"""Per-step anatomy of bench.py's end-to-end loop (pinned host in -> HVP ->
host out, copies on a side stream): GPU time per step from events on the
compute stream, host time per step, clocks sampled during each repetition.
Finds where an occasional slow e2e repetition loses its time.  GPU box:
    python tools/e2e_probe.py [--reps 5] [--steps 20]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.02, order=2)
rng = np.random.default_rng(0)
I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
ev = B.DeformationObjective(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10)).gradient(v)
stream = torch.cuda.current_stream()
host_w = torch.from_numpy(w.values.cpu().numpy()).pin_memory()
host_out = torch.empty_like(host_w).pin_memory()
dev_in = [torch.empty_like(w.values) for _ in range(2)]
copy = torch.cuda.Stream()
in_ready = [torch.cuda.Event() for _ in range(2)]


def pipelined(n, marks=None):
    copy.wait_stream(stream)
    with torch.cuda.stream(copy):
        dev_in[0].copy_(host_w, non_blocking=True)
        in_ready[0].record(copy)
    done_prev = hv = None
    for k in range(n):
        t = time.perf_counter()
        stream.wait_event(in_ready[k % 2])
        if marks is not None:
            marks[k][0].record(stream)
        hv = ev.hessian_vector(B.TimeFlow(dom, dev_in[k % 2], 10, True), gauss_newton=True)
        if marks is not None:
            marks[k][1].record(stream)
        done = torch.cuda.Event()
        done.record(stream)
        with torch.cuda.stream(copy):
            if k + 1 < n:
                if done_prev is not None:
                    copy.wait_event(done_prev)
                dev_in[(k + 1) % 2].copy_(host_w, non_blocking=True)
                in_ready[(k + 1) % 2].record(copy)
            copy.wait_event(done)
            host_out.copy_(hv.values, non_blocking=True)
        hv.values.record_stream(copy)
        done_prev = done
        if marks is not None:
            marks[k][2] = (time.perf_counter() - t) * 1e3
    stream.wait_stream(copy)
    return hv


import gc  # noqa: E402

gc_log = []
_gc_t = {}


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t["t"] = time.perf_counter()
    else:
        gc_log.append((info["generation"], (time.perf_counter() - _gc_t.get("t", time.perf_counter())) * 1e3,
                       info.get("collected", 0)))


gc.callbacks.append(_gc_cb)
pipelined(3)
torch.cuda.synchronize()
for rep in range(a.reps):
    st0 = torch.cuda.memory_stats()
    marks = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), 0.0] for _ in range(a.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.Clocks(0) as clk:
        e0.record(stream)
        pipelined(a.steps, marks)
        e1.record(stream)
        torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    hvp = [m[0].elapsed_time(m[1]) for m in marks]
    gaps = [marks[k][0].elapsed_time(marks[k + 1][0]) - hvp[k] for k in range(a.steps - 1)]
    host = [m[2] for m in marks]
    print(f"rep {rep}: {a.steps / tot * 1e3:.2f} HVP/s total {tot:.1f} ms | HVP ms min {min(hvp):.2f} med "
          f"{np.median(hvp):.2f} max {max(hvp):.2f} | gap ms max {max(gaps):.2f} sum {sum(gaps):.2f} | host ms "
          f"med {np.median(host):.2f} max {max(host):.2f} (step {int(np.argmax(host))}) | clocks {clk.summary()}")
    slow = [(g, round(ms, 1)) for g, ms, _ in gc_log if ms > 2.0]
    print("   gc: %d collections (gen2: %d), slow (gen, ms): %s" % (
        len(gc_log), sum(1 for g, _, _ in gc_log if g == 2), slow))
    gc_log.clear()
    st1 = torch.cuda.memory_stats()
    print("   allocator: segments +%d, cudaMalloc retries +%d, reserved %.2f GB" % (
        st1["segment.all.allocated"] - st0["segment.all.allocated"],
        st1["num_alloc_retries"] - st0["num_alloc_retries"], st1["reserved_bytes.all.current"] / 1e9))
