"""Host-side enqueue cost of one GN HVP at the headline configuration versus its
GPU time: if the host needs longer to issue an HVP than the GPU needs to run
it, the end-to-end number is host-bound.  Usage (GPU box):
    python tools/host_enqueue.py [--objective deformation|state] [--reps 20]
"""
import argparse
import os
import platform
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--objective", default="deformation")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.02, order=2)
rng = np.random.default_rng(0)
I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
cls = B.DeformationObjective if a.objective == "deformation" else B.StateObjective
ev = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10)).gradient(v)
for _ in range(3):
    ev.hessian_vector(w, gauss_newton=True)
torch.cuda.synchronize()
enq = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    t = time.perf_counter()
    ev.hessian_vector(w, gauss_newton=True)
    enq.append((time.perf_counter() - t) * 1e3)
e1.record()
torch.cuda.synchronize()
gpu = e0.elapsed_time(e1) / a.reps
print(f"{a.objective}: host enqueue per HVP median {np.median(enq):.2f} ms (min {min(enq):.2f}, max {max(enq):.2f});"
      f" GPU {gpu:.2f} ms per HVP; cpu {platform.processor() or platform.machine()} x{os.cpu_count()}")
