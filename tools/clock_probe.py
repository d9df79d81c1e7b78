"""Does sampling clocks with nvidia-smi during a timed region perturb it?
Times R repetitions of K GN HVPs with and without the bench's Clocks sampler,
interleaved, and counts slow repetitions (> 3% above the median).  GPU box:
    python tools/clock_probe.py [--reps 15] [--steps 20] [--lms 50]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.02, order=2)
rng = np.random.default_rng(0)
I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
ev = B.DeformationObjective(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10)).gradient(v)
for _ in range(3):
    ev.hessian_vector(w, gauss_newton=True)
torch.cuda.synchronize()


class Null:
    def __enter__(self):
        return self

    def __exit__(self, *e):
        pass


res = {"clocks": [], "none": []}
for r in range(a.reps):
    for kind in ("clocks", "none"):
        ctx = bench.Clocks(0) if kind == "clocks" else Null()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ctx:
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                ev.hessian_vector(w, gauss_newton=True)
            e1.record()
            torch.cuda.synchronize()
        res[kind].append(e0.elapsed_time(e1) / a.steps)
for kind, ms in res.items():
    med = float(np.median(ms))
    slow = [round(x, 2) for x in ms if x > 1.03 * med]
    print(f"{kind}: median {med:.3f} ms/HVP, max {max(ms):.3f}, slow reps {len(slow)}/{len(ms)} {slow}")
