"""Kernel timeline of GN HVPs (CUPTI via torch.profiler): real in-pipeline
durations per kernel category and the idle gaps between consecutive kernels.

    python tools/trace_hvp.py [deformation|state] [float64|float32] > gpurun_out/trace.json
"""
import collections
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402


def main():
    objective = sys.argv[1] if len(sys.argv) > 1 else "deformation"
    dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
    dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.02, order=2, dtype=dtype)
    rng = np.random.default_rng(0)
    I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
    v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
    w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
    cls = B.DeformationObjective if objective == "deformation" else B.StateObjective
    obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10))
    ev = obj.gradient(v)
    for _ in range(3):
        ev.hessian_vector(w, gauss_newton=True)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            ev.hessian_vector(w, gauss_newton=True)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs], key=lambda x: x[0])
    # second HVP only: split at the midpoint of the kernel list
    ks = ks[len(ks) // 2:]
    cat = collections.defaultdict(lambda: [0, 0.0, 0.0])  # n, busy us, gap-before us
    def name(n):
        n = n.replace("void ", "")
        base = n.split("<")[0].split("(")[0].replace("blr::", "")
        if base == "k_zlines":
            op = n.split(">,")[-1].split(">")[0].strip() if ">," in n else "?"
            return f"k_zlines[{op}]"
        return base[:40]
    prev_end = ks[0][0]
    for s, e, n in ks:
        c = cat[name(n)]
        c[0] += 1
        c[1] += e - s
        c[2] += max(0.0, s - prev_end)
        prev_end = max(prev_end, e)
    span = ks[-1][1] - ks[0][0]
    busy = sum(v[1] for v in cat.values())
    out = {"objective": objective, "dtype": dtype, "span_us": span, "busy_us": busy,
           "gap_us": sum(v[2] for v in cat.values()), "kernels": len(ks),
           "by_kernel": {k: {"n": v[0], "us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2),
                             "gap_before_us": round(v[2], 1)}
                         for k, v in sorted(cat.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
