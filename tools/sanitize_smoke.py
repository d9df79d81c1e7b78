"""Small end-to-end run (both objectives, 32^3 / K=8 so the pad engine runs at
L=25 and 28, fp64 and fp32) for compute-sanitizer."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1807_05117_b200 as B
import bench

for dtype in ("float64", "float32"):
    for shape, K in (((32, 32, 32), 8), ((20, 24, 28), 6)):
        dom = B.Domain(shape, (K,) * 3, alpha=0.05, dtype=dtype)
        rng = np.random.default_rng(1)
        I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
        v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.05, 2.0)[None], 4, True)
        w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.05, 2.0)[None], 4, True)
        for cls in (B.StateObjective, B.DeformationObjective):
            obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=4))
            ev = obj.gradient(v)
            hv = ev.hessian_vector(w, gauss_newton=True)
            hv2 = ev.hessian_vector(w, gauss_newton=False)
            print(dtype, shape, cls.__name__, float(hv.values.abs().max()), float(hv2.values.abs().max()))
print("ok")
