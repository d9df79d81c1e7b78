"""End-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck):
both objectives, energy + gradient + GN and Newton HVPs, fp64 and fp32.

    python tools/sanitize_smoke.py [small|l100|l196] [--fused]

small: 32^3/K=8 and 20x24x28/K=6 (pad lengths 25, 28, 20); l100: 128^3/K=32
(the benchmarked L = 100 = 10 x 10 instantiation) at Nt=2; l196: 136^3/K=64
(L = 196 = 14 x 14) at Nt=1.  --fused turns on the cluster forward projection.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import _lib  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "small"
if "--fused" in sys.argv:
    _lib.call("blr_set_fused_forward", 1)
cases = {"small": [((32, 32, 32), 8, 4), ((20, 24, 28), 6, 4)],
         "l100": [((128, 128, 128), 32, 2)],
         "l196": [((136, 136, 136), 64, 1)]}[which]
dtypes = ("float64", "float32") if which == "small" else ("float64",)
for dtype in dtypes:
    for shape, K, nt in cases:
        dom = B.Domain(shape, (K,) * 3, alpha=0.05, dtype=dtype)
        rng = np.random.default_rng(1)
        I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
        v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / shape[0], 2.0)[None], nt, True)
        w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / shape[0], 2.0)[None], nt, True)
        for cls in (B.StateObjective, B.DeformationObjective):
            obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=nt))
            e = obj.energy(v)
            ev = obj.gradient(v)
            hv = ev.hessian_vector(w, gauss_newton=True)
            hv2 = ev.hessian_vector(w, gauss_newton=False)
            print(dtype, shape, dom.pad, cls.__name__, e, float(hv.values.abs().max()),
                  float(hv2.values.abs().max()), flush=True)
print("ok")
