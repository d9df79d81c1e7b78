"""Probe: capture one GN HVP in a CUDA graph and compare replay time with eager launches."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1807_05117_b200 as B


objective = sys.argv[1] if len(sys.argv) > 1 else "deformation"
dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.01, order=2)
rng = np.random.default_rng(0)
import bench  # noqa: E402
I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / 128, 2.0)[None], 10, True)
cls = B.DeformationObjective if objective == "deformation" else B.StateObjective
obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10))
ev = obj.gradient(v)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        ref = ev.hessian_vector(w, gauss_newton=True)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
ref = ref.values.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    out = ev.hessian_vector(w, gauss_newton=True)
e1.record()
torch.cuda.synchronize()
print("eager ms/HVP", e0.elapsed_time(e1) / 20)
g = torch.cuda.CUDAGraph()
t0 = time.perf_counter()
try:
    with torch.cuda.graph(g):
        gout = ev.hessian_vector(w, gauss_newton=True)
except Exception as exc:
    print("capture failed:", exc)
    sys.exit(0)
t1 = time.perf_counter()
g.replay()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"capture {1e3 * (t1 - t0):.1f} ms, first replay (instantiate) {1e3 * (t2 - t1):.1f} ms")
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ev.hessian_vector(w, gauss_newton=True)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print(f"eager host issue time of one HVP (idle queue) {1e3 * min(ts):.2f} ms")
print("graph max |diff|", float((gout.values - ref).abs().max()), "ref max", float(ref.abs().max()))
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
print("graph ms/HVP", e0.elapsed_time(e1) / 20)
