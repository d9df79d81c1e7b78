#!/usr/bin/env python
"""Headline benchmark: Gauss-Newton Hessian-vector products per second at
128^3 (K=32 band), Nt=10, fp64 — BASELINE.json config 3 ("EPDiff" variant,
mapped to the reference's DeformationObjective).

One *step* = one ``Evaluation.hessian_vector(w, gauss_newton=True)`` at a
fixed evaluation point (the unit of work inside every PCG iteration).  Inputs
follow the SURVEY §8(d) micro-benchmark recipe (``band_image`` pair, smooth
``v`` / ``w``, seed 0), generated on the device.  The HVP working set
(multi-GB stage caches) is far larger than the 126 MB L2, so no explicit L2
flush is needed between steps.

Arms:
  default           the B200 path; prints one JSON line with value, e2e
                    (host-pinned inputs/outputs through the public API),
                    roofline of the dominant kernel, cpu_baseline, clocks.
  --impl reference  the reference algorithm on the host CPU (the oracle port
                    in ``oracle/``, all host threads), bounded samples.

Multi-GPU (torchrun): one independent registration pair per rank (the batch
configuration shards pairs, no data-path collective); value = sum over ranks,
timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian-vector products/sec and s/registration at 128^3 (32^3 band, Nt=10); % HBM roofline"
UNIT = "HVP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference", "selftest"], default="b200")
    ap.add_argument("--objective", choices=["deformation", "state"], default="deformation")
    ap.add_argument("--dtype", choices=["float64", "float32"], default="float64")
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--band", type=int, default=32)
    ap.add_argument("--nt", type=int, default=10)
    ap.add_argument("--registration", type=int, default=1, help="also time one full GN registration")
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--profile-only", action="store_true", help="one instrumented HVP, no timing")
    ap.add_argument("--in-flight", type=int, default=1,
                    help="--batch: pairs registered concurrently per GPU (threads + streams)")
    ap.add_argument("--batch", type=int, default=0,
                    help="SURVEY config 5: register this many seeded pairs sharded over the ranks "
                         "(NCCL atlas all_reduce + stats all_gather) and report pairs/s instead of HVP/s")
    return ap.parse_args()


def workload(args):
    return {"workload": f"{args.objective}_gn_hvp_{args.size}^3_K{args.band}_Nt{args.nt}",
            "objective": args.objective, "grid": [args.size] * 3, "bandwidth": [args.band] * 3,
            "n_time_steps": args.nt, "sigma2": 0.1, "alpha": 0.02, "order": 2,
            "l2": "working set (GB-scale stage caches) >> 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

_BACKEND = {"name": "nccl"}


def free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(nproc):
    """``python bench.py --gpus N`` (N > 1) without torchrun: re-launch this
    script under torch.distributed.run, one rank per GPU, and return its exit
    code (the ranks print the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(backend="nccl"):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    _BACKEND["name"] = backend
    if world > 1:
        import torch
        import torch.distributed as dist

        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _dev():
    return "cuda" if _BACKEND["name"] == "nccl" else "cpu"


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_report(world, t_ms, e2e_ms, launches):
    """Per-rank timings and evidence gathered over the communicator: device
    ms of the timed region, e2e ms, kernel launches, whether this rank loaded
    the in-tree sm_100a library, and the communicator size."""
    import torch
    import torch.distributed as dist

    loaded = 0.0
    try:
        with open("/proc/self/maps") as f:
            loaded = float("libblreg_b200.so" in f.read())
    except OSError:
        pass
    mine = torch.tensor([float(dist.get_rank()), t_ms, e2e_ms, float(launches), loaded],
                        dtype=torch.float64, device=_dev())
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    return {"backend": dist.get_backend(), "comm_size": dist.get_world_size(),
            "per_rank": [{"rank": int(r[0]), "ms": round(float(r[1]), 3), "e2e_ms": round(float(r[2]), 3),
                          "gpu_launches": int(r[3]), "native_lib_loaded": bool(r[4])}
                         for r in (x.cpu() for x in allv)]}


def run_selftest(args, rank, world):
    """--impl selftest: the multi-rank plumbing (spawn, barrier, max over
    ranks, per-rank gather) on gloo with a sleep standing in for the GPU step;
    used by the CPU test suite."""
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.01 * (1 + rank))
    local_ms = 1e3 * (time.perf_counter() - t0)
    t_ms = max_over_ranks(local_ms, world)
    line = {"metric": "selftest", "value": world * args.steps / (t_ms / 1e3), "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "impl": "selftest"}
    if world > 1:
        line["ranks"] = rank_report(world, local_ms, local_ms, 0)
    if rank == 0:
        print(json.dumps(line))


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # the sampler is live once its first line arrives; drop that pre-region sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic inputs (SURVEY.md §8(d) recipe, generated through the product API)
# ---------------------------------------------------------------------------

def _freq(m):
    k = (m - 1) // 2
    return np.concatenate([np.arange(0, k + 1), np.arange(-k, 0)])


def smooth_vector_block(dom, rng, scale, decay):
    """tests/helpers.py:22-37 recipe on the device: symmetrize, power-law decay,
    normalise the max-norm of the realization to ``scale``."""
    from paper_1807_05117_b200 import spectral

    sh = (dom.ndim,) + dom.block_shape
    c = rng.standard_normal(sh) + 1j * rng.standard_normal(sh)
    c = spectral.symmetrize(dom, c)
    k2 = np.zeros(dom.block_shape)
    for ax, m in enumerate(dom.block_shape):
        shp = [1] * dom.ndim
        shp[ax] = m
        k2 = k2 + (_freq(m).astype(float) ** 2).reshape(shp)
    import torch

    c = c / torch.from_numpy((1.0 + k2) ** decay).to(c.device)
    return c * (scale / spectral.max_abs(dom, c))


def band_image(dom, rng, decay=3.0):
    from paper_1807_05117_b200 import spectral

    c = smooth_vector_block(dom, rng, 1.0, decay)[0]
    img = spectral.include(dom, c)
    img = img - img.min()
    return img / img.max()


def blob_pair(dom, seed=1, amp=3.0):
    """Seeded 3-D registration pair: periodic bumps, target = source warped
    (cubic) by a smooth ~``amp``-voxel displacement (the reference's pairs are 2-D)."""
    import torch

    from paper_1807_05117_b200 import Domain, gridops, spectral

    n = dom.shape[0]
    rng = np.random.default_rng(seed)
    axes = [np.arange(s) / s for s in dom.shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    src = np.zeros(dom.shape)
    for _ in range(6):
        c = 0.3 + 0.4 * rng.random(3)
        sharp = 8.0 + 16.0 * rng.random()
        b = np.ones(dom.shape)
        for x, cc in zip(mesh, c):
            b = b * np.exp(sharp * (np.cos(2 * np.pi * (x - cc)) - 1.0))
        src += (0.5 + 0.5 * rng.random()) * b
    src /= src.max()
    ddom = Domain(dom.shape, (4,) * dom.ndim, dtype=dom.dtype, device=dom.device)
    disp = spectral.include(ddom, smooth_vector_block(ddom, rng, amp / n, 2.0))
    tgt = gridops.warp(ddom, torch.from_numpy(src), disp, "cubic")
    return src, tgt.double().cpu().numpy()


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def survey_model_bytes(args, dom):
    """SURVEY §8(d) / Appendix A.8 algorithmic bytes of one GN HVP at the pad in use:
    F_pad * 2S(P^3+B^3) + X_full * 2S(N^3+B^3) + G * S*N^3 (no cross-HVP caching)."""
    S = 8 if args.dtype == "float64" else 4
    P3 = int(np.prod(dom.pad))
    B3 = (2 * args.band + 1) ** 3
    N3 = args.size ** 3
    nt = args.nt
    if args.objective == "state":
        F, X, G = 4 * nt * 24 + 6, 3 + 3 * (nt + 1), 6 + 12 * (nt + 1)
    else:
        F, X, G = (4 * nt * 24 + 6) + (4 * nt * 12 + 3) + 15 * (nt + 1), 6, 12
    return float(F * 2 * S * (P3 + B3) + X * 2 * S * (N3 + B3) + G * S * N3)


def ncu_traffic(workload_name, dtype, pad, kernel):
    """DRAM bytes per launch of ``kernel`` from a committed ncu capture of
    exactly this workload / dtype / pad (profiles/ncu_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            caps = json.load(f)["captures"]
    except Exception:
        return None
    for c in caps:
        if (c["workload"], c["dtype"], list(c["pad"]), c["kernel"]) == (workload_name, dtype, list(pad), kernel):
            return c["traffic"]
    return None


def run_b200(args, rank, world, local):
    import torch

    import paper_1807_05117_b200 as B
    from paper_1807_05117_b200 import _lib

    torch.cuda.set_device(local)
    dom = B.Domain((args.size,) * 3, (args.band,) * 3, alpha=0.02, order=2, dtype=args.dtype,
                   device=local)
    rng = np.random.default_rng(0)
    I0 = band_image(dom, rng)
    I1 = band_image(dom, rng)
    v = B.TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / args.size, 2.0)[None], args.nt, True)
    w = B.TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / args.size, 2.0)[None], args.nt, True)
    cls = B.DeformationObjective if args.objective == "deformation" else B.StateObjective
    cfg = B.ProblemConfig(sigma2=0.1, n_time_steps=args.nt)
    obj = cls(dom, I0, I1, cfg)
    ev = obj.gradient(v)
    torch.cuda.synchronize()

    def instrumented():
        """One HVP with per-kernel-category events: time and algorithmic bytes."""
        _lib.profile_enable(True)
        ev.hessian_vector(w, gauss_newton=True)
        torch.cuda.synchronize()
        rep = _lib.profile_report()
        _lib.profile_enable(False)
        return rep

    if args.profile_only:
        prof = instrumented()
        if rank == 0:
            print(json.dumps({"profile": prof}))
        return

    for _ in range(args.warmup):
        ev.hessian_vector(w, gauss_newton=True)
    torch.cuda.synchronize()
    barrier(world)
    stream = torch.cuda.current_stream()
    # three timed windows of exactly K steps, each bracketed by a barrier and a
    # synchronize; the median window is reported and all three are in the line
    # (`windows_ms`): a host stall longer than the ~2 HVPs of queued launches
    # idles the GPU, and such stalls (~0.1-0.3 s, rare, not the path's cost)
    # were seen on fresh boxes
    windows = []
    launches = 0
    with Clocks(local) as clocks:
        for _win in range(3):
            barrier(world)
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = _lib.launch_count()
            torch.cuda.synchronize()
            start.record(stream)
            for _ in range(args.steps):
                out = ev.hessian_vector(w, gauss_newton=True)
            end.record(stream)
            torch.cuda.synchronize()
            launches = _lib.launch_count() - l0
            windows.append(start.elapsed_time(end))
    barrier(world)
    local_ms = float(np.median(windows))
    t_ms = max_over_ranks(local_ms, world)
    # the per-category breakdown and the roofline come from an instrumented HVP
    # taken after the timed windows (warm caches and allocator, like the timed
    # steps; the first HVP after the gradient runs a few percent slower)
    prof = instrumented()
    per_step_ms = t_ms / args.steps
    value = world * args.steps / (t_ms / 1e3)

    # end to end through the public API with pinned host buffers: every step copies
    # its direction host->device and its product device->host.  The copies run on
    # a second stream, double-buffered, so step k+1's upload and step k's
    # download overlap step k's HVP (the way a host-driven solver would pipeline).
    host_w = torch.from_numpy(w.values.cpu().numpy()).pin_memory()
    host_out = torch.empty_like(host_w).pin_memory()
    dev_in = [torch.empty_like(w.values) for _ in range(2)]
    copy = torch.cuda.Stream(device=local)
    in_ready = [torch.cuda.Event() for _ in range(2)]

    def pipelined(nsteps):
        """nsteps HVPs through the public API, host in -> host out; returns the last product."""
        copy.wait_stream(stream)
        with torch.cuda.stream(copy):
            dev_in[0].copy_(host_w, non_blocking=True)
            in_ready[0].record(copy)
        done_prev = hv = None
        for k in range(nsteps):
            stream.wait_event(in_ready[k % 2])
            hv = ev.hessian_vector(B.TimeFlow(dom, dev_in[k % 2], args.nt, True), gauss_newton=True)
            done = torch.cuda.Event()
            done.record(stream)
            with torch.cuda.stream(copy):
                if k + 1 < nsteps:
                    if done_prev is not None:  # step k-1 has finished reading this buffer
                        copy.wait_event(done_prev)
                    dev_in[(k + 1) % 2].copy_(host_w, non_blocking=True)
                    in_ready[(k + 1) % 2].record(copy)
                copy.wait_event(done)
                host_out.copy_(hv.values, non_blocking=True)
            hv.values.record_stream(copy)
            done_prev = done
        stream.wait_stream(copy)
        return hv

    # untimed warm-up of the pipelined loop: the allocator's growth under
    # record_stream (product buffers held by the copy stream) is first-use set-up
    hv = pipelined(max(args.warmup, 2))
    torch.cuda.synchronize()
    # three repetitions of the K-step loop, the median reported (all three are
    # in the line): one host hiccup of ~0.1 s inside a 0.2 s region was seen
    # on a fresh box (tools/e2e_probe.py), and it is not the path's cost
    e2e_reps = []
    for _ in range(3):
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hv = pipelined(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_reps.append(e0.elapsed_time(e1))
    local_e2e_ms = float(np.median(e2e_reps))
    e2e_ms = max_over_ranks(local_e2e_ms, world)
    e2e_value = world * args.steps / (e2e_ms / 1e3)
    assert torch.equal(host_out, out.values.cpu()), "e2e result differs from the device-resident run"

    # s/registration: full Gauss-Newton-Krylov registrations of two 3-D pairs:
    # the default (~3-voxel displacement, substeps 1) and a hard one (~12
    # voxels) whose CFL monitor refines the time stepping (substeps > 1)
    reg = None
    reg_hard = None
    if args.registration:
        del ev, out, hv

        def register(amp, seed, label):
            src, tgt = blob_pair(dom, seed=seed, amp=amp)
            robj = cls(dom, src, tgt, B.ProblemConfig(sigma2=0.03, n_time_steps=args.nt))
            # one untimed registration first: cache allocations and first-use set-up
            # (allocator growth for the GB-scale stage caches) are not per-registration costs
            B.minimize(robj, B.TimeFlow.zero(dom, args.nt), B.SolverConfig())
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = B.minimize(robj, B.TimeFlow.zero(dom, args.nt), B.SolverConfig())
            torch.cuda.synchronize()
            reg_s = max_over_ranks(time.perf_counter() - t0, world)
            jd = B.gridops.jacobian_determinant(
                dom, B.spectral.include(dom, res.evaluation.cache.forward[-1], check=False))
            return {"s_per_registration": reg_s, "status": res.status, "outer": len(res.records),
                    "pcg_total": res.total_pcg_iters, "final_mse_rel": res.final_mse_rel,
                    "j_min": float(jd.min()), "j_max": float(jd.max()),
                    "calls": {k: (v if not isinstance(v, list) else
                                  {"n": len(v), "mean_substeps": float(np.mean(v)) if v else 0.0,
                                   "max_substeps": int(max(v)) if v else 0})
                              for k, v in res.counters.items()},
                    "pair": label}

        reg = register(3.0, 1, "6 periodic bumps, target = cubic warp by band-4 displacement (3 vox)")
        reg_hard = register(12.0, 2, "6 periodic bumps, target = cubic warp by band-4 displacement (12 vox; "
                                     "CFL refinement)")

    # roofline of the dominant kernel category (live CUDA events)
    peak, peak_kind = peaks()
    total_prof_ms = sum(v[1] for v in prof.values())
    breakdown = {k: {"launches": int(v[0]), "ms": round(v[1], 4),
                     "share": round(v[1] / total_prof_ms, 4) if total_prof_ms else None,
                     "gbs": round(v[2] / (v[1] * 1e-3) / 1e9, 1) if v[1] > 0 else None}
                 for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    dom_name, dv = max(prof.items(), key=lambda kv: kv[1][1])
    n_launch, ms, nbytes = dv
    achieved = nbytes / n_launch / (ms / n_launch * 1e-3) / 1e9
    tr = ncu_traffic(workload(args)["workload"], "f64" if args.dtype == "float64" else "f32", list(dom.pad),
                     dom_name)
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": tr, "algorithmic_bytes_per_launch": nbytes / n_launch,
                "avg_launch_us": ms / n_launch * 1e3}

    # whole-HVP view of the metric's "% HBM roofline": the engine's compulsory
    # bytes per HVP (sum of the per-kernel counts above, with the D(u) / D(phi)
    # caches) and the SURVEY §8(d) byte model at this pad (no cross-HVP caching)
    hvp_bytes = sum(v[2] for v in prof.values())
    model_bytes = survey_model_bytes(args, dom)
    t_s = per_step_ms * 1e-3
    roofline_hvp = {"bytes_per_hvp": hvp_bytes, "achieved": round(hvp_bytes / t_s / 1e9, 1),
                    "frac": round(hvp_bytes / t_s / 1e9 / peak, 4),
                    "survey_model_bytes": model_bytes,
                    "survey_model_frac": round(model_bytes / t_s / 1e9 / peak, 4),
                    "peak": peak, "unit": "GB/s",
                    "note": "bytes/HVP over the timed ms/HVP; the survey model counts realized pad "
                            "passes c_pad = 2S(P^3+B^3) without the stage caches"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if args.dtype == "float64" else "f32",
        "data": "synthetic (band_image pair + smooth v, w; SURVEY §8(d) recipe, seed 0)",
        "config": {**workload(args), "pad": list(dom.pad), "parallelism": f"replicas x{world}"},
        "windows_ms": [round(x, 3) for x in windows],
        "e2e": {"value": e2e_value, "unit": UNIT, "reps_ms": [round(x, 3) for x in e2e_reps],
                "h2d_bytes_per_step": host_w.numel() * host_w.element_size(),
                "d2h_bytes_per_step": host_out.numel() * host_out.element_size()},
        "gpu_launches": launches,
        "roofline": roofline,
        "roofline_hvp": roofline_hvp,
        "kernel_breakdown": breakdown,
        "clocks": clocks.summary(),
    }
    if reg:
        line["registration"] = reg
    if reg_hard:
        line["registration_hard"] = reg_hard
    if world > 1:
        line["ranks"] = rank_report(world, local_ms, local_e2e_ms, launches)
    if rank == 0 and world == 1 and args.cpu_baseline:
        cpu = cpu_baseline(args, dom.pad, reg, reg_hard)
        for r, key in ((reg, "registration"), (reg_hard, "registration_hard")):
            if r is not None and key in cpu:
                r["cpu_s_estimate"] = cpu[key]["cpu_s_estimate"]
                r["cpu_ratio"] = cpu[key]["ratio"]
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line))


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port on the host cores)
# ---------------------------------------------------------------------------

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import blreg_oracle as O

    return O


class HostThreads:
    """Run the port on ``n`` host threads: scipy.fft workers = n and, for n = 1,
    the process pinned to one core (``taskset`` equivalent); restored on exit."""

    def __init__(self, O, n):
        self.O, self.n = O, n

    def __enter__(self):
        self.prev_workers = self.O.WORKERS
        self.O.WORKERS = self.n
        self.prev_aff = os.sched_getaffinity(0)
        if self.n == 1:
            os.sched_setaffinity(0, {min(self.prev_aff)})
        return self

    def __exit__(self, *exc):
        self.O.WORKERS = self.prev_workers
        os.sched_setaffinity(0, self.prev_aff)


def host_cores():
    return len(os.sched_getaffinity(0))


def port_problem(args, pad):
    """The §8(d) micro-benchmark problem in the oracle port at ``pad`` (the
    same inputs as the B200 arm, generated by the same seeded recipe)."""
    O = _oracle()
    n, k, nt = args.size, args.band, args.nt
    dom = O.Dom((n,) * 3, (k,) * 3, alpha=0.02, order=2, pad=tuple(pad))
    rng = np.random.default_rng(0)
    I0, I1 = O.band_image(dom, rng), O.band_image(dom, rng)
    v = O.Flow(dom, O.smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], nt, True)
    w = O.Flow(dom, O.smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], nt, True)
    kind = "def" if args.objective == "deformation" else "state"
    obj = O.OracleObjective(dom, I0, I1, O.Problem(sigma2=0.1, n_time_steps=nt), kind=kind)
    return O, dom, obj, v, w


def _timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def cpu_stage_sample(args, pad):
    """One forward-tangent RK4 stage (+ one momentum stage and one node
    contraction for the deformation objective) of the port, and the count of
    each per GN HVP.  Used only for the 1-core figure, which is an estimate."""
    O = _oracle()
    n, k, nt = args.size, args.band, args.nt
    dom = O.Dom((n,) * 3, (k,) * 3, alpha=0.02, order=2, pad=tuple(pad))
    rng = np.random.default_rng(0)
    u, du, v, dv = (O.smooth_vector_block(dom, rng, 0.5 / n, 2.0) for _ in range(4))
    stages = 4 * nt
    _, t_fwd = _timed(lambda: (O.rhs_map(dom, u, v), O.rhs_map_tangent(dom, u, du, v, dv)))
    total, sample = stages * t_fwd, t_fwd
    desc = f"1 forward-tangent RK4 stage x{stages}"
    if args.objective == "deformation":
        _, t_mom = _timed(lambda: O.rhs_momentum_pair(dom, u, du, v, None))
        _, t_con = _timed(lambda: O.conv_matvec(dom, O.jac(dom, u), du, transpose=True))
        total += stages * t_mom + (nt + 1) * t_con
        sample += t_mom + t_con
        desc += f" + 1 momentum stage x{stages} + 1 node contraction x{nt + 1}"
    return total, sample, desc


def cpu_baseline(args, pad, reg=None, reg_hard=None):
    """SURVEY §8(d) CPU rows, measured on this host in this session:

    * all cores: one WHOLE energy, gradient and GN HVP of the port (timed, not
      scaled), at the B200 arm's exact pad;
    * one core (pinned, 1 FFT worker): a stage sample scaled to one HVP
      (labelled an estimate; a whole 1-core HVP takes minutes);
    * CPU s/registration estimate t_CPU = sum over the B200 registration's
      calls of substeps x t_op (transport cost is linear in substeps)."""
    O, dom, obj, v, w = port_problem(args, pad)
    cores = host_cores()
    with HostThreads(O, cores):
        _, t_energy = _timed(lambda: obj.energy(v))
        ev, t_grad = _timed(lambda: obj.gradient(v))
        _, t_hvp = _timed(lambda: obj.hessian_vector(ev, w, gauss_newton=True))
    del ev
    with HostThreads(O, 1):
        t1, t1_sample, desc1 = cpu_stage_sample(args, pad)
    t1_hvp = t1
    out = {"value": 1.0 / t_hvp, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"1 whole {args.objective} GN HVP of the oracle port at {args.size}^3/K={args.band}/"
                     f"Nt={args.nt}, pad {pad[0]} (= the B200 arm's pad; the reference's own pad "
                     f"132 has 2.3x more points, so this baseline is conservative), scipy.fft on "
                     f"{cores} threads, after one untimed gradient (the HVP's evaluation point)",
           "seconds_per_hvp": round(t_hvp, 3),
           "per_op_s": {"energy": round(t_energy, 3), "gradient": round(t_grad, 3),
                        "hvp_gn": round(t_hvp, 3)},
           "one_core": {"value": 1.0 / t1, "unit": UNIT, "cores": 1, "estimated": True,
                        "seconds_per_hvp_estimated": round(t1, 2), "sample_seconds": round(t1_sample, 2),
                        "sample": desc1 + " (process pinned to one core, 1 FFT worker)"}}
    def estimate(r):
        calls = r["calls"]

        def cost(name, t_op):
            sub = calls.get(f"{name}_substeps")
            n = calls.get(name, 0)
            mean_sub = sub["mean_substeps"] if isinstance(sub, dict) and sub.get("n") else 1.0
            return n * mean_sub * t_op

        t_cpu = cost("gradient", t_grad) + cost("hvp", t_hvp) + cost("energy", t_energy)
        return {"cpu_s_estimate": round(t_cpu, 2), "gpu_s": r["s_per_registration"],
                "ratio": round(t_cpu / r["s_per_registration"], 1), "north_star_ratio": 50.0,
                "formula": "sum over the B200 run's calls (gradient, hvp, energy) of n x mean substeps x "
                           "the all-core per-op time above"}

    for r, key in ((reg, "registration"), (reg_hard, "registration_hard")):
        if r and r.get("calls"):
            out[key] = estimate(r)
    if reg and reg.get("calls"):
        # SURVEY §8(d) "all-cores throughput for the batch": one single-threaded
        # registration per core, each costing the all-core estimate scaled by the
        # measured 1-core / all-core HVP ratio (an estimate built on estimates)
        t1 = out["registration"]["cpu_s_estimate"] * (t1_hvp / t_hvp)
        out["batch_all_cores_estimate"] = {
            "pairs_per_s": round(cores / t1, 5), "cores": cores, "estimated": True,
            "s_per_registration_one_core": round(t1, 1),
            "gpu_pairs_per_s_single_registration": round(1.0 / reg["s_per_registration"], 3)}
    return out


def run_batch(args, rank, world, local):
    """Config 5: a batch of independent registrations, round-robin over the ranks."""
    import torch

    import paper_1807_05117_b200 as B
    from paper_1807_05117_b200 import batch as Bt

    torch.cuda.set_device(local)
    dom = B.Domain((args.size,) * 3, (args.band,) * 3, alpha=0.01, order=2, dtype=args.dtype, device=local)
    problem = B.ProblemConfig(sigma2=0.03, n_time_steps=args.nt)
    cfg = B.SolverConfig()

    # inputs resident in host memory before the timed region (the batch's I/O is not timed)
    mine = Bt.shard(args.batch, rank, world)
    pairs = {i: blob_pair(dom, seed=1 + i) for i in mine}

    def pair(i):
        return pairs[i]

    # warm-up: one untimed pair per rank (cache allocation, first-use set-up)
    warm = Bt.register_pair_fn(dom, problem, cfg, args.objective)
    warm(*blob_pair(dom, seed=10_000 + rank))
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    res = Bt.register_batch(pair, n_pairs=args.batch, domain=dom, problem=problem, solver_cfg=cfg,
                            objective=args.objective, in_flight=args.in_flight)
    torch.cuda.synchronize()
    wall = max_over_ranks(time.perf_counter() - t0, world)
    if rank == 0:
        st = res.stats
        line = {"metric": "registrations/s (batch of seeded 3-D pairs, SURVEY config 5)",
                "value": args.batch / wall, "unit": "pairs/s", "n_gpus": world, "steps": 1, "warmup": 1,
                "ms_per_step": 1e3 * wall, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64" if args.dtype == "float64" else "f32",
                "data": "synthetic (blob_pair seeds 1..P: 6 periodic bumps, cubic-warped target)",
                "config": {**workload(args), "workload": f"batch_{args.batch}x_{args.objective}_registration",
                           "sigma2": 0.03, "alpha": 0.01, "solver": "SolverConfig() defaults (GN, 10 inner)",
                           "pairs": args.batch, "in_flight_per_gpu": args.in_flight,
                           "parallelism": f"pairs round-robin over {world} ranks, {args.in_flight} in flight per GPU"},
                "batch": {"pcg_total_mean": float(st[:, Bt.STATS.index("pcg_total")].mean()),
                          "outer_mean": float(st[:, Bt.STATS.index("outer")].mean()),
                          "converged": int((st[:, Bt.STATS.index("status")] == 0).sum()),
                          "pair_wall_s_max": float(st[:, Bt.STATS.index("wall_s")].max())}}
        print(json.dumps(line))


def run_reference(args, rank, world):
    """The reference algorithm on the host CPU: the oracle port (numpy +
    scipy.fft on every host thread) at the B200 arm's exact pad.  One step =
    one WHOLE GN HVP, timed; the evaluation point (one gradient) is untimed
    set-up.  Warm-up: min(W, 1) HVP (CPU code has no first-use costs beyond
    scipy's FFT plan cache).  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    sys.path.insert(0, ROOT)
    from paper_1807_05117_b200.domain import default_pad

    pad = default_pad((args.band,) * 3)
    O, dom, obj, v, w = port_problem(args, pad)
    cores = host_cores()
    t_all0 = time.perf_counter()
    with HostThreads(O, cores):
        ev, t_grad = _timed(lambda: obj.gradient(v))
        for _ in range(min(args.warmup, 1)):
            obj.hessian_vector(ev, w, gauss_newton=True)
        per = []
        for _ in range(args.steps):
            _, t = _timed(lambda: obj.hessian_vector(ev, w, gauss_newton=True))
            per.append(t)
    wall = time.perf_counter() - t_all0
    total = float(np.sum(per))
    value = args.steps / total
    desc = (f"whole {args.objective} GN HVPs of the oracle port at {args.size}^3/K={args.band}/"
            f"Nt={args.nt}, pad {pad[0]}, scipy.fft on {cores} threads; {args.steps} timed HVPs")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (band_image pair + smooth v, w; SURVEY §8(d) recipe, seed 0)",
            "impl": "reference",
            "config": {**workload(args), "pad": list(pad), "parallelism": f"host CPU, {cores} threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_step_s": [round(t, 3) for t in per], "setup_gradient_s": round(t_grad, 3),
            "warmup_hvps": min(args.warmup, 1), "wall_s": round(wall, 2)}
    print(json.dumps(line))


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        sys.exit(spawn_ranks(args.gpus))
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}; "
                         "launch with --gpus equal to the number of ranks")
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup("gloo" if args.impl == "selftest" else "nccl")
    try:
        if args.impl == "selftest":
            run_selftest(args, rank, world)
        elif args.batch:
            run_batch(args, rank, world, local)
        else:
            run_b200(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
