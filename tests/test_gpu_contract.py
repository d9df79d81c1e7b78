"""Boundary contract of the B200 path.

* Concurrency: the reference allows ``hessian_vector`` to be called
  concurrently from several threads against one evaluation
  (``objectives/base.py:69-72``).  Two threads, each on its own torch stream,
  must get results bit-identical to serial calls (the kernels are
  deterministic and every (thread, stream) pair owns its scratch).
* NaN propagation: ``max_abs`` follows ``np.max`` (a NaN anywhere gives NaN),
  so a NaN gradient cannot read as "converged" and a NaN velocity cannot pass
  the CFL check with speed 0 (reference ``solver.py:74-85``,
  ``transport.py:165-185``).
"""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import blreg_oracle as O  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import solver, spectral, transport  # noqa: E402


def _problem(kind, n=32, k=8, nt=6, dtype="float64"):
    odom = O.Dom((n,) * 3, (k,) * 3, alpha=0.02, order=2)
    rng = np.random.default_rng(3)
    I0, I1 = O.band_image(odom, rng), O.band_image(odom, rng)
    v = O.smooth_vector_block(odom, rng, 0.5 / n, decay=2.0)[None]
    ws = [O.smooth_vector_block(odom, rng, 0.5 / n, decay=2.0)[None] for _ in range(3)]
    dom = B.Domain((n,) * 3, (k,) * 3, alpha=0.02, order=2, dtype=dtype)
    cls = B.StateObjective if kind == "state" else B.DeformationObjective
    obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=nt))
    return dom, obj, B.TimeFlow(dom, v, nt, True), [B.TimeFlow(dom, w, nt, True) for w in ws]


@pytest.mark.parametrize("kind", ["def", "state"])
@pytest.mark.parametrize("gn", [True, False])
def test_concurrent_hvp_two_threads_two_streams(kind, gn):
    dom, obj, v, ws = _problem(kind)
    ev = obj.gradient(v)
    torch.cuda.synchronize()
    # serial results first, on the default stream (lazy caches built here
    # for half the cases, inside the threads for the other half)
    if gn:
        serial = [ev.hessian_vector(w, gauss_newton=gn).values.clone() for w in ws]
        torch.cuda.synchronize()
    results, errors = {}, []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(2):
                    for i in (range(3) if tid == 0 else reversed(range(3))):
                        results[(tid, rep, i)] = ev.hessian_vector(ws[i], gauss_newton=gn).values
            s.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    if not gn:
        serial = [ev.hessian_vector(w, gauss_newton=gn).values.clone() for w in ws]
        torch.cuda.synchronize()
    for (tid, rep, i), val in results.items():
        assert torch.equal(val, serial[i]), (tid, rep, i)
    assert dom.ctx().n_handles >= 3  # default stream + one per worker thread


def test_nan_max_abs_propagates():
    dom = B.Domain((16,) * 3, (4,) * 3)
    c = torch.zeros((3,) + dom.block_shape, dtype=torch.complex128, device="cuda")
    c[1, 1, 0, 0] = 0.5
    c[1, -1, 0, 0] = 0.5
    assert spectral.max_abs(dom, c) == pytest.approx(1.0, rel=1e-14)
    c[2, 0, 0, 0] = float("nan")
    assert np.isnan(spectral.max_abs(dom, c))
    flow = B.TimeFlow(dom, c[None], 4, True)
    assert np.isnan(transport.flow_max_abs(flow))
    # a NaN gradient must not read as converged (reference returns NaN)
    assert np.isnan(solver.relative_gradient_norm(flow, None, initial_norm=1.0))


def test_nan_velocity_fails_cfl():
    dom = B.Domain((16,) * 3, (4,) * 3)
    c = torch.zeros((1, 3) + dom.block_shape, dtype=torch.complex128, device="cuda")
    c[0, 0, 0, 0, 0] = float("nan")
    flow = B.TimeFlow(dom, c, 4, True)
    assert np.isnan(flow.max_speed())
    # reference transport.py:184: int(np.ceil(nan)) raises, as here
    with pytest.raises(ValueError):
        transport.check_cfl(flow)


def test_batch_in_flight_pairs_match_serial():
    """Several registrations in flight on one GPU (threads + streams) give the
    same per-pair results and atlas as one at a time (bit-identical: every
    (thread, stream) owns its context, and the atlas is summed in pair order)."""
    import bench
    from paper_1807_05117_b200 import batch as Bt

    dom = B.Domain((32,) * 3, (8,) * 3, alpha=0.01)
    pairs = [bench.blob_pair(dom, seed=s) for s in range(1, 6)]
    prob = B.ProblemConfig(sigma2=0.03, n_time_steps=6)
    cfg = B.SolverConfig(max_outer=6)
    r1 = Bt.register_batch(pairs, domain=dom, problem=prob, solver_cfg=cfg, in_flight=1)
    r3 = Bt.register_batch(pairs, domain=dom, problem=prob, solver_cfg=cfg, in_flight=3)
    keep = [i for i, n in enumerate(Bt.STATS) if n != "wall_s"]
    assert np.array_equal(r1.stats[:, keep], r3.stats[:, keep])
    assert torch.equal(r1.atlas, r3.atlas)
