"""Harness: INI run configuration, deterministic CSV /
text reports, and the CLI (register / synthesize / check-derivatives /
report).  CPU tests cover parsing and reports; GPU tests run the CLI end to
end (reference runconfig.py:78-100, report.py:49-58)."""

import os
import subprocess
import sys

import pytest

from paper_1807_05117_b200.harness import report as R
from paper_1807_05117_b200.harness import runconfig as RC
from paper_1807_05117_b200.solver import IterationRecord

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = """
[domain]
shape = 32 32
bandwidth = 8   ; one value -> every axis
alpha = 0.01
[problem]
objective = deformation
sigma2 = 0.03
auto_refine = off
[optimizer]
max_outer = 12
[run]
source = source.vol
target = target.vol
output_dir = out
"""


def test_config_parses_and_fills_defaults():
    c = RC.loads_config(CFG)
    assert c.objective == "deformation" and c.problem.sigma2 == 0.03 and c.problem.auto_refine is False
    assert c.solver.max_outer == 12 and c.solver.pcg_max_iter == 10  # default
    dom = c.domain
    assert dom.shape == (32, 32) and dom.bandwidth == (8, 8) and dom.alpha == 0.01
    s = RC.effective_settings(c, dom)
    assert s["optimizer.pcg_tol"] == 0.1 and s["problem.quadrature"] == "trapezoid"
    assert s["domain.bandwidth"] == "8 8" and s["run.seed"] == 0


@pytest.mark.parametrize("bad,msg", [
    ("[problem]\nsigma = 1\n", "unknown keys"),
    ("[domain]\nshape = 32 32\n", "without bandwidth"),
    ("[problem]\nobjective = elastic\n", "unknown objective"),
    ("[problem]\nmode = piecewise\n", "unknown mode"),
    ("[optimizer]\nmax_outer = ten\n", "invalid value"),
    ("[problem]\nauto_refine = maybe\n", "invalid value"),
    ("[problem]\nsigma2 = -1\n", "sigma2"),
    ("[domain]\nshape = 32 32\nbandwidth = 40\n", "bandwidth"),
    ("[extras]\nx = 1\n", "unknown sections"),
])
def test_config_errors_fail_loudly(bad, msg):
    with pytest.raises(RC.ConfigError, match=msg):
        RC.loads_config(bad)


def test_domain_for_mismatched_grid():
    c = RC.loads_config(CFG)
    with pytest.raises(RC.ConfigError, match="does not match"):
        c.domain_for((64, 64))


def _records():
    return [IterationRecord(0, 1.5, 100.0, 1.0, 0, 0.0, False, 0.1),
            IterationRecord(1, 0.75, 40.0, 0.2, 3, 1.0, False, 0.2),
            IterationRecord(2, 0.5, 20.0, 0.05, 4, 0.5, True, 0.3)]


def test_csv_is_deterministic_and_excludes_wall_time():
    a, b = R.records_to_csv(_records()), R.records_to_csv(_records())
    assert a == b
    lines = a.splitlines()
    assert lines[0] == ",".join(R.CSV_COLUMNS)
    assert lines[3] == "2,0.5,20.0,0.05,4,0.5,1"
    assert "0.3" not in lines[3]


def test_report_text_and_json_round_trip(tmp_path):
    rep = R.RegistrationReport(records=_records(), status="converged", final_mse_rel=20.0, final_grad_rel=0.05,
                               jacobian_min=0.9, jacobian_max=1.1, settings={"a.b": 1}, dsc={1: 0.8},
                               total_time=1.25, negative_curvature_events=1, total_pcg_iters=7)
    t = R.report_text(rep)
    assert "status: converged" in t and "accepted outer iterations: 2" in t and "label 1: 0.8000" in t
    assert "a.b = 1" in t and "total wall time [s]: 1.25" in t
    R.write_report(rep, tmp_path / "report.txt")
    again = R.RegistrationReport.from_json((tmp_path / "report.json").read_text())
    assert R.report_text(again) == t
    r = subprocess.run([sys.executable, "-m", "paper_1807_05117_b200.harness.cli", "report", str(tmp_path), "--csv"],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.startswith(t) and R.records_to_csv(_records()) in r.stdout


@pytest.mark.parametrize("kw,msg", [(dict(final_mse_rel=-1.0), "negative"), (dict(jacobian_min=2.0), "order"),
                                    (dict(dsc={1: 1.5}), "DSC")])
def test_report_invariants(kw, msg):
    base = dict(records=[], status="converged", final_mse_rel=1.0, final_grad_rel=0.1, jacobian_min=0.9,
                jacobian_max=1.1)
    base.update(kw)
    with pytest.raises(ValueError, match=msg):
        R.RegistrationReport(**base)


def test_cli_config_error_exit_code(tmp_path):
    p = tmp_path / "bad.ini"
    p.write_text("[problem]\nsigmaa = 1\n")
    r = subprocess.run([sys.executable, "-m", "paper_1807_05117_b200.harness.cli", "register", str(p)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 2 and "unknown keys" in r.stderr


torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_cli_register_end_to_end_deterministic(tmp_path):
    cli = [sys.executable, "-m", "paper_1807_05117_b200.harness.cli"]
    r = subprocess.run(cli + ["synthesize", "translation", "--size", "32", "--ndim", "2", "--shift", "0.06",
                              "--out", str(tmp_path)], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    (tmp_path / "run.ini").write_text(CFG.replace("auto_refine = off", "auto_refine = on")
                                      .replace("objective = deformation", "objective = state"))
    outs = []
    for _ in range(2):
        r = subprocess.run(cli + ["register", str(tmp_path / "run.ini")], capture_output=True, text=True, cwd=ROOT)
        assert r.returncode in (0, 5), r.stderr
        outs.append((tmp_path / "out" / "iterations.csv").read_bytes())
    assert outs[0] == outs[1]  # identical config + seed -> byte-identical CSV
    for f in ("warped.vol", "displacement.vol", "difference.vol", "report.txt", "report.json"):
        assert (tmp_path / "out" / f).exists()
    text = (tmp_path / "out" / "report.txt").read_text()
    assert "problem.objective = state" in text and "optimizer.max_outer = 12" in text
    rep = R.RegistrationReport.from_json((tmp_path / "out" / "report.json").read_text())
    assert rep.final_mse_rel < 100.0 and rep.jacobian_min > 0
    # auto_refine off and a step count the CFL condition rejects: category exit code 4
    (tmp_path / "cfl.ini").write_text(CFG.replace("sigma2 = 0.03", "sigma2 = 0.03\nn_time_steps = 1"))
    r = subprocess.run(cli + ["register", str(tmp_path / "cfl.ini")], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 4 and "CFL" in r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_cli_check_derivatives_passes():
    r = subprocess.run([sys.executable, "-m", "paper_1807_05117_b200.harness.cli", "check-derivatives",
                        "--size", "32", "--ndim", "2"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok") == 6
