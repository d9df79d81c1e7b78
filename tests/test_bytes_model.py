"""The SURVEY §8(d) byte model (tools/bytes_model.py) reproduces the survey's
published figures at the reference pad, and bench.py reports the same model."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bytes_model as M  # noqa: E402


def test_reference_pad():
    assert M.reference_pad(32) == 132
    assert M.reference_pad(16) == 66


@pytest.mark.parametrize("call,gb", [("state_gn_hvp", 43.5), ("deformation_gn_hvp", 66.9),
                                     ("state_gradient", 55.9), ("deformation_gradient", 48.6),
                                     ("energy", 20.3)])
def test_survey_figures_at_128(call, gb):
    # 128^3 / K=32 / Nt=10, P=132, fp64
    assert M.model_bytes(call, 3, 128, 32, 132, 10) / 1e9 == pytest.approx(gb, abs=0.05)


def test_bench_uses_the_same_model():
    import types

    import bench
    args = types.SimpleNamespace(dtype="float64", band=32, size=128, nt=10, objective="deformation")
    dom = types.SimpleNamespace(pad=(100, 100, 100))
    assert bench.survey_model_bytes(args, dom) == M.model_bytes("deformation_gn_hvp", 3, 128, 32, 100, 10)
