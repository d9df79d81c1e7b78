"""Post-registration outputs on the host side: BLVOL files byte-identical to
the reference writer (fixture tests/golden/volio.npz) and the metrics'
definitions (metrics.py)."""

import numpy as np
import pytest

from golden_io import load
from paper_1807_05117_b200 import outputs


@pytest.mark.parametrize("tag,spacing", [("scalar", None), ("vector", (0.5, 0.25))])
def test_blvol_bytes_match_reference(tmp_path, tag, spacing):
    g = load("volio")
    path = tmp_path / f"{tag}.vol"
    outputs.write_volume(path, g[tag], spacing)
    assert path.read_bytes() == g[f"{tag}_bytes"].tobytes()
    vals, hdr = outputs.read_volume(path)
    np.testing.assert_array_equal(vals, g[tag].astype("<f4"))
    assert hdr.components == (2 if tag == "vector" else 1)


def test_blvol_rejects_corruption(tmp_path):
    path = tmp_path / "x.vol"
    outputs.write_volume(path, np.zeros((3, 4)))
    data = path.read_bytes()
    path.write_bytes(data[:-4])
    with pytest.raises(outputs.VolumeFormatError):
        outputs.read_volume(path)
    path.write_bytes(b"NOPE" + data[4:])
    with pytest.raises(outputs.VolumeFormatError):
        outputs.read_volume(path)


def test_metrics():
    s = np.zeros((4, 4))
    t = np.ones((4, 4))
    assert outputs.mse_rel(t, s, t) == 0.0
    assert outputs.mse_rel(s, s, t) == pytest.approx(100.0)
    assert outputs.mse_rel(s, t, t) == 0.0
    a = np.array([[1, 1], [0, 0]])
    b = np.array([[1, 0], [0, 0]])
    assert outputs.dice(a, b) == pytest.approx(2 / 3)
    assert outputs.dice(a * 0, b * 0) == 1.0
    assert outputs.jacobian_extrema(np.array([0.5, 2.0])) == (0.5, 2.0)
