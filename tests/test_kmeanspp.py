"""init_kmeanspp (core.py:192-217 of the reference): the drop-in's seeding
reproduces the reference's picks exactly -- the AC01 golden cells were seeded
by the reference's own make_init (tests/test_acceptance.py:108-109) -- on the
host, and with the D^2 updates on the GPU (lk_d2_update)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden

AC01 = golden_names("ac01_")


def _init(data, k, seed):
    from paper_2010_06654_b200.core import RunContext, make_init
    return make_init(RunContext(seed=seed), data, k)


@pytest.mark.parametrize("name", AC01)
def test_host_kmeanspp_matches_reference_golden(name, monkeypatch):
    from paper_2010_06654_b200 import core
    monkeypatch.setattr(core, "KMEANSPP_DEVICE_MIN", 1 << 62)  # host path
    g = load_golden(name)
    seed = int(name.rsplit("_s", 1)[1])
    init = _init(g["data"], int(g["k"]), seed)
    assert np.array_equal(init, g["init"]), name


@pytest.mark.gpu
@pytest.mark.parametrize("name", AC01)
def test_device_kmeanspp_matches_reference_golden(name, monkeypatch):
    from paper_2010_06654_b200 import core
    monkeypatch.setattr(core, "KMEANSPP_DEVICE_MIN", 0)  # D^2 updates on the GPU
    g = load_golden(name)
    seed = int(name.rsplit("_s", 1)[1])
    init = _init(g["data"], int(g["k"]), seed)
    assert np.array_equal(init, g["init"]), name


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 16, 130])
def test_device_kmeanspp_matches_host(d, monkeypatch):
    """Larger cases (pairwise leaves > 128 at d=130): device == host picks."""
    from paper_2010_06654_b200 import core
    rng = np.random.default_rng(d)
    x = (rng.normal(size=(20000, d)) * 3 + rng.integers(0, 5, size=(20000, 1))).astype(np.float32)
    monkeypatch.setattr(core, "KMEANSPP_DEVICE_MIN", 0)
    dev = _init(x, 64, 9)
    monkeypatch.setattr(core, "KMEANSPP_DEVICE_MIN", 1 << 62)
    host = _init(x, 64, 9)
    assert np.array_equal(dev, host)
