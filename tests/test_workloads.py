"""Seeded synthetic inputs (workloads/): shapes, role counts, grids, determinism and the
field's marginal variance sigma2 + tau (Eq.1)."""
import numpy as np
import pytest

import workloads


def test_c1_shapes_roles_grid():
    w = workloads.make("c1")
    assert w.n == 2000 and w.x.dtype == np.float64 and w.role.dtype == np.uint8
    assert (w.role == 0).sum() == 1800 and (w.role == 1).sum() == 200
    assert w.params.tolist() == [[0.1, 1.0, 0.1]]
    assert (w.kx, w.ky, w.delta) == (2, 2, 0.05)
    assert np.all((w.x >= 0) & (w.x <= 1) & (w.y >= 0) & (w.y <= 1))


def test_determinism():
    a = workloads.make("c2", n=3000)
    b = workloads.make("c2", n=3000)
    for f in ("x", "y", "value", "role"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_grids():
    assert workloads.param_grid(workloads.SPECS["c2"]).shape == (75, 3)
    assert workloads.param_grid(workloads.SPECS["c3"]).shape == (27, 3)
    assert workloads.param_grid(workloads.SPECS["c4"]).shape == (64, 3)
    g5 = workloads.param_grid(workloads.SPECS["c5"])
    assert g5.shape == (125, 3)
    assert g5[0].tolist() == [0.5, 0.5, 0.05] and g5[-1] == pytest.approx([2.0, 2.0, 0.2])
    # range outermost, nugget innermost
    assert np.all(g5[:25, 0] == 0.5) and g5[1, 2] > g5[0, 2]


def test_rff_marginal_variance():
    w = workloads.make("c2", n=20000)
    assert np.var(w.value) == pytest.approx(1.1, rel=0.15)


def test_clustered_layout_in_domain():
    w = workloads.make("c4", n=20000)
    assert np.all((w.x >= 0) & (w.x <= 20) & (w.y >= 0) & (w.y <= 20))
    assert (w.role == 2).sum() == 2000
