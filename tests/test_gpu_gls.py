"""GPU parity of row f4 (GLS mean estimation, Eq. GLS; reading R23) through the
C ABI against oracle.gls: the summed normal equations X^T M^-1 X and X^T M^-1 y within 1e-9
relative (1e-9 of the largest entry for entries near 0), beta within 1e-8 of max|beta|
(the p x p solve adds the conditioning of the normal equations)."""
import os

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def pg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_13132_b200 as pg
    return pg


@pytest.fixture(scope="module")
def ctx(pg):
    c = pg.Context(0)
    yield c
    c.close()


def _cov(w):
    return np.stack([np.ones(w.n), w.x / w.domain[1], w.y / w.domain[3], (w.x * w.y) / (w.domain[1] * w.domain[3])], 1)


def _cmp(g, o, rtol=1e-9):
    g, o = np.asarray(g), np.asarray(o)
    scale = np.max(np.abs(o))
    assert np.all(np.abs(g - o) <= rtol * np.maximum(np.abs(o), scale * 1e-3 if o.ndim else np.abs(o))), (g, o)


def test_gls_grid_c2(ctx):
    w = workloads.make("c2")
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    X = _cov(w)
    prm = w.params[37]
    beta, A, b = ctx.gls(X, prm)
    ex, ey = oracle.edges(0.0, 1.0, w.kx), oracle.edges(0.0, 1.0, w.ky)
    rects = np.array([[ex[i], ex[i + 1], ey[j], ey[j + 1]] for j in range(w.ky) for i in range(w.kx)])
    part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    ob, oA, obb = oracle.gls(w.x, w.y, w.value, X, part, rects, w.domain, prm, threads=THREADS)
    _cmp(A, oA)
    _cmp(b, obb)
    assert np.all(np.abs(beta - ob) <= 1e-8 * np.max(np.abs(ob)))


def test_gls_bisect_clustered(ctx):
    w = workloads.make("c4", n=200_000)
    ctx.partition_bisect(w.x, w.y, w.value, w.role, w.domain, 7, 0.15, 300, 5)
    X = _cov(w)[:, :3]
    prm = w.params[21]
    beta, A, b = ctx.gls(X, prm)
    _, rects = oracle.bisect(w.x, w.y, w.role, w.domain, 7, 0.15)
    part = oracle.cap_shells(oracle.partition_rects(w.x, w.y, w.role, w.domain, rects, 0.15), w.x, w.y,
                             w.domain, 300, 5)
    ob, oA, obb = oracle.gls(w.x, w.y, w.value, X, part, rects, w.domain, prm, threads=THREADS)
    _cmp(A, oA)
    _cmp(b, obb)
    assert np.all(np.abs(beta - ob) <= 1e-8 * np.max(np.abs(ob)))


def test_gls_exact_linear_mean_on_gpu(ctx):
    """y = X beta0: beta_hat = beta0 for any division (R23), here tiles with shells."""
    w = workloads.make("c2")
    X = _cov(w)
    beta0 = np.array([0.3, -1.0, 2.5, 0.75])
    ctx.partition(w.x, w.y, X @ beta0, w.role, w.domain, w.kx, w.ky, w.delta)
    beta, _, _ = ctx.gls(X, w.params[10])
    np.testing.assert_allclose(beta, beta0, rtol=1e-9)


def test_gls_single_subset_ragged(ctx):
    for k in (1, 63, 130):
        x, y, v, role = workloads.random_points(900 + k, k + 2, frac_val=0.0)
        role[:2] = 1
        ctx.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
        X = np.stack([np.ones(x.size), x], 1)[:, : (1 if k == 1 else 2)]
        beta, A, b = ctx.gls(X, (0.2, 1.0, 0.1))
        part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
        ob, oA, obb = oracle.gls(x, y, v, X, part, np.array([[0, 1, 0, 1.0]]), (0, 1, 0, 1), (0.2, 1.0, 0.1))
        _cmp(A, oA)
        _cmp(b, obb)


def test_gls_rejects_bad_args(ctx, pg):
    x, y, v, role = workloads.random_points(1, 50)
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.gls(np.ones((50, 9)), (0.2, 1.0, 0.1))
    assert ei.value.code == pg.EINVAL
