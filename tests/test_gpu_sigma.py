"""GPU: per-range covariance reuse in the small kernel (K4s).

Sigma_theta(s) = exp(-D_s / theta) depends on a configuration only through the range
(Eq.3; lambda = nugget / sigma2 moves only the diagonal).  With reuse on,
sigma_kernel writes it once per (subset, range) of a call and every (range, lambda) item
reads it.  The entries come from the same expression as the in-kernel generation, so every
output must be BIT-IDENTICAL to the run that regenerates them (PGPCV_SIGMA_REUSE=0), and
within 1e-9 of the oracle (north_star bar).
"""
import os

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def pg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_13132_b200 as pg
    return pg


def _ctx(pg, reuse, **env):
    saved = {}
    env = dict(env, PGPCV_SIGMA_REUSE=str(reuse))
    for k_, v_ in env.items():
        saved[k_] = os.environ.get(k_)
        os.environ[k_] = v_
    try:
        return pg.Context(0)
    finally:
        for k_, v_ in saved.items():
            if v_ is None:
                del os.environ[k_]
            else:
                os.environ[k_] = v_


def _close(g, o, what):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    bad = ~(np.abs(g - o) <= RTOL * np.abs(o))
    assert not bad.any(), f"{what}: {bad.sum()} beyond 1e-9, gpu {g[bad][:3]} oracle {o[bad][:3]}"


def _bits_equal(a, b, what):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), what


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_reuse_bit_identical_on_grid_steps(pg, name):
    """The bench's step (5 consecutive grid configs: one range, 4-5 distinct lambda) and a
    whole-grid call, with and without reuse: CV losses, -2 log L and the global losses are
    bit-identical; the reuse run launches sigma_kernel (one launch more)."""
    w = workloads.make(name)
    grid = w.params
    calls = [grid[0:5], grid]
    res = {}
    for reuse in (0, 2):
        with _ctx(pg, reuse) as c:
            c.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
            out = []
            for p in calls:
                r = c.evaluate(p, nll=True, subset_nll=True)
                out.append((r, c.last_timing()["launches"]))
            res[reuse] = out
    for i in range(len(calls)):
        (r0, n0), (r2, n2) = res[0][i], res[2][i]
        _bits_equal(r0.subset_loss, r2.subset_loss, f"{name} call {i} subset_loss")
        _bits_equal(r0.subset_nll, r2.subset_nll, f"{name} call {i} subset_nll")
        _bits_equal(r0.loss, r2.loss, f"{name} call {i} loss")
        assert n2 == n0 + 1, (n0, n2)


def test_reuse_against_oracle_c2_step(pg):
    """c2, the first bench step's 5 configs with reuse forced: every per-subset loss and the
    global losses within 1e-9 of the oracle."""
    w = workloads.make("c2")
    p = w.params[0:5]
    with _ctx(pg, 2) as c:
        c.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
        r = c.evaluate(p)
    part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    ref = oracle.cv_loss(w.x, w.y, w.value, part, p, threads=os.cpu_count() or 8)
    _close(r.subset_loss, ref.subset_loss, "c2 subset loss")
    _close(r.loss, ref.loss, "c2 loss")


@pytest.mark.parametrize("border", ["2", "0"])
def test_reuse_bordered_and_ragged_shapes(pg, border):
    """Ragged (k, m) on one tile, several ranges and lambdas per range, reuse forced, with
    every item bordered (the targets' cross-covariance rows come from the block too) and
    none: losses, -2 log L and kriging predictions bit-identical to the regenerating run and
    within 1e-9 of the oracle."""
    p = np.array([[0.2, 1.0, 0.05], [0.2, 2.0, 0.05], [0.2, 1.0, 0.3],
                  [0.07, 1.0, 0.3], [0.07, 0.5, 0.01]])
    c0 = _ctx(pg, 0, PGPCV_BORDER_PRED=border)
    c2 = _ctx(pg, 2, PGPCV_BORDER_PRED=border)
    with c0, c2:
        for k, m in [(1, 1), (5, 70), (33, 31), (64, 64), (100, 3), (300, 65), (700, 9), (1025, 40)]:
            rng = np.random.default_rng(5000 + k + m)
            n = k + m
            x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
            v = rng.standard_normal(n)
            role = np.zeros(n, np.uint8)
            role[rng.permutation(n)[:m]] = 1
            out = []
            for c in (c0, c2):
                c.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
                r = c.evaluate(p, nll=True, subset_nll=True)
                pr = c.predict(p, subset_config=np.array([1], np.int32), target_role=pg.ROLE_VALIDATION)
                out.append((r, pr))
            (r0, p0), (r2, p2) = out
            _bits_equal(r0.subset_loss, r2.subset_loss, f"k={k} m={m} loss")
            _bits_equal(r0.subset_nll, r2.subset_nll, f"k={k} m={m} nll")
            _bits_equal(p0.yhat, p2.yhat, f"k={k} m={m} yhat")
            ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
            ref = oracle.cv_loss(x, y, v, ref_part, p, threads=2)
            _close(r2.subset_loss, ref.subset_loss, f"k={k} m={m}")


def test_reuse_gls_bit_identical(pg):
    """GLS (row f4) on the small kernel: the covariate rows are bordered below y, the
    covariance rows come from the block; normal equations bit-identical with and without."""
    rng = np.random.default_rng(77)
    n = 3000
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    v = rng.standard_normal(n)
    X = np.stack([np.ones(n), x, y], axis=1)
    role = np.zeros(n, np.uint8)
    p = np.array([[0.1, 1.0, 0.1]])
    outs = []
    for reuse in (0, 2):
        with _ctx(pg, reuse) as c:
            c.partition(x, y, v, role, (0, 1, 0, 1), 4, 4, 0.05)
            outs.append(c.gls(X, p[0]))
    for a_, b_ in zip(outs[0], outs[1]):
        if isinstance(a_, np.ndarray) and a_.dtype == np.float64:
            _bits_equal(a_, b_, "gls")
