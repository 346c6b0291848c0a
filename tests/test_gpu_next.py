"""GPU parity of the scope table's NEXT rows through the C ABI:

* f3 -- per-subset -2 log-likelihood (Eq.2) from the same factorization as the CV
  loss (pgpcv_evaluate), against oracle.neg2loglik_all; bar 1e-9 relative (the loss bar).
* f1 -- the grid-search consumer (pgpcv_select: argmin, global/local RMSPE, local winners,
  P:125), exactly equal to oracle.select on the same per-subset losses; and
  test-set prediction with the global and the local choices (pgpcv_predict)
  against oracle.predict: per-subset SSPE within 1e-9 relative, every prediction within
  1e-9 x rms(y) absolute (two FP64 solvers agree to ~kappa*eps in yhat, R18).
"""
import math
import os

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

RTOL = 1e-9
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


_wl = {}


def wl(name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _wl:
        _wl[key] = workloads.make(name, device="cuda", **kw)
    return _wl[key]


def _close(g, o, rtol=RTOL):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    bad = ~(np.abs(g - o) <= rtol * np.abs(o))
    assert not bad.any(), f"{bad.sum()} beyond {rtol}: gpu {g[bad][:4]} oracle {o[bad][:4]}"


def _part(ctx, w):
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    return oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)


# ------------------------------------------------------------------ f3

def test_nll_c2_full_grid_and_loss_unchanged(ctx):
    """All 100 subsets x 75 configs of c2: -2 log L per subset and the composite sum; the
    CV loss computed in the same launch is bit-identical to a loss-only launch."""
    w = wl("c2")
    part = _part(ctx, w)
    both = ctx.evaluate(w.params, nll=True, subset_nll=True)
    only = ctx.cv_loss(w.params)
    assert np.array_equal(both.subset_loss, only.subset_loss)
    assert np.array_equal(both.loss, only.loss)
    tot, per = oracle.neg2loglik_all(w.x, w.y, w.value, part, w.params, threads=THREADS)
    _close(both.subset_nll, per)
    _close(both.nll, tot)
    nll_only = ctx.evaluate(w.params, loss=False, subset_loss=False, nll=True, subset_nll=True)
    assert np.array_equal(nll_only.subset_nll, both.subset_nll)


def test_nll_c4_includes_empty_validation_subsets(ctx):
    """c4 at full size (uneven k, 10 subsets without validation data): the likelihood covers
    every subset with training data; sampled subsets (incl. all empty-validation ones)
    against the oracle."""
    w = wl("c4")
    part = _part(ctx, w)
    p = w.params[[5, 58]]
    res = ctx.evaluate(p, loss=False, subset_loss=False, nll=True, subset_nll=True)
    k, m = part.k(), part.m()
    empty = np.nonzero(m == 0)[0]
    rng = np.random.default_rng(9)
    sub = np.unique(np.concatenate([empty[:12], [int(np.argmax(k)), int(np.argmin(k))],
                                    rng.choice(k.size, 24, replace=False)]))
    _, per = oracle.neg2loglik_all(w.x, w.y, w.value, part, p, subsets=sub, threads=THREADS)
    _close(res.subset_nll[sub], per[sub])
    assert np.all(res.subset_nll[k == 0] == 0.0)
    assert res.nll == pytest.approx(res.subset_nll.sum(axis=0), rel=1e-12)


def test_nll_ragged_and_one_subset(ctx):
    """One tile (the full-data likelihood) at ragged k around the 64/128 blocking."""
    for k in (1, 63, 65, 129, 300):
        x, y, v, role = workloads.random_points(500 + k, k + 3, frac_val=0.0)
        role[:3] = 1
        ctx.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
        p = np.array([[0.2, 1.3, 0.1]])
        res = ctx.evaluate(p, loss=False, subset_loss=False, nll=True, subset_nll=True)
        t = role == 0
        ref = oracle.neg2loglik(x[t], y[t], v[t], 0.2, 1.3, 0.1)
        _close(res.nll, [ref])


# ------------------------------------------------------------------ f1

def test_select_equals_oracle_on_gpu_losses(ctx):
    """pgpcv_select on the c2 grid: exactly the oracle's consumer applied to the same
    per-subset losses (argmin, RMSPE, local winners, win counts)."""
    w = wl("c2")
    part = _part(ctx, w)
    res = ctx.cv_loss(w.params)
    sel = ctx.select()
    best, rmspe, lb, lr, wins = oracle.select(res.loss, res.subset_loss, part.m())
    assert sel.best == best
    np.testing.assert_array_equal(sel.rmspe, rmspe)
    np.testing.assert_array_equal(sel.local_best, lb)
    np.testing.assert_array_equal(sel.local_rmspe, lr)
    np.testing.assert_array_equal(sel.wins, wins)
    assert sel.wins.sum() == (part.m() > 0).sum()


def test_select_needs_an_evaluation(ctx, pg):
    w = wl("c1")
    _part(ctx, w)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx._last_C = 1
        ctx.select()
    assert ei.value.code == pg.ESTATE


def test_predict_validation_targets_reproduce_cv_loss(ctx, pg):
    """pgpcv_predict on the validation points with one config is pgpcv_cv_loss (same
    kernel, bit-identical), and per-subset configs pick the matching columns."""
    w = wl("c2")
    _part(ctx, w)
    p = w.params[[7, 30, 61]]
    cv = ctx.cv_loss(p)
    pr = ctx.predict(p[1:2], target_role=pg.ROLE_VALIDATION)
    assert np.array_equal(pr.subset_sspe, cv.subset_loss[:, 1]) and pr.sspe == cv.loss[1]
    cfg = np.arange(100, dtype=np.int32) % 3
    pr3 = ctx.predict(p, subset_config=cfg, target_role=pg.ROLE_VALIDATION)
    assert np.array_equal(pr3.subset_sspe, cv.subset_loss[np.arange(100), cfg])


def test_test_set_prediction_global_and_local(ctx, pg):
    """The paper's P:466-468 step on c4 (n = 200,000 clustered, 80/10/10): choose
    zeta_hat_CV and the per-subset local bests on the grid, predict the test points with
    both, compare yhat and SSPE with the oracle (sampled subsets for the local choice)."""
    w = wl("c4", n=200_000)
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    toff, tidx = ctx.partition_export_test()
    tpart = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta, core_role=2)
    assert np.array_equal(toff, tpart.val_off) and np.array_equal(tidx, tpart.val_idx)
    grid = w.params[::8]
    ctx.cv_loss(grid)
    sel = ctx.select()
    glob = ctx.predict(grid[sel.best:sel.best + 1])
    o_tot, o_sub, o_yhat = oracle.predict(w.x, w.y, w.value, tpart, grid[sel.best:sel.best + 1],
                                          threads=THREADS)
    scale = float(np.sqrt(np.mean(w.value ** 2)))
    assert np.all(np.abs(glob.yhat - o_yhat) <= RTOL * scale)
    _close(glob.subset_sspe, o_sub)
    _close([glob.sspe], [o_tot])
    cfg = np.where(sel.local_best >= 0, sel.local_best, sel.best).astype(np.int32)
    loc = ctx.predict(grid, subset_config=cfg)
    _, o_sub2, o_yhat2 = oracle.predict(w.x, w.y, w.value, tpart, grid, subset_config=cfg, threads=THREADS)
    assert np.all(np.abs(loc.yhat - o_yhat2) <= RTOL * scale)
    _close(loc.subset_sspe, o_sub2)
    n_test = int((w.role == 2).sum())
    r_glob, r_loc = math.sqrt(glob.sspe / n_test), math.sqrt(loc.sspe / n_test)
    assert 0.1 < r_glob < 1.0 and 0.1 < r_loc < 1.0


def test_predict_rejects_bad_config_index(ctx, pg):
    w = wl("c1")
    _part(ctx, w)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.predict(w.params, subset_config=np.array([0, 1, 0, 0], np.int32))
    assert ei.value.code == pg.EINVAL
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.predict(w.params, target_role=0)
    assert ei.value.code == pg.EINVAL
