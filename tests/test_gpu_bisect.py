"""GPU parity of row f2 (the paper's recursive shell-balanced bisection, and the
shell cap) through the C ABI against the oracle: split tree, leaf rectangles,
membership and capped shells bit-exact; CV losses on bisected subsets within 1e-9."""
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


def _close(g, o):
    g, o = np.asarray(g), np.asarray(o)
    bad = ~(np.abs(g - o) <= RTOL * np.abs(o))
    assert not bad.any(), f"{bad.sum()} beyond {RTOL}: {g[bad][:4]} vs {o[bad][:4]}"


def _check(ctx, x, y, v, role, D, depth, delta, cap=-1, seed=0):
    info = ctx.partition_bisect(x, y, v, role, D, depth, delta, cap, seed)
    _, rects = oracle.bisect(x, y, role, D, depth, delta)
    assert np.array_equal(ctx.partition_rects(), rects)
    part = oracle.partition_rects(x, y, role, D, rects, delta)
    if cap >= 0:
        part = oracle.cap_shells(part, x, y, D, cap, seed)
    toff, tidx, voff, vidx = ctx.partition_export()
    assert np.array_equal(toff, part.train_off) and np.array_equal(tidx, part.train_idx)
    assert np.array_equal(voff, part.val_off) and np.array_equal(vidx, part.val_idx)
    goff, gidx = ctx.partition_export_test()
    tpart = oracle.partition_rects(x, y, role, D, rects, delta, core_role=2)
    assert np.array_equal(goff, tpart.val_off) and np.array_equal(gidx, tpart.val_idx)
    assert info["n_subsets"] == 1 << depth and info["sum_k"] == part.train_off[-1]
    return part


@pytest.mark.parametrize("depth,delta", [(0, 0.0), (1, 0.0), (3, 0.05), (5, 0.02), (6, 0.2), (8, 0.01)])
def test_bisect_tree_and_membership_bit_exact(ctx, depth, delta):
    x, y, v, role = workloads.random_points(300 + depth, 20_000, frac_val=0.1, frac_test=0.1)
    _check(ctx, x, y, v, role, (0, 1, 0, 1), depth, delta)


def test_bisect_clustered_and_ties(ctx):
    """Clustered layout (c4 geometry) and duplicated coordinates (ties between candidate
    splits, repeated values that are not distinct candidates)."""
    w = workloads.make("c4", n=100_000)
    _check(ctx, w.x, w.y, w.value, w.role, w.domain, 7, 0.15)
    rng = np.random.default_rng(4)
    x = np.round(rng.uniform(0, 1, 5000), 2)  # many equal coordinates
    y = np.round(rng.uniform(0, 1, 5000), 2)
    v = rng.standard_normal(5000)
    role = (rng.uniform(size=5000) < 0.2).astype(np.uint8)
    _check(ctx, x, y, v, role, (0, 1, 0, 1), 4, 0.05)


@pytest.mark.parametrize("cap", [0, 40, 500])
def test_shell_cap_bit_exact(ctx, cap):
    x, y, v, role = workloads.random_points(77, 30_000, frac_val=0.1, frac_test=0.1)
    _check(ctx, x, y, v, role, (0, 1, 0, 1), 4, 0.08, cap, 2024)


def test_cv_loss_on_bisected_subsets(ctx):
    """P:394-400's strong-scaling layout (20,000 points on the unit square, 18,000/2,000)
    divided by the bisection at several depths and shell widths: every per-subset loss
    against the oracle (empty-validation subsets are exactly 0)."""
    w = workloads.make("c2")
    p = w.params[[12, 37]]
    for depth, delta in ((3, 0.05), (5, 0.1), (6, 0.2)):
        part = _check(ctx, w.x, w.y, w.value, w.role, w.domain, depth, delta)
        res = ctx.cv_loss(p)
        ref = oracle.cv_loss(w.x, w.y, w.value, part, p, threads=THREADS)
        _close(res.subset_loss, ref.subset_loss)
        _close(res.loss, ref.loss)


def test_c6_paper_division_at_full_size(ctx):
    """c6: the 5M-point c5 data divided into 512 subsets with shells capped at 2,000 (the
    paper's §4.3.3 setup): tree, membership and cap bit-exact at full size; subset sizes in
    the paper's range; sampled subsets' losses against the oracle."""
    w = workloads.make("c6", device="cuda")
    part = _check(ctx, w.x, w.y, w.value, w.role, w.domain, w.depth, w.delta, w.shell_cap, w.cap_seed)
    k = part.k()
    assert 5_000 < k.min() and k.max() < 12_000
    truth = np.array([[1.0, 1.0, 0.1]])
    res = ctx.cv_loss(truth)
    sub = np.array([int(np.argmin(k)), 300])
    ref = oracle.cv_loss(w.x, w.y, w.value, part, truth, subsets=sub, threads=THREADS)
    _close(res.subset_loss[sub], ref.subset_loss[sub])


def test_bisect_rejects_bad_args(ctx, pg):
    x, y, v, role = workloads.random_points(5, 100)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.partition_bisect(x, y, v, role, (0, 1, 0, 1), 21, 0.1)
    assert ei.value.code == pg.EINVAL
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.partition_bisect(x, y, v, role, (0, 1, 0, 1), 2, -0.1)
    assert ei.value.code == pg.EINVAL
