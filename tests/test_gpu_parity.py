"""GPU parity: the CUDA path (through the C ABI, libpgpcv.so) against the CPU oracle on
the same seeded inputs.

Bar (BASELINE.json north_star): subset membership bit-exact; every per-subset and global
CV loss within |g - o| <= 1e-9 |o| (FP64); exact zeros where the method gives them
(R10); bit-exact power-of-two invariants on the GPU itself.
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


_wl_cache = {}


def wl(name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _wl_cache:
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        _wl_cache[key] = workloads.make(name, device=dev, **kw)
    return _wl_cache[key]


def _assert_partition_equal(ctx, w):
    info = ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    toff, tidx, voff, vidx = ctx.partition_export()
    ref = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    assert np.array_equal(toff, ref.train_off)
    assert np.array_equal(voff, ref.val_off)
    assert np.array_equal(tidx, ref.train_idx)
    assert np.array_equal(vidx, ref.val_idx)
    assert info["n_train"] == int((w.role == 0).sum()) and info["n_val"] == int((w.role == 1).sum())
    return ref


def _assert_close(g, o, rtol=RTOL):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    bad = ~(np.abs(g - o) <= rtol * np.abs(o))
    if bad.any():
        i = np.argwhere(bad)[:5]
        raise AssertionError(f"{bad.sum()} entries beyond rtol {rtol}: idx {i.tolist()} "
                             f"gpu {g[bad][:5]} oracle {o[bad][:5]}")


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_partition_bit_exact(ctx, name):
    """Alg.1 lines 2-3: GPU counting-sort membership == brute-force oracle."""
    _assert_partition_equal(ctx, wl(name))


def test_cv_loss_c1_full(ctx):
    w = wl("c1")
    ref_part = _assert_partition_equal(ctx, w)
    res = ctx.cv_loss(w.params)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, w.params, threads=THREADS)
    _assert_close(res.subset_loss, ref.subset_loss)
    _assert_close(res.loss, ref.loss)
    assert res.status.tolist() == [-1]


def test_cv_loss_c2_full_grid(ctx):
    """All 100 subsets x 75 configs of c2 (the paper's 20,000-point size)."""
    w = wl("c2")
    ref_part = _assert_partition_equal(ctx, w)
    res = ctx.cv_loss(w.params)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, w.params, threads=THREADS)
    _assert_close(res.subset_loss, ref.subset_loss)
    _assert_close(res.loss, ref.loss)


def test_repeated_runs_bit_identical_and_exact(ctx):
    """Race regression: the full c2 grid three times -- every run within 1e-9 of the oracle
    and bit-identical to the others (dynamic scheduling must not change any value).  A
    missing cross-proxy fence in the operand pipeline once corrupted ~1e-3 of the items."""
    w = wl("c2")
    ref_part = _assert_partition_equal(ctx, w)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, w.params, threads=THREADS)
    first = None
    for _ in range(3):
        res = ctx.cv_loss(w.params)
        _assert_close(res.subset_loss, ref.subset_loss)
        if first is None:
            first = res.subset_loss.copy()
        assert np.array_equal(res.subset_loss, first)


def test_cv_loss_c3_configs(ctx):
    """All 1,600 subsets of c3 at the grid corners and the truth."""
    w = wl("c3")
    ref_part = _assert_partition_equal(ctx, w)
    p = w.params[[0, 13, 26]]
    res = ctx.cv_loss(p)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, p, threads=THREADS)
    _assert_close(res.subset_loss, ref.subset_loss)
    _assert_close(res.loss, ref.loss)


def _stratified(k, m, n, seed):
    rng = np.random.default_rng(seed)
    N = k.size
    has = np.nonzero(m > 0)[0]
    pick = {int(has[np.argmin(k[has])]), int(has[np.argmax(k[has])]), 0, N - 1}
    pick |= set(rng.choice(has, size=max(0, n - len(pick)), replace=False).tolist())
    return np.array(sorted(pick))


def test_c4_sampled_parity(ctx):
    """c4 (clustered, uneven k up to ~1,800) at full size: sampled subsets x 2 configs."""
    w = wl("c4")
    ref_part = _assert_partition_equal(ctx, w)
    p = w.params[[0, 63]]
    res = ctx.cv_loss(p)
    sub = _stratified(ref_part.k(), ref_part.m(), 48, 4)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, p, subsets=sub, threads=THREADS)
    _assert_close(res.subset_loss[sub], ref.subset_loss[sub])
    # subsets without validation data contribute exactly 0 (R10)
    empty = np.nonzero(ref_part.m() == 0)[0]
    assert np.all(res.subset_loss[empty] == 0.0)
    assert res.loss == pytest.approx(res.subset_loss.sum(axis=0), rel=1e-12)


def test_c5_full_size_sampled(ctx):
    """c5 (5M points, 2,500 subsets, k ~ 4,000) in the bench's launch configuration: all
    subsets at the truth config; 16 stratified subsets checked one by one on the oracle."""
    w = wl("c5")
    ref_part = _assert_partition_equal(ctx, w)
    truth = np.array([[1.0, 1.0, 0.1]])
    res = ctx.cv_loss(truth)
    sub = _stratified(ref_part.k(), ref_part.m(), 16, 5)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, truth, subsets=sub, threads=THREADS)
    _assert_close(res.subset_loss[sub], ref.subset_loss[sub])
    # a nugget-noise floor: RMSPE slightly above sqrt(tau) = 0.316 at the truth
    rmspe = math.sqrt(res.loss[0] / ref_part.m().sum())
    assert 0.3 < rmspe < 0.5


RAGGED_K = [1, 2, 3, 5, 8, 9, 31, 32, 33, 40, 63, 64, 65, 71, 95, 96, 97, 100, 127, 128, 129,
            160, 161, 200, 255, 257, 511, 512, 513, 700]


@pytest.mark.parametrize("k", RAGGED_K)
def test_ragged_single_subset(ctx, k):
    """One tile (Eq.7 with N = 1 is Eq.4): k training points not a multiple of the 64-wide
    block or the 128-row tile, m = 7 validation points. The diagonal block's 8-column
    panels see partial (5, 9, 71: a 7-wide last block) and exact (8, 40) widths, rows
    beyond lane 32 of warp 0 (33, 40, 100) and the panels from column 32 on (40, 100, 200)."""
    m = 7
    rng = np.random.default_rng(1000 + k)
    n = k + m
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    v = rng.standard_normal(n)
    role = np.zeros(n, np.uint8)
    role[rng.permutation(n)[:m]] = 1
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
    p = np.array([[0.1, 1.0, 0.1], [0.5, 2.0, 0.01]])
    res = ctx.cv_loss(p)
    ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
    ref = oracle.cv_loss(x, y, v, ref_part, p, threads=2)
    _assert_close(res.subset_loss, ref.subset_loss)


@pytest.mark.parametrize("variant", ["large", "large_ws", "small"])
def test_ragged_both_kernel_variants(pg, variant):
    """Every ragged k on each kernel variant (the large 8-warp NB = 64 kernel, its
    warp-specialised form (PGPCV_WS=1: two consumer groups and producer warps per CTA), and
    the small 4-warp NB = 32 kernel that by default takes k <= 2048), forced with
    PGPCV_SMALL_K."""
    os.environ["PGPCV_SMALL_K"] = "100000" if variant == "small" else "0"
    os.environ["PGPCV_WS"] = "1" if variant == "large_ws" else "0"
    try:
        c = pg.Context(0)
    finally:
        del os.environ["PGPCV_SMALL_K"]
        del os.environ["PGPCV_WS"]
    with c:
        for k in RAGGED_K + [1000, 1025]:
            m = 5
            rng = np.random.default_rng(2000 + k)
            n = k + m
            x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
            v = rng.standard_normal(n)
            role = np.zeros(n, np.uint8)
            role[rng.permutation(n)[:m]] = 1
            c.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
            p = np.array([[0.2, 1.0, 0.05], [0.05, 1.0, 0.3]])
            res = c.evaluate(p, nll=True, subset_nll=True)
            ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
            ref = oracle.cv_loss(x, y, v, ref_part, p, threads=2)
            _assert_close(res.subset_loss, ref.subset_loss)
            _, nll = oracle.neg2loglik_all(x, y, v, ref_part, p, threads=2)
            _assert_close(res.subset_nll, nll)


@pytest.mark.parametrize("border", ["2", "1", "0"])
def test_bordered_prediction_shapes(pg, border):
    """The small kernel predicts by bordering the m targets below y (w_v = L^{-1} b_v,
    yhat_v = w_v . z); many targets spill over several 64-row tiles and block columns.
    Against the oracle (loss 1e-9 relative, predictions R24) with every item bordered
    (PGPCV_BORDER_PRED=2), the default rule (bordered where m <= k/20) and none (0)."""
    os.environ["PGPCV_BORDER_PRED"] = border
    try:
        c = pg.Context(0)
    finally:
        del os.environ["PGPCV_BORDER_PRED"]
    with c:
        for k, m in [(1, 1), (5, 70), (40, 130), (33, 31), (64, 64), (100, 3), (300, 65), (700, 9)]:
            rng = np.random.default_rng(3000 + k + m)
            n = k + m
            x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
            v = rng.standard_normal(n)
            role = np.zeros(n, np.uint8)
            role[rng.permutation(n)[:m]] = 1
            c.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
            p = np.array([[0.2, 1.0, 0.05], [0.07, 1.0, 0.3]])
            res = c.evaluate(p, nll=True, subset_nll=True)
            ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
            ref = oracle.cv_loss(x, y, v, ref_part, p, threads=2)
            _assert_close(res.subset_loss, ref.subset_loss)
            for ci in range(2):
                pr = c.predict(p[ci:ci + 1], target_role=pg.ROLE_VALIDATION)
                t, w_ = role == 0, role == 1
                _, yref = oracle.subset_cv(x[t], y[t], v[t], x[w_], y[w_], v[w_], *p[ci], return_yhat=True)
                assert np.max(np.abs(pr.yhat - yref)) <= 1e-9 * np.sqrt(np.mean(v ** 2)), (k, m, ci)


def test_empty_and_degenerate_subsets(ctx):
    """Tiles without validation (loss exactly 0, R10), tiles without training (yhat = 0,
    loss = sum y_V^2, R11), and an all-test tile."""
    x = np.array([0.1, 0.2, 0.3, 0.6, 0.7, 0.1, 0.9, 0.8])
    y = np.array([0.1, 0.2, 0.3, 0.1, 0.2, 0.9, 0.9, 0.6])
    v = np.array([1.0, -1.0, 0.5, 2.0, -0.5, 1.5, 0.25, 3.0])
    role = np.array([0, 0, 1, 0, 0, 1, 2, 2], np.uint8)
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 2, 2, 0.0)
    res = ctx.cv_loss([[0.3, 1.0, 0.1]])
    ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 2, 2, 0.0)
    ref = oracle.cv_loss(x, y, v, ref_part, [[0.3, 1.0, 0.1]], threads=1)
    assert res.subset_loss[1, 0] == 0.0 and res.subset_loss[3, 0] == 0.0  # no validation
    assert res.subset_loss[2, 0] == 1.5 ** 2                                # no training
    _assert_close(res.subset_loss, ref.subset_loss)


def test_non_pd_reports_status(ctx, pg):
    """Duplicate sites with zero nugget: ENUMERIC, loss NaN, status = first failing subset;
    the other config is unaffected (R12)."""
    x = np.array([0.1, 0.1, 0.2, 0.8, 0.9, 0.85])
    y = np.array([0.1, 0.1, 0.3, 0.8, 0.7, 0.9])
    v = np.array([1.0, 2.0, 0.5, 0.3, -0.2, 0.4])
    role = np.array([0, 0, 1, 0, 0, 1], np.uint8)
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 2, 1, 0.0)
    res = ctx.cv_loss([[0.2, 1.0, 0.0], [0.2, 1.0, 0.1]])
    assert res.code == pg.ENUMERIC
    assert math.isnan(res.loss[0]) and res.status[0] == 0
    assert res.status[1] == -1
    ref_part = oracle.partition(x, y, role, (0, 1, 0, 1), 2, 1, 0.0)
    ref = oracle.cv_loss(x, y, v, ref_part, [[0.2, 1.0, 0.1]], threads=1)
    _assert_close(res.loss[1:], ref.loss)


def test_invariants_bit_exact_on_gpu(ctx):
    """(2 sigma2, 2 tau) -> identical; y -> 2y -> loss x4 exactly; (x, y, D, delta, theta)
    x2 -> identical membership and loss (R8; exact power-of-two scaling)."""
    w = wl("c2")
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    p = w.params[[3, 40]]
    base = ctx.cv_loss(p).subset_loss
    p2 = p.copy()
    p2[:, 1:] *= 2
    assert np.array_equal(ctx.cv_loss(p2).subset_loss, base)
    again = ctx.cv_loss(p).subset_loss
    assert np.array_equal(again, base)  # deterministic
    one = ctx.cv_loss(p[1:]).subset_loss
    assert np.array_equal(one[:, 0], base[:, 1])  # batching over configs changes nothing
    ctx.partition(w.x, w.y, 2 * w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    assert np.array_equal(ctx.cv_loss(p).subset_loss, 4 * base)
    d2 = tuple(2 * d for d in w.domain)
    ctx.partition(2 * w.x, 2 * w.y, w.value, w.role, d2, w.kx, w.ky, 2 * w.delta)
    p3 = p.copy()
    p3[:, 0] *= 2
    assert np.array_equal(ctx.cv_loss(p3).subset_loss, base)


def test_single_subset_equals_global_and_saturated_shell(ctx):
    """Eq.7 exactness limits on the GPU: one tile, and a shell wider than D."""
    x, y, v, role = workloads.random_points(77, 1500, frac_val=0.1)
    p = [[0.15, 1.0, 0.1]]
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0)
    one = ctx.cv_loss(p).loss[0]
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 3, 3, 1.5)
    sat = ctx.cv_loss(p).loss[0]
    assert sat == pytest.approx(one, rel=1e-12)
    t, w_ = role == 0, role == 1
    ref = oracle.subset_cv(x[t], y[t], v[t], x[w_], y[w_], v[w_], 0.15, 1.0, 0.1)
    assert one == pytest.approx(ref, rel=RTOL)


def test_partition_rejects_bad_input(ctx, pg):
    x, y, v, role = workloads.random_points(3, 100)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.partition(x + 1.5, y, v, role, (0, 1, 0, 1), 2, 2, 0.1)
    assert ei.value.code == pg.EINVAL
    v2 = v.copy()
    v2[5] = np.nan
    with pytest.raises(pg.PgpcvError):
        ctx.partition(x, y, v2, role, (0, 1, 0, 1), 2, 2, 0.1)
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 2, 2, 0.1)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.cv_loss([[0.0, 1.0, 0.1]])
    assert ei.value.code == pg.EINVAL
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.partition(x, y, v, np.full(100, 2, np.uint8), (0, 1, 0, 1), 2, 2, 0.1) and None
        ctx.cv_loss([[0.1, 1.0, 0.1]])
    assert ei.value.code == pg.EEMPTY


def test_partition_device_pointers_match_host(ctx):
    import torch
    w = wl("c2")
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    a = ctx.partition_export()
    la = ctx.cv_loss(w.params[:2]).subset_loss
    t = [torch.as_tensor(arr).cuda() for arr in (w.x, w.y, w.value, w.role)]
    ctx.partition_device(*t, w.domain, w.kx, w.ky, w.delta)
    b = ctx.partition_export()
    for u, q in zip(a, b):
        assert np.array_equal(u, q)
    assert np.array_equal(ctx.cv_loss(w.params[:2]).subset_loss, la)


def test_two_ended_scheduling_is_bit_identical(pg):
    """PGPCV_SCHED=1 (the second CTA of every SM claims items from the back of the LPT list)
    changes only which CTA computes which (subset, config): every value is bit-identical."""
    w = wl("c2")
    out = []
    for sched in ("0", "1"):
        os.environ["PGPCV_SCHED"] = sched
        try:
            with pg.Context(0) as c:
                c.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
                out.append(c.evaluate(w.params, nll=True, subset_nll=True))
        finally:
            del os.environ["PGPCV_SCHED"]
    assert np.array_equal(out[0].subset_loss, out[1].subset_loss)
    assert np.array_equal(out[0].subset_nll, out[1].subset_nll)


def test_warp_specialised_large_kernel_is_bit_identical(pg):
    """The warp-specialised large kernel (PGPCV_WS=1) performs the same arithmetic in the same
    order as the two-CTA kernel; only who issues the operand copies changes.  The c2 grid on
    the large kernel (forced for every k), with a non-positive-definite config mixed in:
    every output bit-identical, including the failure status."""
    w = wl("c2")
    p = np.concatenate([w.params[:20], [[0.1, 1.0, 0.0]]])
    out = []
    for ws in ("0", "1"):
        os.environ["PGPCV_SMALL_K"] = "0"
        os.environ["PGPCV_WS"] = ws
        try:
            with pg.Context(0) as c:
                c.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
                out.append(c.evaluate(p, nll=True, subset_nll=True))
        finally:
            del os.environ["PGPCV_SMALL_K"]
            del os.environ["PGPCV_WS"]
    for a_, b_ in ((out[0].subset_loss, out[1].subset_loss), (out[0].subset_nll, out[1].subset_nll),
                   (out[0].loss, out[1].loss), (out[0].status, out[1].status)):
        assert np.array_equal(np.asarray(a_).view(np.uint8), np.asarray(b_).view(np.uint8))


def test_shard_and_evaluate_argument_rules(ctx, pg):
    """pgpcv_shard at world 1 owns every subset (same losses); bad rank/world -> EINVAL;
    shard after an evaluation of the same partition -> ESTATE; an evaluation with no
    output requested -> EINVAL (include/pgpcv.h)."""
    w = wl("c1")
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    base = ctx.cv_loss(w.params).subset_loss
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    ctx.shard(0, 1, None)
    assert np.array_equal(ctx.cv_loss(w.params).subset_loss, base)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.shard(0, 1, None)
    assert ei.value.code == pg.ESTATE
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.shard(1, 1, None)
    assert ei.value.code == pg.EINVAL
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.evaluate(w.params, loss=False, subset_loss=False, nll=False, subset_nll=False)
    assert ei.value.code == pg.EINVAL
    # world > 1 without an ncclUniqueId: EINVAL, and the ctx stays at world 1 (it owns
    # every subset and runs no collective), so the next evaluation is the world-1 one
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    with pytest.raises(pg.PgpcvError) as ei:
        ctx.shard(0, 2, None)
    assert ei.value.code == pg.EINVAL
    assert np.array_equal(ctx.cv_loss(w.params).subset_loss, base)
    assert "NCCL" in pg.nccl_library()


def test_partition_boundary_points_bit_exact(ctx, golden_dir):
    """The hand-worked golden partition (points on tile edges, on dilated bounds after
    rounding, the closed domain top, the double just below an edge) and a lattice of points
    exactly on every tile edge and every dilated bound of a 7 x 5 grid, plus duplicates:
    GPU membership == the golden lists and == the brute-force oracle bit for bit."""
    import json
    g = json.load(open(os.path.join(golden_dir, "partition_small.json")))
    pts = np.array(g["points"])
    ctx.partition(pts[:, 0], pts[:, 1], np.ones(len(pts)), pts[:, 2].astype(np.uint8), g["domain"],
                  g["kx"], g["ky"], g["delta"])
    toff, tidx, voff, vidx = ctx.partition_export()
    for s in range(4):
        assert tidx[toff[s]:toff[s + 1]].tolist() == g["train"][s]
        assert vidx[voff[s]:voff[s + 1]].tolist() == g["val"][s]
    D, kx, ky, delta = (0.0, 3.5, -1.0, 1.5), 7, 5, 0.05
    ex, ey = oracle.edges(D[0], D[1], kx), oracle.edges(D[2], D[3], ky)
    xs = np.unique(np.clip(np.concatenate([ex, ex - delta, ex + delta, np.nextafter(ex, -np.inf)]), D[0], D[1]))
    ys = np.unique(np.clip(np.concatenate([ey, ey - delta, ey + delta, np.nextafter(ey, np.inf)]), D[2], D[3]))
    X, Y = np.meshgrid(xs, ys)
    x = np.concatenate([X.ravel(), X.ravel()[:50]])  # with duplicates
    y = np.concatenate([Y.ravel(), Y.ravel()[:50]])
    role = (np.arange(x.size) % 3 == 1).astype(np.uint8) + (np.arange(x.size) % 7 == 0).astype(np.uint8)
    ctx.partition(x, y, np.ones(x.size), role, D, kx, ky, delta)
    toff, tidx, voff, vidx = ctx.partition_export()
    ref = oracle.partition(x, y, role, D, kx, ky, delta)
    assert np.array_equal(toff, ref.train_off) and np.array_equal(tidx, ref.train_idx)
    assert np.array_equal(voff, ref.val_off) and np.array_equal(vidx, ref.val_idx)
