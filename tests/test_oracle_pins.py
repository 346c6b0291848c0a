"""Pins for the CPU oracle (oracle/): each test checks it against something other than
itself -- closed forms, values worked from the paper, library routines (numpy/scipy),
exactness limits of Eq.7 and bit-exact metamorphic invariants -- chosen so that a dropped
term, wrong sign/index or transposed operand anywhere in oracle.c fails one of them.

Citations: P:n = PAPER.md line n (Gerber & Nychka, arXiv 1912.13132); R# = DESIGN.md reading.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
import scipy.stats

import oracle
import workloads


def _cov(ax, ay, bx, by, theta):
    d = np.sqrt((ax[:, None] - bx[None, :]) ** 2 + (ay[:, None] - by[None, :]) ** 2)
    return np.exp(-d / theta)


def _cv_numpy(tx, ty, tv, vx, vy, vv, theta, lam):
    """Eq.4 with Eq.3 via LAPACK (scipy cho_factor/cho_solve): an independent library route."""
    if len(vx) == 0:
        return 0.0
    if len(tx) == 0:
        return float(np.sum(vv ** 2))
    A = _cov(tx, ty, tx, ty, theta) + lam * np.eye(len(tx))
    B = _cov(vx, vy, tx, ty, theta)
    alpha = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A, lower=True), tv)
    e = B @ alpha - vv
    return float(e @ e)


# ----------------------------------------------------------------- closed forms (Eq.3)

def test_exp_covariance_values(golden_dir):
    """c(s1,s2,theta) = exp(-||s1-s2||/theta): a k=1 system with zero nugget
    predicts c(v,t) * y_t exactly, so each golden covariance value is pinned."""
    g = json.load(open(os.path.join(golden_dir, "closed_forms.json")))
    for case in g["exp_cov"]:
        t, v = case["s1"], case["s2"]
        yv = 0.25
        loss = oracle.subset_cv([t[0]], [t[1]], [1.0], [v[0]], [v[1]], [yv], case["theta"], 1.0, 0.0)
        assert loss == pytest.approx((case["value"] - yv) ** 2, rel=1e-14)


def test_kriging_k1_closed_form(golden_dir):
    """n = 1: yhat = c(v,t) y_t / (1 + lambda), lambda = tau / sigma2."""
    c = json.load(open(os.path.join(golden_dir, "closed_forms.json")))["k1"]
    yv = -0.7
    loss = oracle.subset_cv([c["t"][0]], [c["t"][1]], [c["y_t"]], [c["v"][0]], [c["v"][1]], [yv],
                            c["range"], c["sigma2"], c["nugget"])
    assert loss == pytest.approx((c["yhat"] - yv) ** 2, rel=1e-14)


def test_kriging_k2_closed_form():
    """k = 2: with a = 1+lambda, r = c(t1,t2), c_i = c(v,t_i):
    yhat = [a(c1 y1 + c2 y2) - r(c1 y2 + c2 y1)] / (a^2 - r^2)  (2x2 inverse of Eq.3)."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        t = rng.uniform(0, 1, (2, 2))
        v = rng.uniform(0, 1, 2)
        y1, y2, yv = rng.standard_normal(3)
        theta = rng.uniform(0.1, 1.0)
        sigma2, nugget = rng.uniform(0.5, 2.0), rng.uniform(0.0, 0.5)
        a = 1.0 + nugget / sigma2
        r = math.exp(-math.dist(t[0], t[1]) / theta)
        c1 = math.exp(-math.dist(v, t[0]) / theta)
        c2 = math.exp(-math.dist(v, t[1]) / theta)
        yhat = (a * (c1 * y1 + c2 * y2) - r * (c1 * y2 + c2 * y1)) / (a * a - r * r)
        loss = oracle.subset_cv(t[:, 0], t[:, 1], [y1, y2], [v[0]], [v[1]], [yv], theta, sigma2, nugget)
        assert loss == pytest.approx((yhat - yv) ** 2, rel=1e-11)


def test_kriging_k3_adjugate_closed_form():
    """k = 3: A = [[a,p,q],[p,a,s],[q,s,a]], det = a^3 + 2pqs - a(p^2+q^2+s^2),
    adj = [[a^2-s^2, qs-ap, ps-aq], [qs-ap, a^2-q^2, pq-as], [ps-aq, pq-as, a^2-p^2]],
    yhat = c^T adj y / det; two validation points (loss sums both, Eq.4)."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        t = rng.uniform(0, 1, (3, 2))
        vs = rng.uniform(0, 1, (2, 2))
        y = rng.standard_normal(3)
        yv = rng.standard_normal(2)
        theta = rng.uniform(0.1, 1.0)
        sigma2, nugget = rng.uniform(0.5, 2.0), rng.uniform(0.01, 0.5)
        a = 1.0 + nugget / sigma2
        p = math.exp(-math.dist(t[0], t[1]) / theta)
        q = math.exp(-math.dist(t[0], t[2]) / theta)
        s = math.exp(-math.dist(t[1], t[2]) / theta)
        det = a ** 3 + 2 * p * q * s - a * (p * p + q * q + s * s)
        adj = np.array([[a * a - s * s, q * s - a * p, p * s - a * q],
                        [q * s - a * p, a * a - q * q, p * q - a * s],
                        [p * s - a * q, p * q - a * s, a * a - p * p]])
        expected = 0.0
        for i in range(2):
            cvec = np.array([math.exp(-math.dist(vs[i], t[j]) / theta) for j in range(3)])
            e = cvec @ adj @ y / det - yv[i]
            expected += e * e
        loss = oracle.subset_cv(t[:, 0], t[:, 1], y, vs[:, 0], vs[:, 1], yv, theta, sigma2, nugget)
        assert loss == pytest.approx(expected, rel=1e-10)


def test_interpolation_at_observed_sites_zero_nugget():
    """tau = 0: the kriging predictor interpolates, yhat(t_j) = y_j (Eq.3 with lambda = 0)."""
    rng = np.random.default_rng(3)
    k = 40
    t = rng.uniform(0, 1, (k, 2))
    y = rng.standard_normal(k)
    for j in (0, 17, 39):
        # validation value y_j + 1 at the site of t_j: the error is exactly 1 when yhat = y_j
        loss = oracle.subset_cv(t[:, 0], t[:, 1], y, [t[j, 0]], [t[j, 1]], [y[j] + 1.0], 0.2, 1.0, 0.0)
        assert loss == pytest.approx(1.0, abs=1e-9)


def test_far_field_predicts_zero():
    """Validation >= 50 theta from every training point: yhat = 0 (zero-mean prior, Eq.1)."""
    rng = np.random.default_rng(5)
    t = rng.uniform(0, 1, (30, 2))
    y = rng.standard_normal(30)
    theta = 0.02
    vx, vy, vv = [1.0 + 50 * theta, 3.0], [1.0 + 50 * theta, 2.0], [0.4, -1.3]
    loss = oracle.subset_cv(t[:, 0], t[:, 1], y, vx, vy, vv, theta, 1.0, 0.1)
    assert loss == pytest.approx(0.4 ** 2 + 1.3 ** 2, rel=1e-10)


def test_degenerate_subsets():
    """R10: m = 0 -> loss exactly 0; R11: k = 0 -> yhat = 0, loss = sum y_V^2."""
    assert oracle.subset_cv([0.1], [0.2], [1.0], [], [], [], 0.3, 1.0, 0.1) == 0.0
    assert oracle.subset_cv([], [], [], [0.5, 0.2], [0.5, 0.1], [2.0, -3.0], 0.3, 1.0, 0.1) == 13.0
    assert oracle.subset_cv([], [], [], [], [], [], 0.3, 1.0, 0.1) == 0.0


def test_non_positive_definite_is_reported():
    """R12: duplicate sites with zero nugget make Sigma singular -> ENUMERIC (no jitter)."""
    with pytest.raises(oracle.OracleError) as ei:
        oracle.subset_cv([0.3, 0.3], [0.4, 0.4], [1.0, 2.0], [0.5], [0.5], [0.0], 0.5, 1.0, 0.0)
    assert ei.value.code == oracle.ENUMERIC
    with pytest.raises(oracle.OracleError) as ei:
        oracle.subset_cv([0.3], [0.4], [1.0], [0.5], [0.5], [0.0], -1.0, 1.0, 0.0)
    assert ei.value.code == oracle.EINVAL


def test_matches_lapack_cho_solve():
    """Special case that reduces to a library routine: Eq.3 + Eq.4 via scipy's LAPACK
    Cholesky solve (k = 120, m = 15) agrees to 1e-12 relative."""
    rng = np.random.default_rng(19)
    for theta, sigma2, nugget in ((0.1, 1.0, 0.1), (0.5, 2.0, 0.05), (0.03, 0.7, 0.3)):
        t = rng.uniform(0, 1, (120, 2))
        v = rng.uniform(0, 1, (15, 2))
        y = rng.standard_normal(120)
        yv = rng.standard_normal(15)
        lo = oracle.subset_cv(t[:, 0], t[:, 1], y, v[:, 0], v[:, 1], yv, theta, sigma2, nugget)
        ref = _cv_numpy(t[:, 0], t[:, 1], y, v[:, 0], v[:, 1], yv, theta, nugget / sigma2)
        assert lo == pytest.approx(ref, rel=1e-12)


def test_long_double_variant_agrees():
    rng = np.random.default_rng(23)
    t = rng.uniform(0, 1, (200, 2))
    v = rng.uniform(0, 1, (20, 2))
    y = rng.standard_normal(200)
    yv = rng.standard_normal(20)
    a = oracle.subset_cv(t[:, 0], t[:, 1], y, v[:, 0], v[:, 1], yv, 0.2, 1.0, 0.1)
    b = oracle.subset_cv(t[:, 0], t[:, 1], y, v[:, 0], v[:, 1], yv, 0.2, 1.0, 0.1, long_double=True)
    assert a == pytest.approx(b, rel=1e-11)


# ------------------------------------------------------------- -2 log-likelihood (Eq.2)

def test_neg2loglik_closed_form_and_library():
    """Eq.2: n = 1 -> log 2pi + log(sigma2 + tau) + y^2/(sigma2 + tau);
    n = 50 -> -2 * scipy multivariate_normal.logpdf."""
    got = oracle.neg2loglik([0.2], [0.3], [1.5], 0.4, 2.0, 0.5)
    assert got == pytest.approx(math.log(2 * math.pi) + math.log(2.5) + 1.5 ** 2 / 2.5, rel=1e-14)
    rng = np.random.default_rng(29)
    t = rng.uniform(0, 1, (50, 2))
    y = rng.standard_normal(50)
    cov = 1.3 * _cov(t[:, 0], t[:, 1], t[:, 0], t[:, 1], 0.25) + 0.2 * np.eye(50)
    ref = -2 * scipy.stats.multivariate_normal(np.zeros(50), cov).logpdf(y)
    assert oracle.neg2loglik(t[:, 0], t[:, 1], y, 0.25, 1.3, 0.2) == pytest.approx(ref, rel=1e-11)


# --------------------------------------------------------------------- partition pins

def test_golden_partition(golden_dir):
    """Hand-worked membership (tests/golden/partition_small.json)."""
    g = json.load(open(os.path.join(golden_dir, "partition_small.json")))
    pts = np.array(g["points"])
    part = oracle.partition(pts[:, 0], pts[:, 1], pts[:, 2].astype(np.uint8), g["domain"],
                            g["kx"], g["ky"], g["delta"])
    for s in range(4):
        assert part.train(s).tolist() == g["train"][s]
        assert part.val(s).tolist() == g["val"][s]


def test_edges_rule():
    """R4: e_i = a + i*w with w = (b-a)/K, e_K = b exactly."""
    e = oracle.edges(0.0, 50.0, 50)
    assert e[-1] == 50.0 and e[0] == 0.0
    assert all(e[i] == 0.0 + i * 1.0 for i in range(50))
    e = oracle.edges(0.0, 1.0, 3)
    assert e.tolist() == [0.0, 1.0 / 3.0, 2 * (1.0 / 3.0), 1.0]


def _independent_membership(x, y, role, domain, kx, ky, delta):
    """Vectorised numpy membership by the same readings (R2-R6), as sets."""
    xmin, xmax, ymin, ymax = domain
    ex = np.array([xmin + i * ((xmax - xmin) / kx) for i in range(kx)] + [xmax])
    ey = np.array([ymin + i * ((ymax - ymin) / ky) for i in range(ky)] + [ymax])
    cx = np.clip(np.searchsorted(ex, x, side="right") - 1, 0, kx - 1)
    cy = np.clip(np.searchsorted(ey, y, side="right") - 1, 0, ky - 1)
    train, val = [], []
    for s in range(kx * ky):
        ix, iy = s % kx, s // kx
        hx = np.inf if ix == kx - 1 else ex[ix + 1] + delta
        hy = np.inf if iy == ky - 1 else ey[iy + 1] + delta
        inx = (ex[ix] - delta <= x) & (x < hx)
        iny = (ey[iy] - delta <= y) & (y < hy)
        train.append(np.nonzero((role == 0) & inx & iny)[0])
        val.append(np.nonzero((role == 1) & (cx == ix) & (cy == iy))[0])
    return train, val


@pytest.mark.parametrize("delta", [0.0, 0.02, 0.13])
def test_partition_invariants(delta):
    """Sum m = n_V without duplicates; delta = 0 training lists partition y_T; lists are
    ascending; equal to an independent vectorised membership; deterministic."""
    x, y, v, role = workloads.random_points(31, 3000, frac_val=0.1, frac_test=0.1)
    dom = (0.0, 1.0, 0.0, 1.0)
    part = oracle.partition(x, y, role, dom, 7, 5, delta)
    assert part.m().sum() == (role == 1).sum()
    assert np.array_equal(np.sort(part.val_idx), np.nonzero(role == 1)[0])
    for s in range(part.n_subsets):
        assert np.all(np.diff(part.train(s)) > 0) and np.all(np.diff(part.val(s)) > 0)
    if delta == 0.0:
        assert np.array_equal(np.sort(part.train_idx), np.nonzero(role == 0)[0])
    tr, va = _independent_membership(x, y, role, dom, 7, 5, delta)
    for s in range(part.n_subsets):
        assert np.array_equal(part.train(s), tr[s]) and np.array_equal(part.val(s), va[s])
    again = oracle.partition(x, y, role, dom, 7, 5, delta)
    assert np.array_equal(again.train_idx, part.train_idx) and np.array_equal(again.train_off, part.train_off)


def test_partition_nesting():
    """delta1 <= delta2 -> every training list for delta1 is a subset of delta2's."""
    x, y, v, role = workloads.random_points(37, 2000)
    a = oracle.partition(x, y, role, (0, 1, 0, 1), 4, 4, 0.01)
    b = oracle.partition(x, y, role, (0, 1, 0, 1), 4, 4, 0.05)
    for s in range(16):
        assert set(a.train(s).tolist()) <= set(b.train(s).tolist())
        assert np.array_equal(a.val(s), b.val(s))


def test_partition_rejects_bad_input():
    x, y, v, role = workloads.random_points(41, 50)
    with pytest.raises(oracle.OracleError):
        oracle.partition(x + 2.0, y, role, (0, 1, 0, 1), 2, 2, 0.1)  # outside D
    with pytest.raises(oracle.OracleError):
        oracle.partition(x, y, role, (0, 1, 0, 1), 0, 2, 0.1)  # kx < 1
    with pytest.raises(oracle.OracleError):
        oracle.partition(x, y, role, (0, 1, 0, 1), 2, 2, -0.1)  # delta < 0


# -------------------------------------------------------------- Eq.7 exactness limits

def _setup(seed=43, n=600):
    x, y, v, role = workloads.random_points(seed, n, frac_val=0.15)
    return x, y, v, role


def test_single_subset_reproduces_global_cv():
    """N = 1 (one tile): Eq.7 reduces to Eq.4 over all data."""
    x, y, v, role = _setup()
    part = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
    t, w = role == 0, role == 1
    for theta, s2, tau in ((0.1, 1.0, 0.1), (0.3, 2.0, 0.05)):
        rep = oracle.cv_loss(x, y, v, part, [[theta, s2, tau]], threads=1)
        ref = _cv_numpy(x[t], y[t], v[t], x[w], y[w], v[w], theta, tau / s2)
        assert rep.loss[0] == pytest.approx(ref, rel=1e-11)


def test_delta_saturating_domain_reproduces_global_cv():
    """A shell wider than D makes every y~^i_T the whole y_T: sum_i CV_i = CV."""
    x, y, v, role = _setup()
    part = oracle.partition(x, y, role, (0, 1, 0, 1), 3, 2, 1.5)
    assert all(part.k() == (role == 0).sum())
    one = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
    p = [[0.15, 1.0, 0.1]]
    a = oracle.cv_loss(x, y, v, part, p, threads=2).loss[0]
    b = oracle.cv_loss(x, y, v, one, p, threads=1).loss[0]
    assert a == pytest.approx(b, rel=1e-12)
    t, w = role == 0, role == 1
    assert a == pytest.approx(_cv_numpy(x[t], y[t], v[t], x[w], y[w], v[w], 0.15, 0.1), rel=1e-11)


def test_delta_zero_is_sum_of_independent_tile_cvs():
    """delta = 0: Eq.5 generalised -- each tile's own training predicts its own validation
    (P:144-151); checked per subset against LAPACK on independently selected tiles."""
    x, y, v, role = _setup(47, 900)
    part = oracle.partition(x, y, role, (0, 1, 0, 1), 3, 3, 0.0)
    tr, va = _independent_membership(x, y, role, (0, 1, 0, 1), 3, 3, 0.0)
    rep = oracle.cv_loss(x, y, v, part, [[0.2, 1.0, 0.1]], threads=2)
    total = 0.0
    for s in range(9):
        ref = _cv_numpy(x[tr[s]], y[tr[s]], v[tr[s]], x[va[s]], y[va[s]], v[va[s]], 0.2, 0.1)
        assert rep.subset_loss[s, 0] == pytest.approx(ref, rel=1e-11)
        total += ref
    assert rep.loss[0] == pytest.approx(total, rel=1e-12)


# ------------------------------------------------------ bit-exact metamorphic invariants

def test_power_of_two_invariants_bit_exact():
    """(2 sigma2, 2 tau) leaves lambda bit-identical (R8) -> identical loss; y -> 2y scales
    every op by 2 exactly -> loss x4 exactly; (x, y, D, delta, theta) x2 -> identical
    membership and loss (sqrt(4s) = 2 sqrt(s) under correct rounding)."""
    x, y, v, role = _setup(53, 800)
    dom = (0.0, 1.0, 0.0, 1.0)
    part = oracle.partition(x, y, role, dom, 2, 2, 0.1)
    base = oracle.cv_loss(x, y, v, part, [[0.2, 1.0, 0.1]], threads=2)
    sc = oracle.cv_loss(x, y, v, part, [[0.2, 2.0, 0.2]], threads=2)
    assert np.array_equal(base.subset_loss, sc.subset_loss)
    vv = oracle.cv_loss(x, y, 2 * v, part, [[0.2, 1.0, 0.1]], threads=2)
    assert np.array_equal(vv.subset_loss, 4 * base.subset_loss)
    part2 = oracle.partition(2 * x, 2 * y, role, (0.0, 2.0, 0.0, 2.0), 2, 2, 0.2)
    assert np.array_equal(part2.train_idx, part.train_idx) and np.array_equal(part2.val_idx, part.val_idx)
    cc = oracle.cv_loss(2 * x, 2 * y, v, part2, [[0.4, 1.0, 0.1]], threads=2)
    assert np.array_equal(cc.subset_loss, base.subset_loss)


def test_permutation_invariance():
    """Permuting the input order permutes member indices; losses agree to 1e-12."""
    x, y, v, role = _setup(59, 700)
    perm = np.random.default_rng(1).permutation(x.size)
    inv = np.argsort(perm)
    a = oracle.partition(x, y, role, (0, 1, 0, 1), 3, 2, 0.08)
    b = oracle.partition(x[perm], y[perm], role[perm], (0, 1, 0, 1), 3, 2, 0.08)
    for s in range(6):
        assert set(a.train(s).tolist()) == set(perm[b.train(s)].tolist())
        assert set(a.val(s).tolist()) == set(perm[b.val(s)].tolist())
    pa = oracle.cv_loss(x, y, v, a, [[0.1, 1.0, 0.1]], threads=2)
    pb = oracle.cv_loss(x[perm], y[perm], v[perm], b, [[0.1, 1.0, 0.1]], threads=2)
    np.testing.assert_allclose(pb.subset_loss, pa.subset_loss, rtol=1e-12)
    assert inv.size == x.size


def test_status_reports_first_failing_subset():
    """R12 / SPEC S:422: a non-PD subset makes loss[c] NaN and status[c] its id; other
    configs are unaffected."""
    x = np.array([0.1, 0.1, 0.2, 0.8, 0.9, 0.85])
    y = np.array([0.1, 0.1, 0.3, 0.8, 0.7, 0.9])
    v = np.array([1.0, 2.0, 0.5, 0.3, -0.2, 0.4])
    role = np.array([0, 0, 1, 0, 0, 1], np.uint8)
    part = oracle.partition(x, y, role, (0, 1, 0, 1), 2, 1, 0.0)
    rep = oracle.cv_loss(x, y, v, part, [[0.2, 1.0, 0.0], [0.2, 1.0, 0.1]], threads=1)
    assert math.isnan(rep.loss[0]) and rep.status[0] == 0
    assert rep.status[1] == -1 and np.isfinite(rep.loss[1])


# ----------------------------------------------------------------- row f1: grid-search consumer

def _nan(v):
    return np.array([[math.nan if e == "nan" else e for e in row] for row in v], np.float64) \
        if isinstance(v[0], list) else np.array([math.nan if e == "nan" else e for e in v], np.float64)


def test_select_hand_worked_golden(golden_dir):
    """argmin / RMSPE / local winners on a hand-worked 4 x 3 case with a
    tie, a failed (NaN) config and an empty-validation subset (tests/golden/select_small.json)."""
    g = json.load(open(os.path.join(golden_dir, "select_small.json")))
    best, rmspe, lb, lr, wins = oracle.select(_nan(g["loss"]), _nan(g["subset_loss"]), g["m"])
    assert best == g["best"]
    np.testing.assert_allclose(rmspe, _nan(g["rmspe"]), rtol=1e-15, equal_nan=True)
    assert lb.tolist() == g["local_best"]
    np.testing.assert_allclose(lr, _nan(g["local_rmspe"]), rtol=1e-15, equal_nan=True)
    assert wins.tolist() == g["wins"]


def test_test_role_partition_invariants():
    """Test points (role 2) are listed per core tile exactly once (the held-out data the
    chosen parameters predict); checked by an independent vectorised floor rule
    away from tile edges, and against the validation rule applied to relabelled roles."""
    w = workloads.make("c4", n=50_000)  # clustered layout, 80/10/10 roles (R7)
    pt = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta, core_role=2)
    pv = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta, core_role=1)
    assert np.array_equal(pt.train_off, pv.train_off) and np.array_equal(pt.train_idx, pv.train_idx)
    test = np.nonzero(w.role == 2)[0]
    assert test.size == 5_000 and pt.val_off[-1] == test.size
    assert np.array_equal(np.sort(pt.val_idx), test)
    # swapping roles 1 <-> 2 turns the test lists into validation lists
    swapped = w.role.copy()
    swapped[w.role == 1], swapped[w.role == 2] = 2, 1
    ps = oracle.partition(w.x, w.y, swapped, w.domain, w.kx, w.ky, w.delta, core_role=1)
    assert np.array_equal(ps.val_off, pt.val_off) and np.array_equal(ps.val_idx, pt.val_idx)
    # core tile by floor away from edges
    wx = (w.domain[1] - w.domain[0]) / w.kx
    ix = np.floor((w.x[test] - w.domain[0]) / wx).astype(int)
    iy = np.floor((w.y[test] - w.domain[2]) / wx).astype(int)
    s_of = np.empty(w.n, np.int64)
    for s in range(pt.n_subsets):
        s_of[pt.val(s)] = s
    safe = (np.abs((w.x[test] - w.domain[0]) / wx - np.round((w.x[test] - w.domain[0]) / wx)) > 1e-9) & \
           (np.abs((w.y[test] - w.domain[2]) / wx - np.round((w.y[test] - w.domain[2]) / wx)) > 1e-9)
    assert np.array_equal(s_of[test][safe], (iy * w.kx + ix)[safe])


def test_predict_yhat_closed_forms(golden_dir):
    """The per-point predictions the oracle returns are Eq.3's yhat: k = 1 closed form
    (golden) and k = 2 closed form, plus LAPACK cho_solve at k = 60."""
    c = json.load(open(os.path.join(golden_dir, "closed_forms.json")))["k1"]
    _, yh = oracle.subset_cv([c["t"][0]], [c["t"][1]], [c["y_t"]], [c["v"][0]], [c["v"][1]], [0.0],
                             c["range"], c["sigma2"], c["nugget"], return_yhat=True)
    assert yh[0] == pytest.approx(c["yhat"], rel=1e-14)
    t = np.array([[0.1, 0.2], [0.4, 0.3]])
    y1, y2 = 0.8, -1.3
    v = np.array([0.3, 0.1])
    theta, lam = 0.3, 0.2
    r = math.exp(-math.dist(t[0], t[1]) / theta)
    c1, c2 = (math.exp(-math.dist(v, t[i]) / theta) for i in range(2))
    a = 1 + lam
    expect = (a * (c1 * y1 + c2 * y2) - r * (c1 * y2 + c2 * y1)) / (a * a - r * r)
    _, yh = oracle.subset_cv(t[:, 0], t[:, 1], [y1, y2], [v[0]], [v[1]], [0.0], theta, 1.0, lam,
                             return_yhat=True)
    assert yh[0] == pytest.approx(expect, rel=1e-13)
    rng = np.random.default_rng(7)
    tx, ty, tv = rng.uniform(0, 1, 60), rng.uniform(0, 1, 60), rng.normal(size=60)
    vx, vy = rng.uniform(0, 1, 9), rng.uniform(0, 1, 9)
    A = _cov(tx, ty, tx, ty, 0.2) + 0.1 * np.eye(60)
    ref = _cov(vx, vy, tx, ty, 0.2) @ scipy.linalg.cho_solve(scipy.linalg.cho_factor(A, lower=True), tv)
    _, yh = oracle.subset_cv(tx, ty, tv, vx, vy, np.zeros(9), 0.2, 1.0, 0.1, return_yhat=True)
    np.testing.assert_allclose(yh, ref, rtol=1e-10, atol=1e-12)


def test_predict_with_validation_targets_is_cv_loss():
    """Predicting the validation points with one config reproduces Eq.7 per subset
    (the per-subset SSPE is the same sum), and a per-subset config picks per-subset rows."""
    w = workloads.make("c1")
    part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    p = np.array([[0.1, 1.0, 0.1], [0.2, 1.0, 0.05]])
    cv = oracle.cv_loss(w.x, w.y, w.value, part, p, threads=4)
    tot, sub, yhat = oracle.predict(w.x, w.y, w.value, part, p, threads=4)
    assert np.array_equal(sub, cv.subset_loss[:, 0]) and tot == cv.loss[0]
    cfg = np.array([1, 0, 1, 0])
    _, sub2, _ = oracle.predict(w.x, w.y, w.value, part, p, subset_config=cfg, threads=4)
    assert np.array_equal(sub2, cv.subset_loss[np.arange(4), cfg])
    e = yhat - w.value[part.val_idx]
    for s in range(4):
        sl = slice(part.val_off[s], part.val_off[s + 1])
        assert float(e[sl] @ e[sl]) == pytest.approx(sub[s], rel=1e-13)


# ----------------------------------------------------------------- row f3: -2 log-likelihood

def test_neg2loglik_composite_is_sum_of_subset_likelihoods():
    """Per-subset -2 log L (Eq.2) over y~^i_T; with one subset (kx = ky = 1) it is
    the full-data Gaussian likelihood (scipy multivariate_normal), and the composite is the
    ascending-s sum of the per-subset values."""
    rng = np.random.default_rng(3)
    n = 150
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    v = rng.normal(size=n)
    role = np.zeros(n, np.uint8)
    role[::5] = 1
    part1 = oracle.partition(x, y, role, (0, 1, 0, 1), 1, 1, 0.0)
    prm = np.array([[0.15, 1.7, 0.2]])
    tot, per = oracle.neg2loglik_all(x, y, v, part1, prm, threads=2)
    tr = role == 0
    S = 1.7 * _cov(x[tr], y[tr], x[tr], y[tr], 0.15) + 0.2 * np.eye(int(tr.sum()))
    ref = -2 * scipy.stats.multivariate_normal(mean=np.zeros(int(tr.sum())), cov=S).logpdf(v[tr])
    assert tot[0] == pytest.approx(ref, rel=1e-11)
    part4 = oracle.partition(x, y, role, (0, 1, 0, 1), 2, 2, 0.1)
    tot4, per4 = oracle.neg2loglik_all(x, y, v, part4, prm, threads=2)
    assert tot4[0] == per4[0, 0] + per4[1, 0] + per4[2, 0] + per4[3, 0]


# ----------------------------------------------------------------- row f2: bisection, shell cap

def _bisect_numpy(x, y, role, domain, depth, delta):
    """Independent brute force of the same rule (R19-R21): every candidate split of every
    node is counted with boolean masks over all points (no sorting, no binary search)."""
    xmin, xmax, ymin, ymax = domain
    counted = role <= 1
    rects = {1: (xmin, xmax, ymin, ymax)}
    splits = {}

    def dil(u, lo, hi, top):
        h = np.inf if hi == top else hi + delta
        return (lo - delta <= u) & (u < h)

    def core(u, lo, hi, top):
        return (lo <= u) & ((u < hi) | ((hi == top) & (u == top)))

    for d in range(depth):
        ax = d & 1
        for nid in range(1 << d, 1 << (d + 1)):
            x0, x1, y0, y1 = rects[nid]
            u = y if ax else x
            lo, hi, top = (y0, y1, ymax) if ax else (x0, x1, xmax)
            other = dil(x, x0, x1, xmax) if ax else dil(y, y0, y1, ymax)
            incore = counted & core(x, x0, x1, xmax) & core(y, y0, y1, ymax)
            vals = np.unique(u[incore])
            best, bc = None, 0.5 * (lo + hi)
            for j in range(vals.size - 1):
                c = 0.5 * (vals[j] + vals[j + 1])
                left = int(np.sum(counted & other & (lo - delta <= u) & (u < c + delta)))
                right = int(np.sum(counted & other & (c - delta <= u) & (u < (np.inf if hi == top else hi + delta))))
                sc = abs(left - right)
                if best is None or sc < best:
                    best, bc = sc, c
            splits[nid] = bc
            r = list(rects[nid])
            lc, rc = list(r), list(r)
            lc[2 * ax + 1] = bc
            rc[2 * ax] = bc
            rects[2 * nid], rects[2 * nid + 1] = tuple(lc), tuple(rc)
    leaves = np.array([rects[(1 << depth) + s] for s in range(1 << depth)])
    return splits, leaves


def test_bisect_spec_example_median_split():
    """q = 1, delta = 0, 10 points with distinct x: the split lies midway between the 5th
    and 6th smallest x and leaves 5 / 5 (SPEC recursive_partition example)."""
    rng = np.random.default_rng(11)
    x, y = rng.uniform(0, 1, 10), rng.uniform(0, 1, 10)
    splits, rects = oracle.bisect(x, y, np.zeros(10, np.uint8), (0, 1, 0, 1), 1, 0.0)
    xs = np.sort(x)
    assert splits[1] == 0.5 * (xs[4] + xs[5])
    assert rects.tolist() == [[0, splits[1], 0, 1], [splits[1], 1, 0, 1]]


@pytest.mark.parametrize("depth,delta", [(1, 0.0), (2, 0.1), (3, 0.05), (4, 0.02)])
def test_bisect_matches_independent_brute_force(depth, delta):
    """Splits and leaves equal (bit for bit) a boolean-mask brute force of the rule, with
    test-role points present (they never count, R20)."""
    x, y, v, role = workloads.random_points(20 + depth, 160, frac_val=0.2, frac_test=0.1)
    splits, rects = oracle.bisect(x, y, role, (0, 1, 0, 1), depth, delta)
    ref_splits, ref_rects = _bisect_numpy(x, y, role, (0, 1, 0, 1), depth, delta)
    for nid, c in ref_splits.items():
        assert splits[nid] == c, nid
    assert np.array_equal(rects, ref_rects)


def test_bisect_structure_and_balance():
    """Leaves tile D (every point in exactly one core), axes alternate (even depths split
    x), and with delta = 0 and distinct coordinates every split is balanced to one point."""
    x, y, v, role = workloads.random_points(5, 3000, frac_val=0.1, frac_test=0.1)
    depth = 5
    splits, rects = oracle.bisect(x, y, role, (0, 1, 0, 1), depth, 0.0)
    part = oracle.partition_rects(x, y, np.zeros_like(role), (0, 1, 0, 1), rects, 0.0, core_role=0)
    assert part.train_off[-1] == x.size  # delta = 0: train lists partition all points
    counted = (role <= 1)
    per_leaf = np.array([counted[part.train(s)].sum() for s in range(1 << depth)])
    # sibling leaves (and recursively every split) balance to within one point
    level = per_leaf
    while level.size > 1:
        assert np.all(np.abs(level[0::2] - level[1::2]) <= 1)
        level = level[0::2] + level[1::2]
    for s in range(1 << depth):
        x0, x1, y0, y1 = rects[s]
        assert x0 < x1 and y0 < y1
    # depth-0 split is a vertical line: the two halves of the leaf list share x ranges
    assert np.all(rects[: 1 << (depth - 1), 1] <= splits[1]) and np.all(rects[1 << (depth - 1):, 0] >= splits[1])


def test_rect_membership_equals_grid_membership():
    """The rectangle-list membership with the grid's tiles as rectangles is the grid
    partition bit for bit (two independent routines of R2-R5)."""
    w = workloads.make("c2")
    ex, ey = oracle.edges(0.0, 1.0, w.kx), oracle.edges(0.0, 1.0, w.ky)
    rects = np.array([[ex[i], ex[i + 1], ey[j], ey[j + 1]] for j in range(w.ky) for i in range(w.kx)])
    g = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    r = oracle.partition_rects(w.x, w.y, w.role, w.domain, rects, w.delta)
    for a in ("train_off", "train_idx", "val_off", "val_idx"):
        assert np.array_equal(getattr(g, a), getattr(r, a)), a


def test_splitmix64_reference_vector():
    """SplitMix64 seeded with 0: the published first outputs (Vigna's splitmix64.c)."""
    assert oracle.splitmix64(0, 1) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64(0, 2) == 0x6E789E6AA1B965F4
    assert oracle.splitmix64(0, 3) == 0x06C45D188009454F


def test_shell_cap_rules():
    """cap >= every shell: unchanged; cap = 0: only the core training points (= the
    delta = 0 lists); otherwise min(shell, cap) shell points kept, core whole, a subset of
    the original list, deterministic in the seed and dependent on it."""
    x, y, v, role = workloads.random_points(9, 4000, frac_val=0.1)
    D = (0, 1, 0, 1)
    _, rects = oracle.bisect(x, y, role, D, 3, 0.08)
    part = oracle.partition_rects(x, y, role, D, rects, 0.08)
    big = oracle.cap_shells(part, x, y, D, 10**6, 1)
    assert np.array_equal(big.train_idx, part.train_idx)
    zero = oracle.cap_shells(part, x, y, D, 0, 1)
    core_only = oracle.partition_rects(x, y, role, D, rects, 0.0)
    assert np.array_equal(zero.train_off, core_only.train_off) and np.array_equal(zero.train_idx, core_only.train_idx)
    cap = 60
    a = oracle.cap_shells(part, x, y, D, cap, 123)
    b = oracle.cap_shells(part, x, y, D, cap, 123)
    c = oracle.cap_shells(part, x, y, D, cap, 124)
    assert np.array_equal(a.train_idx, b.train_idx) and not np.array_equal(a.train_idx, c.train_idx)
    for s in range(8):
        full, kept, core = set(part.train(s)), a.train(s), set(core_only.train(s))
        assert np.all(np.diff(kept) > 0) and set(kept) <= full and core <= set(kept)
        assert len(set(kept) - core) == min(len(full - core), cap)



def test_shell_cap_hand_worked_golden(golden_dir):
    """Which shell members the cap keeps (R22), pinned by hand: tests/golden/shell_cap_small.json
    chooses the seed so that subset 1's keys are SplitMix64's published reference outputs
    (Vigna, seed 0: outputs 1-3), so the kept sets for caps 3, 2, 1, 0 follow by sorting
    three known numbers.  Pins: smallest keys are kept, the key index is s*2^32 + p + 1,
    the core is kept whole and a shell within the cap is untouched."""
    import json
    g = json.load(open(os.path.join(golden_dir, "shell_cap_small.json")))
    pts = np.array(g["points"])
    x, y, role = pts[:, 0], pts[:, 1], pts[:, 2].astype(np.uint8)
    rects = np.array(g["rects"])
    part = oracle.partition_rects(x, y, role, g["domain"], rects, g["delta"])
    for s in range(2):
        assert part.train(s).tolist() == g["train_uncapped"][s]
        assert part.val(s).tolist() == g["val"][s]
    gamma = 0x9e3779b97f4a7c15
    for p, key in g["keys_subset1"].items():  # the golden's key derivation, checked
        assert oracle.splitmix64(g["seed"], (1 << 32) + int(p) + 1) == int(key, 16)
        assert (g["seed"] + ((1 << 32) + int(p) + 1) * gamma) % (1 << 64) == (int(p) + 1) * gamma % (1 << 64)
    for cap, lists in g["capped"].items():
        capped = oracle.cap_shells(part, x, y, g["domain"], int(cap), g["seed"])
        for s in range(2):
            assert capped.train(s).tolist() == lists[s], (cap, s)


# ----------------------------------------------------------------- row f4: GLS

def _gls_setup(seed, n, depth, delta):
    x, y, v, role = workloads.random_points(seed, n, frac_val=0.1)
    X = np.stack([np.ones(n), x - 0.5, (y - 0.5) ** 2], 1)
    _, rects = oracle.bisect(x, y, role, (0, 1, 0, 1), depth, delta)
    part = oracle.partition_rects(x, y, role, (0, 1, 0, 1), rects, delta)
    return x, y, v, role, X, rects, part


def test_gls_single_subset_is_dense_gls():
    """One subset: the GLS estimate of Eq. GLS exactly, against a dense LAPACK
    route (scipy cho_solve of M, numpy solve of the normal equations)."""
    x, y, v, role, X, rects, part = _gls_setup(31, 400, 0, 0.0)
    prm = (0.15, 1.3, 0.2)
    beta, A, b = oracle.gls(x, y, v, X, part, rects, (0, 1, 0, 1), prm)
    t = role == 0
    M = _cov(x[t], y[t], x[t], y[t], prm[0]) + (prm[2] / prm[1]) * np.eye(int(t.sum()))
    cf = scipy.linalg.cho_factor(M, lower=True)
    MiX, Miy = scipy.linalg.cho_solve(cf, X[t]), scipy.linalg.cho_solve(cf, v[t])
    np.testing.assert_allclose(A, X[t].T @ MiX, rtol=1e-10)
    np.testing.assert_allclose(b, X[t].T @ Miy, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(beta, np.linalg.solve(X[t].T @ MiX, X[t].T @ Miy), rtol=1e-9)


def test_gls_reproduces_exact_linear_mean_on_any_division():
    """y = X beta0 exactly: A beta0 = b holds term by term for every subset division, so
    beta_hat = beta0 whatever the subsets and shells (a property of reading R23)."""
    x, y, v, role, X, rects, part = _gls_setup(32, 1500, 3, 0.1)
    beta0 = np.array([0.7, -1.25, 2.0])
    beta, _, _ = oracle.gls(x, y, X @ beta0, X, part, rects, (0, 1, 0, 1), (0.1, 1.0, 0.05))
    np.testing.assert_allclose(beta, beta0, rtol=1e-9)


def test_gls_large_nugget_is_ols_mean():
    """X = 1 and lambda -> infinity: M ~ lambda I, the GLS estimate tends to mean(y_T)."""
    x, y, v, role, X, rects, part = _gls_setup(33, 500, 2, 0.05)
    beta, _, _ = oracle.gls(x, y, v, X[:, :1], part, rects, (0, 1, 0, 1), (0.1, 1.0, 1e9))
    assert beta[0] == pytest.approx(v[role == 0].mean(), rel=1e-6)


def test_gls_rows_match_the_papers_prediction_identity():
    """M^{-1} = (1/lambda)(I - H), H = Sigma (Sigma + lambda I)^{-1}: the
    subset GLS sums equal the ones built from the oracle's kriging predictions of the X
    columns at the training sites (the paper's 'spatial prediction operation')."""
    x, y, v, role, X, rects, part = _gls_setup(34, 300, 1, 0.1)
    prm = (0.2, 1.0, 0.3)
    lam = prm[2] / prm[1]
    _, A, b = oracle.gls(x, y, v, X, part, rects, (0, 1, 0, 1), prm)
    A2, b2 = np.zeros_like(A), np.zeros_like(b)
    for s in range(2):
        ti = part.train(s)
        x0, x1, y0, y1 = rects[s]
        core = (x0 <= x[ti]) & ((x[ti] < x1) | (x1 == 1.0)) & (y0 <= y[ti]) & ((y[ti] < y1) | (y1 == 1.0))
        cols = []
        for col in [v[ti]] + [X[ti, j] for j in range(X.shape[1])]:
            # Eq.3 predicting the training sites themselves gives H col (the cross-covariance
            # row of a training site is its Sigma row), so M^{-1} col = (col - H col) / lambda
            _, pred = oracle.subset_cv(x[ti], y[ti], col, x[ti], y[ti], np.zeros(ti.size), *prm, return_yhat=True)
            cols.append((col - pred) / lam)
        Wy, WX = cols[0], np.stack(cols[1:], 1)
        A2 += X[ti][core].T @ WX[core]
        b2 += X[ti][core].T @ Wy[core]
    np.testing.assert_allclose(A, A2, rtol=1e-8)
    np.testing.assert_allclose(b, b2, rtol=1e-8, atol=1e-9)
