"""The CV kernel's elementary FP64 functions (pgpcv_device_math runs the exact inlined
device code) against correctly rounded references: every covariance entry is
exp(-||t_i - t_j|| / range), so these bound the assembly's error.

* exp_neg(x), x in [-708, 0]: table-driven (2^(j/64) x degree-5 polynomial); reference
  mpmath at 60 digits, rounded to double.  Claim: <= 1 ulp.
* sqrt_nb(x), x >= 0 the squared distances: hardware rsqrt estimate + corrections;
  reference IEEE sqrt (numpy, correctly rounded).  Claim: <= 1 ulp; x < 2^-1000 -> 0.
* rsqrt_nb(x), x > 0 the Cholesky pivots: reference mpmath 1/sqrt.  Claim: <= 1 ulp.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_13132_b200 as pg
    c = pg.Context(0)
    yield c
    c.close()


def _ulp_diff(a, b):
    """|a - b| in units in the last place (both finite, same sign)."""
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    return np.abs(ia - ib)


def _mp(fn, xs):
    import mpmath
    mpmath.mp.dps = 60
    return np.array([float(fn(mpmath.mpf(float(v)))) for v in xs])


def test_exp_neg_within_one_ulp(ctx):
    import paper_1912_13132_b200 as pg
    rng = np.random.default_rng(1)
    ln2_64 = np.log(2.0) / 64
    x = np.concatenate([
        -rng.uniform(0, 708, 20000),
        -rng.exponential(1.0, 10000),                # the covariance's typical range
        -np.arange(0, 708 / ln2_64, 97) * ln2_64,    # table/reduction boundaries
        -np.arange(0, 708 / ln2_64, 97) * ln2_64 - 1e-12,
        [0.0, -0.0, -1e-300, -5e-324, -1e-16, -708.0, -707.9999999],
    ])
    y = ctx.device_math(pg.MATH_EXP_NEG, x)
    ref = _mp(lambda t: __import__("mpmath").exp(t), x)
    d = _ulp_diff(y, ref)
    assert d.max() <= 1, (d.max(), x[np.argmax(d)])
    assert y[x.size - 7] == 1.0 and y[x.size - 6] == 1.0


def test_sqrt_nb_within_one_ulp(ctx):
    import paper_1912_13132_b200 as pg
    rng = np.random.default_rng(2)
    x = np.concatenate([
        rng.uniform(0, 2 * 50.0 ** 2, 20000),        # squared distances on c5's domain
        rng.uniform(0, 1, 10000) ** 4,               # near-coincident points
        10.0 ** rng.uniform(-300, 3, 10000),
        np.arange(1, 2000, dtype=np.float64) ** 2,   # perfect squares
        [4.0, 0.25, 2.0 ** -998, 2.0 ** -999],
    ])
    y = ctx.device_math(pg.MATH_SQRT, x)
    d = _ulp_diff(y, np.sqrt(x))
    assert d.max() <= 1, (d.max(), x[np.argmax(d)])
    # scaling by 4 scales the result by exactly 2 (the power-of-two invariants, R8)
    y4 = ctx.device_math(pg.MATH_SQRT, 4 * x[:20000])
    assert np.array_equal(y4, 2 * y[:20000])
    z = ctx.device_math(pg.MATH_SQRT, np.array([0.0, 2.0 ** -1001, 1e-310]))
    assert np.all(z == 0.0)


def test_rsqrt_nb_within_one_ulp(ctx):
    import paper_1912_13132_b200 as pg
    rng = np.random.default_rng(3)
    x = np.concatenate([10.0 ** rng.uniform(-12, 6, 20000), rng.uniform(0.5, 2.5, 10000), [1.0, 4.0, 0.25]])
    y = ctx.device_math(pg.MATH_RSQRT, x)
    ref = _mp(lambda t: 1 / __import__("mpmath").sqrt(t), x)
    d = _ulp_diff(y, ref)
    assert d.max() <= 1, (d.max(), x[np.argmax(d)])
