"""zeta dedup (Eq.3's prediction depends on zeta only through (range, lambda),
lambda = nugget / sigma2): pgpcv_evaluate factors every bit-identical (range, lambda) pair
once per call and shares the factor.  The results must be bit-identical to evaluating each
configuration on its own (one config per call: nothing to share), the -2 log-likelihood
(which does depend on sigma2, Eq.2) included, and the executed work is reported honestly."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


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


def _distinct(params):
    lam = params[:, 2] / params[:, 1]
    return len({(a.tobytes(), b.tobytes()) for a, b in zip(params[:, 0], lam)})


def test_c2_grid_dedup_bit_identical_to_one_config_per_call(ctx):
    w = workloads.make("c2", device="cuda")
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    C = len(w.params)
    U = _distinct(w.params)
    assert U < C  # the c2 grid has repeated (range, lambda) pairs
    res = ctx.evaluate(w.params, nll=True, subset_nll=True)
    t = ctx.last_timing()
    assert t["n_configs_executed"] == U
    N = ctx.info["n_subsets"]
    k = np.diff(ctx.partition_export()[0]).astype(np.float64)
    assert t["n_evals"] == N * U  # with the likelihood every subset is factored
    f = k ** 3 / 3 + k ** 2 / 2 + k / 6 + 2 * k ** 2 + 0.0
    assert t["flops"] < f.sum() * C  # executed work only
    for c in range(C):
        one = ctx.evaluate(w.params[c:c + 1], nll=True, subset_nll=True)
        assert ctx.last_timing()["n_configs_executed"] == 1
        assert np.array_equal(one.subset_loss[:, 0], res.subset_loss[:, c]), c
        assert np.array_equal(one.subset_nll[:, 0], res.subset_nll[:, c]), c
        assert one.loss[0] == res.loss[c] and one.nll[0] == res.nll[c]


def test_duplicates_share_loss_but_not_likelihood(ctx):
    """(range, 2 sigma2, 2 nugget) has the bit-identical lambda: same CV loss, but the
    likelihood differs by the sigma2 terms of Eq.2 -- both against the oracle."""
    x, y, v, role = workloads.random_points(5, 900, frac_val=0.1)
    ctx.partition(x, y, v, role, (0, 1, 0, 1), 2, 2, 0.1)
    p = np.array([[0.2, 1.0, 0.1], [0.2, 2.0, 0.2], [0.2, 0.5, 0.05], [0.3, 1.0, 0.1]])
    res = ctx.evaluate(p, nll=True, subset_nll=True)
    assert ctx.last_timing()["n_configs_executed"] == 2
    assert np.array_equal(res.subset_loss[:, 0], res.subset_loss[:, 1])
    assert np.array_equal(res.subset_loss[:, 0], res.subset_loss[:, 2])
    part = oracle.partition(x, y, role, (0, 1, 0, 1), 2, 2, 0.1)
    _, nll = oracle.neg2loglik_all(x, y, v, part, p, threads=4)
    assert np.all(np.abs(res.subset_nll - nll) <= 1e-9 * np.abs(nll))
    ref = oracle.cv_loss(x, y, v, part, p, threads=4)
    assert np.all(np.abs(res.subset_loss - ref.subset_loss) <= 1e-9 * np.abs(ref.subset_loss))
