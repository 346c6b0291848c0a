"""CPU oracle for the parallel cross-validation loss (Gerber & Nychka, arXiv 1912.13132).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product path (``paper_1912_13132_b200``) never imports, links or calls it, and the
two share no code: this is the plain definition of Eq.7 evaluated by
Algorithm 1, written in ``oracle.c`` (fp64, ``-ffp-contract=off``) and driven
from here with ctypes.  Every function cites the passage it follows; DESIGN.md lists the
readings (R1..R18) taken where the paper is silent.

Pins (tests/test_oracle_pins.py, all ``-m "not gpu"``): closed-form kriging for k = 1, 2,
3; exp-covariance values; interpolation at observed sites with zero nugget; far-field
zero prediction; N = 1 and delta-saturation exactness (Eq.7 == Eq.4); power-of-two
metamorphic invariants (bit-exact); permutation invariance; partition invariants and
hand-worked golden partitions (tests/golden/).  The per-config global losses at the
BASELINE sizes c2..c5 have no printed value in the paper: "parity unpinned" beyond the
agreement of the two independent implementations.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, EINVAL, ENUMERIC, ENOMEM = 0, -2, -3, -6


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2 -ffp-contract=off; no FMA, IEEE doubles)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-std=c11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            d, i32, i64, p = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
            lib.oracle_edges.argtypes = [d, d, i32, p]
            u8 = ctypes.c_uint8
            lib.oracle_partition_count.argtypes = [i64, p, p, p, d, d, d, d, i32, i32, d, u8, p, p]
            lib.oracle_partition_fill.argtypes = [i64, p, p, p, d, d, d, d, i32, i32, d, u8, p, p, p, p]
            for f in (lib.oracle_subset_cv, lib.oracle_subset_cv_ld):
                f.argtypes = [i64, p, p, p, i64, p, p, p, d, d, d, p, p]
            lib.oracle_neg2loglik.argtypes = [i64, p, p, p, d, d, d, p]
            u64 = ctypes.c_uint64
            lib.oracle_bisect.argtypes = [i64, p, p, p, d, d, d, d, i32, d, p, p]
            lib.oracle_partition_rects_count.argtypes = [i64, p, p, p, d, d, i64, p, d, u8, p, p]
            lib.oracle_partition_rects_fill.argtypes = [i64, p, p, p, d, d, i64, p, d, u8, p, p, p, p]
            lib.oracle_splitmix64.argtypes = [u64, u64]
            lib.oracle_splitmix64.restype = u64
            lib.oracle_cap_shell.argtypes = [i64, p, p, p, p, d, d, i64, u64, i64, p, p]
            lib.oracle_gls_subset.argtypes = [i64, p, p, p, p, p, i32, d, d, d, p, p]
            lib.oracle_solve_small.argtypes = [i32, p, p, p]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


def edges(a: float, b: float, K: int) -> np.ndarray:
    """Tile edges e_0..e_K of [a, b) in K equal tiles (reading R4; P:242-246 divides D)."""
    e = np.empty(K + 1, np.float64)
    rc = _load().oracle_edges(a, b, K, _ptr(e))
    if rc:
        raise OracleError(rc, "edges")
    return e


class Partition:
    """CSR membership lists of Alg.1 lines 2-3: train (core + shell)
    and validation (core only, Eq.7) per subset s = iy*kx + ix."""

    def __init__(self, train_off, train_idx, val_off, val_idx, kx, ky):
        self.train_off, self.train_idx = train_off, train_idx
        self.val_off, self.val_idx = val_off, val_idx
        self.kx, self.ky = kx, ky

    @property
    def n_subsets(self) -> int:
        return self.kx * self.ky

    def k(self) -> np.ndarray:
        return np.diff(self.train_off)

    def m(self) -> np.ndarray:
        return np.diff(self.val_off)

    def train(self, s: int) -> np.ndarray:
        return self.train_idx[self.train_off[s]:self.train_off[s + 1]]

    def val(self, s: int) -> np.ndarray:
        return self.val_idx[self.val_off[s]:self.val_off[s + 1]]


def partition(x, y, role, domain, kx: int, ky: int, delta: float, core_role: int = 1) -> Partition:
    """Brute-force subset membership (Alg.1 lines 2-3; shell of width delta, P:154-159;
    readings R1-R6).  Every point is tested against every tile interval on each axis.
    ``core_role`` selects the points listed per core tile: 1 = validation (y^i_V), 2 = test
    (the held-out points predicted with the chosen parameters)."""
    lib = _load()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    role = np.ascontiguousarray(role, np.uint8)
    n = x.shape[0]
    N = kx * ky
    tc = np.zeros(N, np.int64)
    vc = np.zeros(N, np.int64)
    xmin, xmax, ymin, ymax = (float(v) for v in domain)
    rc = lib.oracle_partition_count(n, _ptr(x), _ptr(y), _ptr(role), xmin, xmax, ymin, ymax,
                                    kx, ky, float(delta), int(core_role), _ptr(tc), _ptr(vc))
    if rc:
        raise OracleError(rc, "partition")
    toff = np.zeros(N + 1, np.int64)
    voff = np.zeros(N + 1, np.int64)
    np.cumsum(tc, out=toff[1:])
    np.cumsum(vc, out=voff[1:])
    tidx = np.empty(int(toff[-1]), np.int32)
    vidx = np.empty(int(voff[-1]), np.int32)
    rc = lib.oracle_partition_fill(n, _ptr(x), _ptr(y), _ptr(role), xmin, xmax, ymin, ymax,
                                   kx, ky, float(delta), int(core_role), _ptr(toff), _ptr(tidx),
                                   _ptr(voff), _ptr(vidx))
    if rc:
        raise OracleError(rc, "partition")
    return Partition(toff, tidx, voff, vidx, kx, ky)


def subset_cv(tx, ty, tv, vx, vy, vv, range_: float, sigma2: float, nugget: float,
              long_double: bool = False, return_yhat: bool = False):
    """CV(y~_T, y_V, zeta) of Eq.4 with Eq.3's predictor for one
    subset and one (range, sigma^2, nugget).  Raises OracleError(ENUMERIC) if not PD.
    With ``return_yhat`` also returns the predictions yhat_v (Eq.3) as an array."""
    lib = _load()
    a = [np.ascontiguousarray(v, np.float64) for v in (tx, ty, tv, vx, vy, vv)]
    out = np.zeros(1, np.float64)
    yhat = np.zeros(a[3].shape[0], np.float64)
    f = lib.oracle_subset_cv_ld if long_double else lib.oracle_subset_cv
    rc = f(a[0].shape[0], _ptr(a[0]), _ptr(a[1]), _ptr(a[2]), a[3].shape[0], _ptr(a[3]),
           _ptr(a[4]), _ptr(a[5]), float(range_), float(sigma2), float(nugget), _ptr(out),
           _ptr(yhat) if return_yhat else None)
    if rc:
        raise OracleError(rc, "subset_cv")
    return (float(out[0]), yhat) if return_yhat else float(out[0])


def neg2loglik(tx, ty, tv, range_: float, sigma2: float, nugget: float) -> float:
    """-2 log-likelihood of Eq.2 for one training vector (NEXT row f3)."""
    lib = _load()
    a = [np.ascontiguousarray(v, np.float64) for v in (tx, ty, tv)]
    out = np.zeros(1, np.float64)
    rc = lib.oracle_neg2loglik(a[0].shape[0], _ptr(a[0]), _ptr(a[1]), _ptr(a[2]),
                               float(range_), float(sigma2), float(nugget), _ptr(out))
    if rc:
        raise OracleError(rc, "neg2loglik")
    return float(out[0])


class CvReport:
    """loss[c] = sum over subsets in ascending s (Alg.1 line 9; reading R13);
    subset_loss[s, c]; status[c] = -1 ok else first subset whose factorization failed."""

    def __init__(self, loss, subset_loss, status):
        self.loss, self.subset_loss, self.status = loss, subset_loss, status


def cv_loss(x, y, v, part: Partition, params, subsets=None, threads: int | None = None,
            long_double: bool = False) -> CvReport:
    """C~V of Eq.7 for each params row (range, sigma2, nugget), evaluated per
    Algorithm 1: independent per-subset SSPE z_i, then z = sum z_i.

    ``subsets`` restricts the evaluation to a sample (others left NaN and excluded from
    the sum -- used only for bounded baselines and sampled parity).  The thread pool over
    (subset, config) tasks is the parfor of Alg.1 line 4; it does not change any value.
    """
    params = np.asarray(params, np.float64).reshape(-1, 3)
    C = params.shape[0]
    N = part.n_subsets
    sub = np.arange(N) if subsets is None else np.asarray(subsets, np.int64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    res = np.full((N, C), np.nan)
    st = np.zeros((N, C), np.int32)
    k = part.k()
    tasks = [(int(s), c) for s in sub for c in range(C)]
    tasks.sort(key=lambda t: -int(k[t[0]]) ** 3)  # LPT order; does not change values

    def run(t):
        s, c = t
        ti, vi = part.train(s), part.val(s)
        try:
            res[s, c] = subset_cv(x[ti], y[ti], v[ti], x[vi], y[vi], v[vi], *params[c],
                                  long_double=long_double)
        except OracleError as e:
            if e.code != ENUMERIC:
                raise
            st[s, c] = 1

    nthreads = threads or os.cpu_count() or 1
    if nthreads == 1:
        for t in tasks:
            run(t)
    else:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(run, tasks))
    loss = np.zeros(C)
    status = np.full(C, -1, np.int32)
    for c in range(C):
        acc = 0.0
        for s in sub:  # ascending subset order (Alg.1 line 9)
            if st[s, c]:
                if status[c] < 0:
                    status[c] = s
                continue
            acc = acc + float(res[s, c])
        loss[c] = math.nan if status[c] >= 0 else acc
    return CvReport(loss, res, status)


def subset_flops(k, m) -> float:
    """Algorithmic flop count of one (subset, config) evaluation:
    k^3/3 + k^2/2 + k/6 (Cholesky) + 2k^2 (two triangular solves) + 2mk + 3m."""
    k = np.asarray(k, np.float64)
    m = np.asarray(m, np.float64)
    f = k ** 3 / 3 + k ** 2 / 2 + k / 6 + 2 * k ** 2 + 2 * m * k + 3 * m
    return np.where(m > 0, f, 0.0)


def neg2loglik_all(x, y, v, part: Partition, params, subsets=None, threads: int | None = None):
    """Row f3: per-subset -2 log-likelihood (Eq.2) of each subset's training data
    y~^i_T, and their sum over subsets in ascending s (a composite likelihood; NaN when a
    subset's covariance is not PD).  Returns (total[C], per_subset[N, C])."""
    params = np.asarray(params, np.float64).reshape(-1, 3)
    C, N = params.shape[0], part.n_subsets
    sub = np.arange(N) if subsets is None else np.asarray(subsets, np.int64)
    res = np.full((N, C), np.nan)
    tasks = [(int(s), c) for s in sub for c in range(C)]

    def run(t):
        s, c = t
        ti = part.train(s)
        try:
            res[s, c] = neg2loglik(x[ti], y[ti], v[ti], *params[c])
        except OracleError as e:
            if e.code != ENUMERIC:
                raise

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(run, tasks))
    total = np.zeros(C)
    for c in range(C):
        acc = 0.0
        for s in sub:
            acc = acc + float(res[s, c])
        total[c] = acc
    return total, res


def select(loss, subset_loss, m):
    """Row f1, the grid-search consumer, written out plainly:
    best = argmin_c loss[c] (ties -> lowest c, NaN never wins); global RMSPE
    sqrt(loss / n_V); local RMSPE sqrt(z_{s,c} / m_s); local best argmin_c z_{s,c}
    (-1 when m_s = 0); wins[c] = number of subsets whose local best is c."""
    loss = np.asarray(loss, np.float64)
    subset_loss = np.asarray(subset_loss, np.float64)
    m = np.asarray(m, np.int64)
    N, C = subset_loss.shape
    n_v = int(m.sum())
    best, bl = -1, None
    for c in range(C):
        if not math.isnan(loss[c]) and (best < 0 or loss[c] < bl):
            best, bl = c, loss[c]
    rmspe = np.array([math.sqrt(loss[c] / n_v) if not math.isnan(loss[c]) else math.nan for c in range(C)])
    local_best = np.full(N, -1, np.int32)
    local_rmspe = np.full((N, C), np.nan)
    wins = np.zeros(C, np.int32)
    for s in range(N):
        if m[s] == 0:
            continue
        b, bz = -1, None
        for c in range(C):
            z = subset_loss[s, c]
            if math.isnan(z):
                continue
            local_rmspe[s, c] = math.sqrt(z / m[s])
            if b < 0 or z < bz:
                b, bz = c, z
        local_best[s] = b
        if b >= 0:
            wins[b] += 1
    return best, rmspe, local_best, local_rmspe, wins


def predict(x, y, v, part: Partition, params, subset_config=None, threads: int | None = None):
    """Kriging prediction of each subset's core-tile targets (``part`` built with
    core_role=2 for the test points) with params[subset_config[s]].  Returns
    (sspe total in ascending s, per-subset sspe[N], yhat in the target CSR order)."""
    params = np.asarray(params, np.float64).reshape(-1, 3)
    N = part.n_subsets
    cfg = np.zeros(N, np.int64) if subset_config is None else np.asarray(subset_config, np.int64)
    sub = np.zeros(N)
    yhat = np.zeros(int(part.val_off[-1]))

    def run(s):
        ti, vi = part.train(s), part.val(s)
        if vi.size == 0:
            return
        l, yh = subset_cv(x[ti], y[ti], v[ti], x[vi], y[vi], v[vi], *params[cfg[s]], return_yhat=True)
        sub[s] = l
        yhat[part.val_off[s]:part.val_off[s + 1]] = yh

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(run, range(N)))
    total = 0.0
    for s in range(N):
        total = total + float(sub[s])
    return total, sub, yhat


# ----------------------------------------------------------------- row f2: bisection

class RectPartition(Partition):
    """Partition over an explicit list of N leaf rectangles (x0, x1, y0, y1)."""

    def __init__(self, train_off, train_idx, val_off, val_idx, rects):
        super().__init__(train_off, train_idx, val_off, val_idx, len(rects), 1)
        self.rects = rects


def bisect(x, y, role, domain, depth: int, delta: float):
    """Recursive shell-balanced bisection of D into 2^depth rectangles (readings
    R19-R21 in oracle.c).  Returns (splits[2^depth] by node id, rects[2^depth, 4])."""
    lib = _load()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    role = np.ascontiguousarray(role, np.uint8)
    N = 1 << depth
    rects = np.zeros((N, 4), np.float64)
    splits = np.zeros(N, np.float64)
    xmin, xmax, ymin, ymax = (float(v) for v in domain)
    rc = lib.oracle_bisect(x.shape[0], _ptr(x), _ptr(y), _ptr(role), xmin, xmax, ymin, ymax, int(depth),
                           float(delta), _ptr(rects), _ptr(splits))
    if rc:
        raise OracleError(rc, "bisect")
    return splits, rects


def partition_rects(x, y, role, domain, rects, delta: float, core_role: int = 1) -> RectPartition:
    """Brute-force membership over leaf rectangles: training = role 0 in the dilation by
    delta (R2/R3), core lists = role core_role in the rectangle; ascending index."""
    lib = _load()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    role = np.ascontiguousarray(role, np.uint8)
    rects = np.ascontiguousarray(rects, np.float64).reshape(-1, 4)
    N = rects.shape[0]
    xmax, ymax = float(domain[1]), float(domain[3])
    tc = np.zeros(N, np.int64)
    vc = np.zeros(N, np.int64)
    lib.oracle_partition_rects_count(x.shape[0], _ptr(x), _ptr(y), _ptr(role), xmax, ymax, N, _ptr(rects),
                                     float(delta), int(core_role), _ptr(tc), _ptr(vc))
    toff = np.zeros(N + 1, np.int64)
    voff = np.zeros(N + 1, np.int64)
    np.cumsum(tc, out=toff[1:])
    np.cumsum(vc, out=voff[1:])
    tidx = np.empty(int(toff[-1]), np.int32)
    vidx = np.empty(int(voff[-1]), np.int32)
    lib.oracle_partition_rects_fill(x.shape[0], _ptr(x), _ptr(y), _ptr(role), xmax, ymax, N, _ptr(rects),
                                    float(delta), int(core_role), _ptr(toff), _ptr(tidx), _ptr(voff), _ptr(vidx))
    return RectPartition(toff, tidx, voff, vidx, rects)


def splitmix64(seed: int, i: int) -> int:
    """Output i >= 1 of SplitMix64 seeded with ``seed`` (the shell-cap sampling keys)."""
    return int(_load().oracle_splitmix64(seed & (2**64 - 1), i & (2**64 - 1)))


def cap_shells(part: RectPartition, x, y, domain, cap: int, seed: int) -> RectPartition:
    """Shell cap (reading R22): in every subset whose shell (training points
    outside the core rectangle) exceeds ``cap``, keep the ``cap`` shell members with the
    smallest SplitMix64 keys (ties: smaller index); the core part is kept whole."""
    lib = _load()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    xmax, ymax = float(domain[1]), float(domain[3])
    N = part.n_subsets
    lists = []
    for s in range(N):
        idx = np.ascontiguousarray(part.train(s), np.int32)
        out = np.empty(max(idx.size, 1), np.int32)
        kout = np.zeros(1, np.int64)
        rect = np.ascontiguousarray(part.rects[s], np.float64)
        lib.oracle_cap_shell(idx.size, _ptr(idx), _ptr(x), _ptr(y), _ptr(rect), xmax, ymax, int(cap),
                             seed & (2**64 - 1), s, _ptr(out), _ptr(kout))
        lists.append(out[:int(kout[0])].copy())
    toff = np.zeros(N + 1, np.int64)
    np.cumsum([l.size for l in lists], out=toff[1:])
    tidx = np.concatenate(lists) if lists else np.empty(0, np.int32)
    return RectPartition(toff, tidx.astype(np.int32), part.val_off, part.val_idx, part.rects)


# ----------------------------------------------------------------- row f4: GLS

def gls(x, y, v, X, part, rects, domain, param, subsets=None, threads: int | None = None):
    """Row f4 (Eq. GLS; reading R23): beta_hat = A^{-1} b with
    A = sum_s sum_{p in core_s} X_p^T (M_s^{-1} X^s)_p and b likewise with y, summed over
    subsets in ascending s; ``part`` gives the training lists, ``rects`` the cores (a
    training point is in core s iff it lies in rectangle s, R3).  Returns (beta, A, b)."""
    lib = _load()
    X = np.ascontiguousarray(X, np.float64)
    p = X.shape[1]
    rects = np.asarray(rects, np.float64).reshape(-1, 4)
    xmax, ymax = float(domain[1]), float(domain[3])
    N = part.n_subsets
    sub = np.arange(N) if subsets is None else np.asarray(subsets, np.int64)
    As = np.zeros((N, p, p))
    bs = np.zeros((N, p))

    def core_mask(s, ti):
        x0, x1, y0, y1 = rects[s]
        cx = (x0 <= x[ti]) & ((x[ti] < x1) | ((x1 == xmax) & (x[ti] == xmax)))
        cy = (y0 <= y[ti]) & ((y[ti] < y1) | ((y1 == ymax) & (y[ti] == ymax)))
        return np.ascontiguousarray(cx & cy, np.uint8)

    def run(s):
        ti = part.train(s)
        a = [np.ascontiguousarray(arr[ti], np.float64) for arr in (x, y, v)]
        Xs = np.ascontiguousarray(X[ti])
        cm = core_mask(s, ti)
        A = np.zeros(p * p)
        b = np.zeros(p)
        rc = lib.oracle_gls_subset(ti.size, _ptr(a[0]), _ptr(a[1]), _ptr(a[2]), _ptr(Xs), _ptr(cm), p,
                                   float(param[0]), float(param[1]), float(param[2]), _ptr(A), _ptr(b))
        if rc:
            raise OracleError(rc, "gls_subset")
        As[s] = A.reshape(p, p)
        bs[s] = b

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(run, [int(s) for s in sub]))
    A = np.zeros((p, p))
    b = np.zeros(p)
    for s in sub:  # ascending subset order
        A = A + As[s]
        b = b + bs[s]
    beta = np.zeros(p)
    Ac, bc = np.ascontiguousarray(A), np.ascontiguousarray(b)
    rc = lib.oracle_solve_small(p, _ptr(Ac), _ptr(bc), _ptr(beta))
    if rc:
        raise OracleError(rc, "solve_small")
    return beta, A, b
