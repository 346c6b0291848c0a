"""libpgpcv -- B200-native parallel cross-validation for Gaussian-process models.

Thin ctypes binding over the C ABI in ``include/pgpcv.h`` with the same names.  It does
argument marshalling only: every step of the hot path (partition, covariance assembly,
FP64 Cholesky, solves, prediction, loss reduction, the NCCL combine) runs in the CUDA
kernels of ``csrc/``.  There is no CPU fallback: importing this package without the built
``libpgpcv.so`` raises, and ``Context()`` fails without an sm_100 GPU.

Method: Gerber & Nychka, "Parallel cross-validation: a scalable fitting method for
Gaussian process models" (arXiv 1912.13132), Eq.7 evaluated by
Algorithm 1.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGPCV_LIB") or os.path.join(_HERE, "libpgpcv.so")

OK, EINVAL, ENUMERIC, EEMPTY, ECUDA, ENOMEM, ENCCL, ESTATE = 0, -2, -3, -4, -5, -6, -7, -8
ERROR_NAMES = {EINVAL: "EINVAL", ENUMERIC: "ENUMERIC", EEMPTY: "EEMPTY", ECUDA: "ECUDA",
               ENOMEM: "ENOMEM", ENCCL: "ENCCL", ESTATE: "ESTATE"}
NCCL_UNIQUE_ID_BYTES = 128
MAX_K = 65536

# Symbols include/pgpcv.h declares (checked by tests/test_abi.py).
EXPORTED = ("pgpcv_version", "pgpcv_create", "pgpcv_destroy", "pgpcv_last_error",
            "pgpcv_set_stream", "pgpcv_partition", "pgpcv_partition_device",
            "pgpcv_partition_bisect", "pgpcv_partition_bisect_device", "pgpcv_partition_rects",
            "pgpcv_partition_export", "pgpcv_shard", "pgpcv_nccl_get_unique_id",
            "pgpcv_cv_loss", "pgpcv_evaluate", "pgpcv_select", "pgpcv_predict",
            "pgpcv_partition_export_test", "pgpcv_gls", "pgpcv_last_timing", "pgpcv_lpt_assign",
            "pgpcv_nccl_library", "pgpcv_device_math")
ROLE_TRAIN, ROLE_VALIDATION, ROLE_TEST = 0, 1, 2
ABI_VERSION = 5
MATH_EXP_NEG, MATH_SQRT, MATH_RSQRT = 0, 1, 2


class PgpcvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


class Rect(ctypes.Structure):
    _fields_ = [("xmin", ctypes.c_double), ("xmax", ctypes.c_double),
                ("ymin", ctypes.c_double), ("ymax", ctypes.c_double)]


class Param(ctypes.Structure):
    _fields_ = [("range", ctypes.c_double), ("sigma2", ctypes.c_double), ("nugget", ctypes.c_double)]


class PartitionInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("n_subsets", "sum_k", "sum_m", "max_k", "max_m",
                                               "n_empty_val", "n_train", "n_val", "n_test",
                                               "max_test")]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class Outputs(ctypes.Structure):
    """pgpcv_outputs: host output pointers (NULL to skip)."""
    _fields_ = [(f, ctypes.c_void_p) for f in ("loss", "subset_loss", "status", "nll", "subset_nll")]


class Timing(ctypes.Structure):
    _fields_ = [("kernel_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("n_evals", ctypes.c_int64),
                ("launches", ctypes.c_int32), ("n_slots", ctypes.c_int32),
                ("n_configs_executed", ctypes.c_int32), ("reserved", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load_library():
    """Load the in-tree libpgpcv.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpgpcv.so is not built ({LIB_PATH}); run __graft_entry__.build() "
                          "or python paper_1912_13132_b200/_build.py")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    p, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.pgpcv_version.restype = ctypes.c_int
    lib.pgpcv_create.argtypes = [ctypes.c_int, ctypes.POINTER(p)]
    lib.pgpcv_destroy.argtypes = [p]
    lib.pgpcv_destroy.restype = None
    lib.pgpcv_last_error.argtypes = [p]
    lib.pgpcv_last_error.restype = ctypes.c_char_p
    lib.pgpcv_set_stream.argtypes = [p, p]
    lib.pgpcv_partition.argtypes = [p, i64, p, p, p, p, Rect, i32, i32, d, ctypes.POINTER(PartitionInfo)]
    lib.pgpcv_partition_device.argtypes = lib.pgpcv_partition.argtypes
    lib.pgpcv_partition_bisect.argtypes = [p, i64, p, p, p, p, Rect, i32, d, i64, ctypes.c_uint64,
                                           ctypes.POINTER(PartitionInfo)]
    lib.pgpcv_partition_bisect_device.argtypes = lib.pgpcv_partition_bisect.argtypes
    lib.pgpcv_partition_rects.argtypes = [p, p]
    lib.pgpcv_partition_export.argtypes = [p, p, p, p, p]
    lib.pgpcv_shard.argtypes = [p, ctypes.c_int, ctypes.c_int, p]
    lib.pgpcv_nccl_get_unique_id.argtypes = [p]
    lib.pgpcv_cv_loss.argtypes = [p, ctypes.POINTER(Param), i32, p, p, p]
    lib.pgpcv_evaluate.argtypes = [p, ctypes.POINTER(Param), i32, ctypes.POINTER(Outputs)]
    lib.pgpcv_select.argtypes = [p, p, p, p, p, p]
    lib.pgpcv_predict.argtypes = [p, ctypes.POINTER(Param), i32, p, i32, p, p, p]
    lib.pgpcv_partition_export_test.argtypes = [p, p, p]
    lib.pgpcv_gls.argtypes = [p, p, i32, Param, p, p, p]
    lib.pgpcv_last_timing.argtypes = [p, ctypes.POINTER(Timing)]
    lib.pgpcv_lpt_assign.argtypes = [i64, p, i32, p]
    lib.pgpcv_nccl_library.argtypes = [p, i64]
    lib.pgpcv_device_math.argtypes = [p, i32, i64, p, p]
    for name in EXPORTED:
        if name not in ("pgpcv_destroy", "pgpcv_last_error"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def version() -> int:
    return load_library().pgpcv_version()


def lpt_assign(cost, world: int) -> np.ndarray:
    """pgpcv_lpt_assign: owner rank of each item (host-only, no GPU needed)."""
    cost = np.ascontiguousarray(cost, np.float64)
    owner = np.empty(cost.shape[0], np.int32)
    rc = load_library().pgpcv_lpt_assign(cost.shape[0], _ptr(cost), world, _ptr(owner))
    if rc:
        raise PgpcvError(rc, "pgpcv_lpt_assign")
    return owner


def nccl_library() -> str:
    """pgpcv_nccl_library: the libnccl the library bound, "path (NCCL x.y.z)" (or why none)."""
    buf = ctypes.create_string_buffer(4096)
    load_library().pgpcv_nccl_library(buf, len(buf))
    return buf.value.decode()


def nccl_unique_id() -> bytes:
    """pgpcv_nccl_get_unique_id (rank 0), to be broadcast to the other ranks."""
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    rc = load_library().pgpcv_nccl_get_unique_id(buf)
    if rc:
        raise PgpcvError(rc, "pgpcv_nccl_get_unique_id")
    return buf.raw


@dataclass
class CvResult:
    loss: np.ndarray          # [C] global C~V (SSPE), Eq.7
    subset_loss: np.ndarray | None  # [N, C] per-subset SSPE z_i, or None
    status: np.ndarray        # [C] -1 ok, else first non-PD subset
    code: int                 # OK or ENUMERIC
    nll: np.ndarray | None = None         # [C] sum_s -2 log L_s (Eq.2 per subset)
    subset_nll: np.ndarray | None = None  # [N, C]


@dataclass
class Selection:
    best: int                 # argmin_c loss[c] (zeta_hat_CV), -1 if every config failed
    rmspe: np.ndarray         # [C] global RMSPE sqrt(loss / n_V)
    local_best: np.ndarray    # [N] per-subset argmin_c (-1 when no validation data)
    local_rmspe: np.ndarray   # [N, C]
    wins: np.ndarray          # [C] subsets won per config


@dataclass
class Prediction:
    sspe: float               # sum of squared prediction errors over all targets
    subset_sspe: np.ndarray   # [N]
    yhat: np.ndarray | None   # [n_targets] in target CSR order
    code: int                 # OK or ENUMERIC


class Context:
    """One libpgpcv context (one GPU).  Mirrors the ABI: partition -> [shard] -> cv_loss."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.pgpcv_create(int(device), ctypes.byref(h))
        if rc:
            raise PgpcvError(rc, self._lib.pgpcv_last_error(None).decode())
        self._h = h
        self.info: dict | None = None
        self._last_C = 0  # configs of the last CV evaluation (the shape pgpcv_select returns)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pgpcv_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int, what: str):
        if rc:
            raise PgpcvError(rc, f"{what}: {self._lib.pgpcv_last_error(self._h).decode()}")

    def set_stream(self, stream_ptr: int | None):
        self._check(self._lib.pgpcv_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)), "set_stream")

    def partition(self, x, y, value, role, domain, kx: int, ky: int, delta: float) -> dict:
        """pgpcv_partition with host arrays (Alg.1 lines 2-3)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        v = np.ascontiguousarray(value, np.float64)
        r = np.ascontiguousarray(role, np.uint8)
        n = x.shape[0]
        if not (y.shape[0] == v.shape[0] == r.shape[0] == n):
            raise ValueError("x, y, value, role must have equal length")
        info = PartitionInfo()
        rc = self._lib.pgpcv_partition(self._h, n, _ptr(x), _ptr(y), _ptr(v), _ptr(r), Rect(*domain),
                                       int(kx), int(ky), float(delta), ctypes.byref(info))
        self._check(rc, "pgpcv_partition")
        self.info = info.as_dict()
        return self.info

    def partition_device(self, x, y, value, role, domain, kx: int, ky: int, delta: float) -> dict:
        """pgpcv_partition_device: x, y, value (float64) and role (uint8) are CUDA tensors
        (or raw device pointers) on this context's device; n = len(x)."""
        def dp(t):
            return ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())
        n = x.numel() if hasattr(x, "numel") else int(len(x))
        info = PartitionInfo()
        rc = self._lib.pgpcv_partition_device(self._h, n, dp(x), dp(y), dp(value), dp(role),
                                              Rect(*domain), int(kx), int(ky), float(delta),
                                              ctypes.byref(info))
        self._check(rc, "pgpcv_partition_device")
        self.info = info.as_dict()
        return self.info

    def partition_bisect(self, x, y, value, role, domain, depth: int, delta: float, shell_cap: int = -1,
                         seed: int = 0) -> dict:
        """pgpcv_partition_bisect with host arrays (row f2: recursive shell-balanced bisection
        into 2^depth subsets, optional shell cap)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        v = np.ascontiguousarray(value, np.float64)
        r = np.ascontiguousarray(role, np.uint8)
        n = x.shape[0]
        if not (y.shape[0] == v.shape[0] == r.shape[0] == n):
            raise ValueError("x, y, value, role must have equal length")
        info = PartitionInfo()
        rc = self._lib.pgpcv_partition_bisect(self._h, n, _ptr(x), _ptr(y), _ptr(v), _ptr(r), Rect(*domain),
                                              int(depth), float(delta), int(shell_cap), int(seed) & (2**64 - 1),
                                              ctypes.byref(info))
        self._check(rc, "pgpcv_partition_bisect")
        self.info = info.as_dict()
        return self.info

    def partition_bisect_device(self, x, y, value, role, domain, depth: int, delta: float, shell_cap: int = -1,
                                seed: int = 0) -> dict:
        """pgpcv_partition_bisect_device: CUDA tensors on this context's device."""
        def dp(t):
            return ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())
        n = x.numel() if hasattr(x, "numel") else int(len(x))
        info = PartitionInfo()
        rc = self._lib.pgpcv_partition_bisect_device(self._h, n, dp(x), dp(y), dp(value), dp(role), Rect(*domain),
                                                     int(depth), float(delta), int(shell_cap),
                                                     int(seed) & (2**64 - 1), ctypes.byref(info))
        self._check(rc, "pgpcv_partition_bisect_device")
        self.info = info.as_dict()
        return self.info

    def partition_rects(self) -> np.ndarray:
        """pgpcv_partition_rects: [N, 4] (x0, x1, y0, y1) per subset."""
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        out = np.empty((self.info["n_subsets"], 4), np.float64)
        self._check(self._lib.pgpcv_partition_rects(self._h, _ptr(out)), "pgpcv_partition_rects")
        return out

    def partition_export(self):
        """(train_off, train_idx, val_off, val_idx) CSR membership of the partition."""
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        N = self.info["n_subsets"]
        toff = np.empty(N + 1, np.int64)
        voff = np.empty(N + 1, np.int64)
        tidx = np.empty(self.info["sum_k"], np.int32)
        vidx = np.empty(self.info["sum_m"], np.int32)
        self._check(self._lib.pgpcv_partition_export(self._h, _ptr(toff), _ptr(tidx), _ptr(voff),
                                                     _ptr(vidx)), "pgpcv_partition_export")
        return toff, tidx, voff, vidx

    def shard(self, rank: int, world: int, unique_id: bytes | None = None):
        buf = ctypes.create_string_buffer(unique_id, NCCL_UNIQUE_ID_BYTES) if unique_id else None
        self._check(self._lib.pgpcv_shard(self._h, int(rank), int(world), buf), "pgpcv_shard")

    def cv_loss(self, params, want_subset_loss: bool = True) -> CvResult:
        """pgpcv_cv_loss for params rows (range, sigma2, nugget) -> CvResult."""
        params = np.ascontiguousarray(params, np.float64).reshape(-1, 3)
        C = params.shape[0]
        par = (Param * C)(*[Param(*row) for row in params.tolist()])
        loss = np.empty(C, np.float64)
        status = np.empty(C, np.int32)
        sub = None
        if want_subset_loss:
            if self.info is None:
                raise PgpcvError(ESTATE, "no partition")
            sub = np.empty((self.info["n_subsets"], C), np.float64)
        rc = self._lib.pgpcv_cv_loss(self._h, par, C, _ptr(loss), _ptr(sub) if sub is not None else None,
                                     _ptr(status))
        if rc not in (OK, ENUMERIC):
            self._check(rc, "pgpcv_cv_loss")
        self._last_C = C
        return CvResult(loss, sub, status, rc)

    def evaluate(self, params, loss: bool = True, subset_loss: bool = True, nll: bool = False,
                 subset_nll: bool = False) -> CvResult:
        """pgpcv_evaluate: CV loss and/or per-subset -2 log-likelihood from one factorization."""
        params = np.ascontiguousarray(params, np.float64).reshape(-1, 3)
        C = params.shape[0]
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        N = self.info["n_subsets"]
        par = (Param * C)(*[Param(*row) for row in params.tolist()])
        arr = {"loss": np.empty(C) if loss else None,
               "subset_loss": np.empty((N, C)) if subset_loss else None,
               "status": np.empty(C, np.int32),
               "nll": np.empty(C) if nll else None,
               "subset_nll": np.empty((N, C)) if subset_nll else None}
        out = Outputs(**{k: (v.ctypes.data if v is not None else None) for k, v in arr.items()})
        rc = self._lib.pgpcv_evaluate(self._h, par, C, ctypes.byref(out))
        if rc not in (OK, ENUMERIC):
            self._check(rc, "pgpcv_evaluate")
        self._last_C = C if (loss or subset_loss) else 0
        return CvResult(arr["loss"], arr["subset_loss"], arr["status"], rc, arr["nll"], arr["subset_nll"])

    def select(self) -> Selection:
        """pgpcv_select on the last CV evaluation (grid-search consumer)."""
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        N = self.info["n_subsets"]
        C = self._last_C
        if C <= 0:
            raise PgpcvError(ESTATE, "pgpcv_select needs a preceding CV evaluation")
        best = np.empty(1, np.int32)
        rmspe = np.empty(C)
        lb = np.empty(N, np.int32)
        lr = np.empty((N, C))
        wins = np.empty(C, np.int32)
        self._check(self._lib.pgpcv_select(self._h, _ptr(best), _ptr(rmspe), _ptr(lb), _ptr(lr), _ptr(wins)),
                    "pgpcv_select")
        return Selection(int(best[0]), rmspe, lb, lr, wins)

    def predict(self, params, subset_config=None, target_role: int = ROLE_TEST,
                want_yhat: bool = True) -> Prediction:
        """pgpcv_predict: kriging predictions of the targets with params[subset_config[s]]."""
        params = np.ascontiguousarray(params, np.float64).reshape(-1, 3)
        C = params.shape[0]
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        N = self.info["n_subsets"]
        par = (Param * C)(*[Param(*row) for row in params.tolist()])
        cfg = None if subset_config is None else np.ascontiguousarray(subset_config, np.int32)
        if cfg is not None and cfg.shape != (N,):
            raise ValueError("subset_config must have one entry per subset")
        n_t = self.info["n_test"] if target_role == ROLE_TEST else self.info["sum_m"]
        yhat = np.empty(n_t) if want_yhat else None
        sub = np.empty(N)
        tot = np.empty(1)
        rc = self._lib.pgpcv_predict(self._h, par, C, _ptr(cfg) if cfg is not None else None, int(target_role),
                                     _ptr(yhat) if yhat is not None else None, _ptr(sub), _ptr(tot))
        if rc not in (OK, ENUMERIC):
            self._check(rc, "pgpcv_predict")
        return Prediction(float(tot[0]), sub, yhat, rc)

    def gls(self, X, param):
        """pgpcv_gls (row f4): (beta, X^T M^-1 X, X^T M^-1 y) for covariates X [n, p] of the
        partition's points and one (range, sigma2, nugget)."""
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        X = np.ascontiguousarray(X, np.float64)
        if X.ndim != 2:
            raise ValueError("X must be [n, p]")
        p = X.shape[1]
        beta = np.empty(p)
        A = np.empty((p, p))
        b = np.empty(p)
        rc = self._lib.pgpcv_gls(self._h, _ptr(X), p, Param(*[float(v) for v in param]), _ptr(beta), _ptr(A),
                                 _ptr(b))
        if rc not in (OK, ENUMERIC):
            self._check(rc, "pgpcv_gls")
        return beta, A, b

    def partition_export_test(self):
        """(test_off, test_idx): CSR lists of the test points (role 2) per core tile."""
        if self.info is None:
            raise PgpcvError(ESTATE, "no partition")
        N = self.info["n_subsets"]
        off = np.empty(N + 1, np.int64)
        idx = np.empty(self.info["n_test"], np.int32)
        self._check(self._lib.pgpcv_partition_export_test(self._h, _ptr(off), _ptr(idx)),
                    "pgpcv_partition_export_test")
        return off, idx

    def device_math(self, fn: int, x) -> np.ndarray:
        """pgpcv_device_math (diagnostic): the CV kernel's exp_neg / sqrt / rsqrt on x."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._check(self._lib.pgpcv_device_math(self._h, int(fn), x.size, _ptr(x), _ptr(y)), "pgpcv_device_math")
        return y

    def last_timing(self) -> dict:
        t = Timing()
        self._check(self._lib.pgpcv_last_timing(self._h, ctypes.byref(t)), "pgpcv_last_timing")
        return t.as_dict()


def subset_flops(k, m) -> np.ndarray:
    """Algorithmic FP64 flops of one (subset, config) evaluation."""
    k = np.asarray(k, np.float64)
    m = np.asarray(m, np.float64)
    return np.where(m > 0, k ** 3 / 3 + k ** 2 / 2 + k / 6 + 2 * k ** 2 + 2 * m * k + 3 * m, 0.0)
