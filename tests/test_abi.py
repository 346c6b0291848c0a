"""The C-ABI library loads and exports every symbol include/pgpcv.h declares; host-only
entry points (no GPU) behave as documented.  No compute calls here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1912_13132_b200 as pg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "pgpcv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pgpcv_[a-z_]+)\s*\(", src)))


def test_header_declares_the_binding_names():
    assert _declared_symbols() == sorted(pg.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = pg.load_library()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert pg.version() == pg.ABI_VERSION == 5


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {pg.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out and "sm_90" not in out


def test_lpt_assign_rule():
    """LPT: descending cost (ties: ascending index), each to the least-loaded rank (ties:
    lowest rank) -- the rule pgpcv_shard applies."""
    cost = np.array([5.0, 9.0, 9.0, 1.0, 4.0, 7.0])
    owner = pg.lpt_assign(cost, 2)
    # order 1(9),2(9),5(7),0(5),4(4),3(1): r0<-1, r1<-2, r1<-5 (9<16? r1 has 9 -> tie? r0=9,r1=9 -> r0)
    loads = np.zeros(2)
    expect = np.empty(6, np.int32)
    for i in sorted(range(6), key=lambda i: (-cost[i], i)):
        r = int(np.argmin(loads))
        expect[i] = r
        loads[r] += cost[i]
    assert owner.tolist() == expect.tolist()
    assert pg.lpt_assign(cost, 1).tolist() == [0] * 6
    big = np.random.default_rng(0).uniform(1, 100, 1000) ** 3
    o8 = pg.lpt_assign(big, 8)
    loads = np.bincount(o8, weights=big, minlength=8)
    assert loads.max() / loads.mean() < 1.01
    assert np.array_equal(o8, pg.lpt_assign(big, 8))  # deterministic


def test_lpt_rejects_bad_args():
    lib = pg.load_library()
    assert lib.pgpcv_lpt_assign(3, None, 2, None) == pg.EINVAL
    c = np.ones(3)
    o = np.empty(3, np.int32)
    assert lib.pgpcv_lpt_assign(3, c.ctypes.data, 0, o.ctypes.data) == pg.EINVAL


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pg.PgpcvError) as ei:
        pg.Context(0)
    assert ei.value.code in (pg.ECUDA, pg.EINVAL)
    lib = pg.load_library()
    assert lib.pgpcv_partition(None, 0, None, None, None, None, pg.Rect(0, 1, 0, 1), 1, 1, 0.0, None) == pg.EINVAL
    assert lib.pgpcv_destroy(None) is None


def test_product_path_does_not_import_oracle():
    """The CUDA path shares no code with the oracle and never routes through it."""
    pkg = os.path.join(ROOT, "paper_1912_13132_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "oracle.c" not in txt, f


def test_max_k_constant_matches_binding_and_library():
    src = open(os.path.join(ROOT, "include", "pgpcv.h")).read()
    hdr = int(re.search(r"#define PGPCV_MAX_K (\d+)", src).group(1))
    internal = open(os.path.join(ROOT, "paper_1912_13132_b200", "csrc", "pgpcv_internal.h")).read()
    assert hdr == pg.MAX_K == int(re.search(r"#define PGPCV_MAX_K_INTERNAL (\d+)", internal).group(1))


def test_nccl_library_reuses_the_loaded_copy():
    """With torch imported, the library binds torch's NCCL (one NCCL per process); the
    report names the path and version (pgpcv_nccl_library)."""
    import subprocess
    import sys
    code = ("import torch, paper_1912_13132_b200 as pg; print(pg.nccl_library())")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = out.stdout.strip()
    assert "libnccl" in line and "(NCCL 2." in line, line
    assert "nvidia/nccl" in line, line


def test_device_math_rejects_bad_args_without_gpu():
    lib = pg.load_library()
    x = np.zeros(4)
    assert lib.pgpcv_device_math(None, 0, 4, x.ctypes.data, x.ctypes.data) == pg.EINVAL
