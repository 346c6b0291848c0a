"""Row a8 / (e) on hardware: the library's own world > 1 path (pgpcv_shard + NCCL) with two
ranks on two GPUs (torch.multiprocessing, one process per GPU, gloo only to pass the
ncclUniqueId).  Skips with fewer than 2 GPUs (the round-end GPU box has one).

Alg.1's parfor over subsets and the combine z = sum z_i:
  * gather mode (per-subset arrays requested): every (s, c) entry has one owner, so the
    per-subset losses / likelihoods and loss[] are bit-identical to world 1;
  * vector mode: one all-reduce of the per-config loss vector, within 1e-12 of world 1;
  * the status MIN all-reduce reports the same first failing subset for a non-PD config;
  * predict and GLS at world 2 equal world 1 bit for bit;
  * a rank-local failure on one rank makes the other return ENCCL instead of hanging
    (the error-flag lockstep), and the ctx can be sharded again afterwards.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, shim=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if shim:  # loopback: every rank on cuda:0, the combine through the host-memory shim
        os.environ["PGPCV_NCCL_LIB"] = shim
    import torch
    import torch.distributed as dist

    import paper_1912_13132_b200 as pg
    import workloads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = 0 if shim else rank
    torch.cuda.set_device(dev)
    out = {"nccl_library": pg.nccl_library()}

    def uid():
        obj = [pg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    w = workloads.make("c2", device="cpu")
    params = w.params[[0, 7, 37, 52, 74]]
    X = np.stack([np.ones(w.n), w.x, w.y], 1)
    with pg.Context(dev) as ctx:
        def part():
            ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
        part()
        one = ctx.evaluate(params, nll=True, subset_nll=True)
        part()
        one_vec = ctx.cv_loss(params, want_subset_loss=False).loss
        part()
        one_pred = ctx.predict(params[2:3], target_role=pg.ROLE_TEST)
        part()
        one_gls = ctx.gls(X, params[2])
        # world 2
        part()
        ctx.shard(rank, world, uid())
        two = ctx.evaluate(params, nll=True, subset_nll=True)
        out["gather_subset_loss_equal"] = bool(np.array_equal(two.subset_loss, one.subset_loss))
        out["gather_subset_nll_equal"] = bool(np.array_equal(two.subset_nll, one.subset_nll))
        out["gather_loss_equal"] = bool(np.array_equal(two.loss, one.loss) and np.array_equal(two.nll, one.nll))
        out["my_evals"] = int(ctx.last_timing()["n_evals"])
        vec = ctx.cv_loss(params, want_subset_loss=False).loss
        out["vector_rel_err"] = float(np.max(np.abs(vec - one_vec) / np.abs(one_vec)))
        pr = ctx.predict(params[2:3], target_role=pg.ROLE_TEST)
        out["predict_equal"] = bool(np.array_equal(pr.yhat, one_pred.yhat) and pr.sspe == one_pred.sspe)
        g = ctx.gls(X, params[2])
        out["gls_equal"] = bool(all(np.array_equal(a, b) for a, b in zip(g, one_gls)))
        # a rank-local failure on rank 1: both ranks return, rank 0 with ENCCL
        os.environ["PGPCV_TEST_FAIL_RANK"] = "1"
        try:
            ctx.cv_loss(params)
            out["fault_code"] = 0
        except pg.PgpcvError as e:
            out["fault_code"] = e.code
        del os.environ["PGPCV_TEST_FAIL_RANK"]
        after = ctx.cv_loss(params)  # the communicator survives an agreed failure
        out["after_fault_equal"] = bool(np.array_equal(after.subset_loss, one.subset_loss))
        # non-PD (duplicate sites, zero nugget): the same status as world 1
        xs = np.array([0.1, 0.1, 0.2, 0.8, 0.9, 0.85, 0.3, 0.7])
        ys = np.array([0.1, 0.1, 0.3, 0.8, 0.7, 0.9, 0.6, 0.2])
        vs = np.array([1.0, 2.0, 0.5, 0.3, -0.2, 0.4, 0.1, 0.9])
        rs = np.array([0, 0, 1, 0, 0, 1, 0, 1], np.uint8)
        pp = [[0.2, 1.0, 0.0], [0.2, 1.0, 0.1]]
        ctx.partition(xs, ys, vs, rs, (0, 1, 0, 1), 2, 1, 0.0)
        r1 = ctx.cv_loss(pp)
        ctx.partition(xs, ys, vs, rs, (0, 1, 0, 1), 2, 1, 0.0)
        ctx.shard(rank, world, uid())
        r2 = ctx.cv_loss(pp, want_subset_loss=False)
        out["nonpd_status"] = [r1.status.tolist(), r2.status.tolist()]
        out["nonpd_loss1_equal"] = bool(r1.loss[1] == r2.loss[1] or abs(r1.loss[1] - r2.loss[1]) <= 1e-12 * r1.loss[1])
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([out], dtype=object))
    dist.destroy_process_group()


def _check(outs, library):
    for r, o in enumerate(outs):
        assert library in o["nccl_library"], o["nccl_library"]
        assert o["gather_subset_loss_equal"] and o["gather_subset_nll_equal"] and o["gather_loss_equal"], o
        assert o["vector_rel_err"] <= 1e-12, o
        assert o["predict_equal"] and o["gls_equal"], o
        assert o["after_fault_equal"], o
        assert o["nonpd_status"][0] == o["nonpd_status"][1] and o["nonpd_loss1_equal"], o
    assert outs[0]["my_evals"] > 0 and outs[1]["my_evals"] > 0  # both ranks worked
    import paper_1912_13132_b200 as pg
    assert outs[0]["fault_code"] == pg.ENCCL and outs[1]["fault_code"] == pg.ENOMEM


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs (one rank per GPU)")
def test_two_rank_shard_nccl(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    _check([np.load(tmp_path / f"r{r}.npy", allow_pickle=True)[0] for r in range(2)],
           "nvidia/nccl")  # torch's NCCL reused


def _build_shim(out_dir):
    import subprocess

    from paper_1912_13132_b200._build import _nccl_include
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "nccl_loopback", "loopback_nccl.c")
    lib = os.path.join(out_dir, "libloopback_nccl.so")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-I", _nccl_include(), "-I", "/usr/local/cuda/include",
                           src, "-o", lib, "-ldl", "-lrt"])
    return lib


@pytest.mark.skipif(_ngpu() < 1, reason="needs a GPU")
def test_two_rank_shard_loopback_one_gpu(tmp_path):
    """The same two-rank checks on ONE GPU: both ranks on cuda:0 and the eight NCCL entry
    points bound from tests/nccl_loopback (PGPCV_NCCL_LIB; a host shared-memory all-reduce,
    test infrastructure only).  Everything the library does at world > 1 -- LPT ownership,
    gather and vector combines, the status MIN all-reduce, the error-flag lockstep and
    re-sharding after an agreed failure -- runs on the GPU; only the transport is a stand-in."""
    import torch.multiprocessing as mp
    shim = _build_shim(str(tmp_path))
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), shim), nprocs=2, join=True)
    _check([np.load(tmp_path / f"r{r}.npy", allow_pickle=True)[0] for r in range(2)], "libloopback_nccl.so")
