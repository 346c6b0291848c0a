"""Multi-rank host logic of the sharded path on CPU (world_size 2, gloo, 127.0.0.1).

After pgpcv_shard every CV evaluation assigns the whole subsets it factors (those with
validation data) to ranks by LPT on k^3 (the library's pgpcv_lpt_assign, host-only, over
those subsets in ascending id) and the combine step (Alg.1 line 9) all-reduces either the per-config
loss vector or the per-subset array (each entry with one owner).  Here each rank computes
its owned subsets with the CPU oracle and the same two all-reduces run over gloo; the
result must equal the single-process evaluation (bit-exact for the per-subset array)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    import workloads
    w = workloads.make("c2", n=3000)
    return w


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_1912_13132_b200 as pg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _data()
    part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    k, m = part.k().astype(np.float64), part.m()
    ids = np.nonzero(m > 0)[0]
    owner = np.full(part.n_subsets, -1, np.int32)
    owner[ids] = pg.lpt_assign(k[ids] ** 3, world)  # the C ABI's host-only LPT rule
    mine = np.nonzero((owner == rank) & (m > 0))[0]
    params = w.params[[0, 37, 74]]
    rep = oracle.cv_loss(w.x, w.y, w.value, part, params, subsets=mine, threads=2)
    sub = np.zeros((part.n_subsets, len(params)))
    sub[mine] = rep.subset_loss[mine]
    own = torch.zeros(part.n_subsets, dtype=torch.float64)
    own[torch.as_tensor(mine)] = 1.0
    dist.all_reduce(own)
    t_loss = torch.as_tensor(sub.sum(axis=0))  # this rank's partial C~V per config
    dist.all_reduce(t_loss)                    # loss-vector combine
    t_sub = torch.as_tensor(sub.copy())
    dist.all_reduce(t_sub)                     # per-subset combine (deterministic mode)
    np.save(os.path.join(out_dir, f"r{rank}_sub.npy"), t_sub.numpy())
    np.save(os.path.join(out_dir, f"r{rank}_loss.npy"), t_loss.numpy())
    np.save(os.path.join(out_dir, f"r{rank}_own.npy"), own.numpy())
    np.save(os.path.join(out_dir, f"r{rank}_owner.npy"), owner)
    dist.destroy_process_group()


def test_two_rank_shard_and_combine(tmp_path):
    import oracle

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = _data()
    part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    params = w.params[[0, 37, 74]]
    ref = oracle.cv_loss(w.x, w.y, w.value, part, params, threads=4)
    m = part.m()
    for r in range(world):
        own = np.load(tmp_path / f"r{r}_own.npy")
        assert np.all(own[m > 0] == 1.0)                    # every subset owned exactly once
        sub = np.load(tmp_path / f"r{r}_sub.npy")
        assert np.array_equal(sub[m > 0], ref.subset_loss[m > 0])   # bit-exact per subset
        loss = np.load(tmp_path / f"r{r}_loss.npy")
        np.testing.assert_allclose(loss, ref.loss, rtol=1e-12)
    o0, o1 = np.load(tmp_path / "r0_owner.npy"), np.load(tmp_path / "r1_owner.npy")
    assert np.array_equal(o0, o1)                           # identical on every rank
    k = part.k().astype(float)
    loads = np.bincount(o0[m > 0], weights=k[m > 0] ** 3, minlength=2)
    assert loads.max() / loads.sum() < 0.52                 # LPT balance on k^3
