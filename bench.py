#!/usr/bin/env python
"""Benchmark of the parallel-CV hot path (BASELINE.json metric: subset CV-loss evals/sec and
sec per parameter configuration at 5M points; FP64 % of peak).

A "step" is one pass of the whole hot path (Alg.1 lines 4-9) over all
2,500 subsets of the 5M-point workload c5 for a batch of `--configs-per-step` (default 5)
(range, sigma2, nugget) configurations of its 125-point grid (steps walk through the grid):
covariance assembly, FP64 Cholesky, solves, prediction, loss reduction (and the NCCL
combine when N > 1).  `--configs-per-step 125` streams the whole grid through one call
(bit-identical (range, lambda) pairs are then factored once; `configs_executed`).
The partition (Alg.1 lines 2-3, "done once") happens before the timed region for
`value`, and inside every step for `e2e` (host arrays -> C ABI -> host loss).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1..c6] [--mode cv|cv_nll|nll|predict|gls]

N > 1: launched by torchrun (one rank per GPU), or, without WORLD_SIZE in the environment,
bench.py launches torchrun itself; times are CUDA-event times, max over ranks.
`--impl reference` times the CPU oracle (the reference arm of this tier) on rank 0.
`--dry-run` exercises the multi-rank launch and combine on CPU (gloo, no GPU).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ncu --set full capture of the dominant kernel (dram bytes per launch -> roofline.traffic)
PROFILE_JSON = "r02e_cv_kernel_c5_ncu.json"
METRIC = "subset CV-loss evals/sec at 5M pts (sec per param config and FP64 % of peak alongside)"
METRICS = {"cv": METRIC,
           "cv_nll": "subset CV-loss + -2 log-lik evals/sec (one factorization per subset and config)",
           "nll": "subset -2 log-likelihood evals/sec",
           "predict": "subset test-set kriging evals/sec (one config per step)",
           "gls": "subset GLS normal-equation evals/sec (covariates 1, x, y; one config per step)"}
# Configurations per step: a grid search streams the configurations through one call
# (pgpcv_cv_loss(params[], n_params)); 5 per step gives 12,500 (subset, config)
# items at c5, so the dynamic schedule's last partial wave stays small at 1-8 GPUs.
CONFIGS_PER_STEP = 5
UNIT = "subset-evals/s"


def _env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region,
    plus one synchronous snapshot when it starts and one when it stops (so a timed region
    shorter than the sampling period still has a clock record)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def _snapshot(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            self.lines.extend(ln.strip() for ln in out.stdout.splitlines() if ln.strip())
        except (OSError, subprocess.TimeoutExpired):
            pass

    def start(self):
        self._snapshot()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self._snapshot()
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm, smax, power, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _peaks():
    """FP64 peak (the denominator): P0's measured DMMA number (profiles/r01_p0_fp64_peak.json),
    with the bf16-derived figure (MEASURED_PEAKS.json x nominal FP64/BF16 ratio) beside it."""
    p0 = os.path.join(ROOT, "profiles", "r01_p0_fp64_peak.json")
    meas = None
    if os.path.exists(p0):
        meas = json.load(open(p0)).get("dmma_tflops_sustained")
    derived = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        bf16 = json.load(open(mp)).get("bf16_tflops_sustained")
        if bf16:
            derived = bf16 * 45.0 / 2250.0  # guide: B200 FP64 tensor 45 TF vs bf16 2.25 PF dense
    return meas, derived


def _traffic(configs):
    """DRAM bytes (read + write) of one cv_kernel launch over `configs` configurations: the
    ncu --set full capture of a one-configuration c5 launch, scaled (every configuration
    factors every subset once, so the traffic is linear in the configurations)."""
    f = os.path.join(ROOT, "profiles", PROFILE_JSON)
    if os.path.exists(f):
        try:
            d = json.load(open(f))
            per = d.get("dram_bytes_per_config", d.get("dram_bytes_per_launch"))
            return per * configs if per is not None else None
        except Exception:
            return None
    return None


def _stratified_sample(k, m, count, seed=5):
    rng = np.random.default_rng(seed)
    has = np.nonzero(m > 0)[0]
    order = has[np.argsort(k[has], kind="stable")]
    pick = set(order[np.linspace(0, order.size - 1, min(count, order.size)).astype(int)].tolist())
    while len(pick) < min(count, has.size):
        pick.add(int(rng.choice(has)))
    return np.array(sorted(pick))


def run_reference(args, rank, world):
    """The reference arm of this tier: the CPU oracle (oracle/) as it stands, timed on the
    host cores, on the same workload/metric; rank 0 only."""
    if rank != 0:
        return 0
    import workloads

    dev = "cuda" if _has_cuda() else "cpu"
    w = workloads.make(args.workload, device=dev)
    part = _oracle_partition(w, core_role=2 if args.mode == "predict" else 1)
    k, m = part.k(), part.m()
    cores = os.cpu_count() or 1
    sample = _stratified_sample(k, m, cores)
    t_total, evals = 0.0, 0
    for step in range(args.warmup + args.steps):
        p = w.params[step % len(w.params)][None, :]
        t0 = time.perf_counter()
        _oracle_step(w, part, p, sample, cores, args.mode)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            t_total += dt
            evals += sample.size
    value = evals / t_total
    desc = (f"{sample.size} stratified {args.workload} subsets (k {int(k[sample].min())}-"
            f"{int(k[sample].max())}) x 1 config per step, oracle.c (-O2, no FMA) as it stands")
    line = {
        "impl": "reference", "metric": METRICS[args.mode], "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(args, w, part),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _has_cuda():
    import torch
    return torch.cuda.is_available()


def _config(args, w, part_or_info):
    if isinstance(part_or_info, dict):
        N, nv = part_or_info["n_subsets"], part_or_info["n_val"]
    else:
        N, nv = part_or_info.n_subsets, int(part_or_info.m().sum())
    div = (f"{w.kx}x{w.ky} tiles" if w.depth is None else
           f"recursive bisection into 2^{w.depth} subsets, shell cap {w.shell_cap}")
    mode = {"cv": "", "cv_nll": ", CV loss + per-subset -2 log-lik (one factorization)",
            "nll": ", per-subset -2 log-lik only", "predict": ", test-set kriging prediction",
            "gls": ", GLS mean estimate with covariates (1, x, y)"}[args.mode]
    return {"workload": f"{args.workload}: n={w.n:,} on [{w.domain[0]:g},{w.domain[1]:g}]^2, "
                        f"{div}, delta={w.delta:g}, {len(w.params)}-config grid "
                        f"({_cps(args)} config(s) per step){mode}, FP64",
            "n_points": w.n, "n_subsets": N, "n_val": nv, "grid_configs": len(w.params),
            "configs_per_step": _cps(args),
            "parallelism": f"whole subsets sharded by LPT on k^3 over {args.gpus} GPU(s), one rank per GPU",
            "l2": "no flush: per-step factor working set (296 slots x up to 73 MB) >> 126 MB L2"}


def _cps(args):
    return 1 if args.mode in ("predict", "gls") else args.configs_per_step


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1912_13132_b200 as pg
    import workloads

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    w = workloads.make(args.workload, device="cuda")
    C = len(w.params)
    # inputs resident in HBM (value) and pinned host copies (e2e)
    dx = torch.as_tensor(w.x, device="cuda")
    dy = torch.as_tensor(w.y, device="cuda")
    dv = torch.as_tensor(w.value, device="cuda")
    dr = torch.as_tensor(w.role, device="cuda")
    hx, hy, hv, hr = (torch.as_tensor(a).pin_memory().numpy() for a in (w.x, w.y, w.value, w.role))

    ctx = pg.Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    def part_device():
        if w.depth is None:
            return ctx.partition_device(dx, dy, dv, dr, w.domain, w.kx, w.ky, w.delta)
        return ctx.partition_bisect_device(dx, dy, dv, dr, w.domain, w.depth, w.delta, w.shell_cap, w.cap_seed)

    def part_host():
        if w.depth is None:
            return ctx.partition(hx, hy, hv, hr, w.domain, w.kx, w.ky, w.delta)
        return ctx.partition_bisect(hx, hy, hv, hr, w.domain, w.depth, w.delta, w.shell_cap, w.cap_seed)

    info = part_device()
    # Alg.1 lines 2-3 (done once per dataset): timed on a second call (allocations warm)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    info = part_device()
    p1.record(stream)
    torch.cuda.synchronize()
    partition_ms = p0.elapsed_time(p1)
    uid = None
    if world > 1:
        obj = [pg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx.shard(rank, world, uid)
    toff, _, voff, _ = ctx.partition_export()
    goff, _ = ctx.partition_export_test()
    kk, mm, gg = np.diff(toff), np.diff(voff), np.diff(goff)
    # (subset, config) evaluations per step over all ranks: subsets with validation data
    # (cv), every subset (the likelihood needs no targets), subsets with test points (predict)
    cps = _cps(args)
    evals_per_step = cps * {"cv": int((mm > 0).sum()), "cv_nll": int(kk.size), "nll": int(kk.size),
                            "predict": int((gg > 0).sum()), "gls": int((kk > 0).sum())}[args.mode]
    X = None
    if args.mode == "gls":  # covariates of the paper's extended model: 1, x, y (scaled)
        X = np.stack([np.ones(w.n), w.x / w.domain[1], w.y / w.domain[3]], 1)

    def step(i):
        p = w.params[[(i * cps + q) % C for q in range(cps)]]
        if args.mode == "cv":
            return ctx.cv_loss(p, want_subset_loss=False).loss[0]
        if args.mode == "cv_nll":
            return ctx.evaluate(p, subset_loss=False, nll=True).loss[0]
        if args.mode == "nll":
            return ctx.evaluate(p, loss=False, subset_loss=False, nll=True).nll[0]
        if args.mode == "gls":
            return ctx.gls(X, p[0])[0][0]
        return ctx.predict(p, want_yhat=False).sspe

    for i in range(args.warmup):
        step(i)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern_ms, kern_flops, launches, losses, executed = 0.0, 0.0, 0, [], 0
    e0.record(stream)
    for i in range(args.steps):
        r = step(args.warmup + i)
        t = ctx.last_timing()
        kern_ms += t["kernel_ms"]
        kern_flops += t["flops"]
        launches += t["launches"]
        executed += t["n_configs_executed"]
        losses.append(float(r))
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())

    # e2e: host arrays through the public API every step (H2D of the points, partition,
    # cv_loss, D2H of the loss); timed with events around synchronous calls.
    barrier()
    ctx.set_stream(stream.cuda_stream)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for i in range(args.steps):
        part_host()
        step(args.warmup + i)
    f1.record(stream)
    barrier()
    e2e_ms = f0.elapsed_time(f1)
    if dist:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    # dominant kernel roofline (FP64 tensor path), this rank's launches
    achieved = kern_flops / (kern_ms * 1e-3) / 1e12 if kern_ms > 0 else 0.0
    peak, derived = _peaks()
    value = evals_per_step * args.steps / (t_ms * 1e-3)
    n = w.n
    line = {
        "metric": METRICS[args.mode], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, w, info),
        "sec_per_config": t_ms / args.steps / 1e3 / cps,
        "configs_per_step": cps,
        "configs_executed_per_step": executed / args.steps,
        "fp64_pct_of_peak": 100.0 * achieved / peak if peak else None,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": _traffic(executed / args.steps) if args.workload == "c5" and args.mode == "cv" else None,
                     "kernel": "cv_kernel (assembly + DMMA Cholesky + solves + prediction + SSPE)",
                     "kernel_ms_per_launch": kern_ms / args.steps,
                     "flops_per_launch": kern_flops / args.steps,
                     "peak_source": "measured FP64 DMMA, probes/p0_fp64_peak (profiles/r01_p0_fp64_peak.json)",
                     "peak_bf16_derived": derived},
        "e2e": {"value": evals_per_step * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": int(n * (8 * 3 + 1) + 24 * cps), "d2h_bytes_per_step": 12 * cps},
        "gpu_launches": launches,
        "clocks": clk,
        "subset_k": {"min": int(kk[mm > 0].min()), "median": float(np.median(kk[mm > 0])),
                     "max": int(kk.max())},
        "loss_first_step": losses[0],
        "partition_ms_once_per_dataset": partition_ms,
    }
    if world > 1:
        line["nccl_library"] = pg.nccl_library()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(w, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


def _oracle_partition(w, core_role=1):
    """The oracle's own membership (independent of the GPU): brute-force tiles, or the
    oracle's bisection + rectangle membership + shell cap for c6."""
    import oracle

    if w.depth is None:
        return oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta, core_role=core_role)
    _, rects = oracle.bisect(w.x, w.y, w.role, w.domain, w.depth, w.delta)
    part = oracle.partition_rects(w.x, w.y, w.role, w.domain, rects, w.delta, core_role=core_role)
    return oracle.cap_shells(part, w.x, w.y, w.domain, w.shell_cap, w.cap_seed) if w.shell_cap >= 0 else part


def _oracle_step(w, part, p, sample, cores, mode):
    """One bounded oracle step of the bench's mode on `sample` subsets."""
    import oracle

    if mode in ("cv", "cv_nll"):
        oracle.cv_loss(w.x, w.y, w.value, part, p, subsets=sample, threads=cores)
    if mode in ("cv_nll", "nll"):
        oracle.neg2loglik_all(w.x, w.y, w.value, part, p, subsets=sample, threads=cores)
    if mode == "gls":
        import oracle as _o
        if w.depth is None:
            ex, ey = _o.edges(w.domain[0], w.domain[1], w.kx), _o.edges(w.domain[2], w.domain[3], w.ky)
            rects = np.array([[ex[i], ex[i + 1], ey[j], ey[j + 1]] for j in range(w.ky) for i in range(w.kx)])
        else:
            rects = part.rects
        X = np.stack([np.ones(w.n), w.x / w.domain[1], w.y / w.domain[3]], 1)
        oracle.gls(w.x, w.y, w.value, X, part, rects, w.domain, p[0], subsets=sample, threads=cores)
    if mode == "predict":  # part holds the test lists as its core lists
        sub = oracle.Partition(part.train_off, part.train_idx, part.val_off, part.val_idx, part.n_subsets, 1)
        keep = np.zeros(part.n_subsets, bool)
        keep[sample] = True
        oracle.cv_loss(w.x, w.y, w.value, sub, p, subsets=np.nonzero(keep)[0], threads=cores)


def _cpu_baseline(w, args):
    """The oracle as it stands on the host cores: a bounded sample of the same workload
    (one subset per core x 1 config, ~15 s at c5), scaled to evals/s."""
    part = _oracle_partition(w, core_role=2 if args.mode == "predict" else 1)
    cores = os.cpu_count() or 1
    sample = _stratified_sample(part.k(), part.m(), cores)
    p = w.params[args.warmup % len(w.params)][None, :]
    t0 = time.perf_counter()
    _oracle_step(w, part, p, sample, cores, args.mode)
    dt = time.perf_counter() - t0
    out = {"value": sample.size / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{sample.size} stratified {args.workload} subsets x 1 config "
                     f"(k {int(part.k()[sample].min())}-{int(part.k()[sample].max())}), "
                     f"{dt:.1f} s on {cores} threads"}
    if args.mode == "cv":
        out["lapack_context"] = _lapack_baseline(w, part, sample, p[0])
    return out


def _lapack_baseline(w, part, sample, prm):
    """Context only: the same sample with LAPACK through scipy (cho_factor /
    cho_solve on the host's threaded BLAS) -- a strong CPU implementation of Eq.3-4, not
    the oracle and not a parity reference."""
    import scipy.linalg

    theta, lam = float(prm[0]), float(prm[2]) / float(prm[1])
    t0 = time.perf_counter()
    for s in sample:
        ti, vi = part.train(s), part.val(s)
        tx, ty, tv = w.x[ti], w.y[ti], w.value[ti]
        d = np.sqrt((tx[:, None] - tx[None, :]) ** 2 + (ty[:, None] - ty[None, :]) ** 2)
        A = np.exp(-d / theta)
        A[np.diag_indices_from(A)] += lam
        alpha = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A, lower=True, overwrite_a=True), tv)
        dv = np.sqrt((w.x[vi][:, None] - tx[None, :]) ** 2 + (w.y[vi][:, None] - ty[None, :]) ** 2)
        e = np.exp(-dv / theta) @ alpha - w.value[vi]
        float(e @ e)
    dt = time.perf_counter() - t0
    return {"value": sample.size / dt, "unit": UNIT, "kind": "scipy/LAPACK cho_factor (threaded BLAS), same sample",
            "seconds": dt}


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int:
    """--gpus N without a torchrun environment: run this script under torchrun, one rank
    per GPU on this node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args, rank, world, local_rank):
    """Multi-rank plumbing without a GPU: gloo process group, the library's LPT ownership
    rule over c5-sized synthetic subsets, the max-over-ranks timing reduction; rank 0 prints
    one JSON line naming every rank it saw."""
    import torch
    import torch.distributed as dist

    import paper_1912_13132_b200 as pg

    if world > 1:
        dist.init_process_group("gloo")
    k = np.random.default_rng(0).integers(2600, 4300, 2500).astype(np.float64)
    owner = pg.lpt_assign(k ** 3, world)
    mine = int((owner == rank).sum())
    me = torch.tensor([rank, local_rank, world, os.getpid(), mine], dtype=torch.float64)
    rows = [me.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(rows, me)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "ranks": [[int(v) for v in r.tolist()] for r in rows],
                          "subsets_per_rank": [int(r[4]) for r in rows]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "c6"])
    ap.add_argument("--mode", default="cv", choices=["cv", "cv_nll", "nll", "predict", "gls"],
                    help="cv: the headline CV loss; cv_nll / nll: row f3; predict: row f1 test-set kriging")
    ap.add_argument("--configs-per-step", type=int, default=CONFIGS_PER_STEP)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank launch/combine on CPU (gloo), no GPU")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to run", file=sys.stderr)
        return 2
    if args.dry_run:
        return run_dry(args, rank, world, local_rank)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    if torch.cuda.device_count() < world:
        print(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s); refusing to run",
              file=sys.stderr)
        return 2
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
