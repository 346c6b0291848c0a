#!/usr/bin/env python
"""Parity report ("a parity JSON per config"): GPU path through the C ABI vs the
CPU oracle -- membership bit-exactness and the max relative error of per-subset and global
CV losses.  Writes one JSON object to stdout.  Needs a GPU; the oracle runs on the host
cores (all of them).

Plans:
  sampled  (default) c1..c6: full where the oracle is fast, stratified samples at c4-c6.
  c5_full  c5 at the truth config (grid index 62, (1, 1, 0.1)) over ALL 2,500 subsets with
           the global loss[0] ("all 2,500 subsets x 1 config"), the grid's
           conditioning extremes (c5 #120 = (2, 2, 0.05): lambda 0.025, the largest range;
           c5 #4 = (0.5, 0.5, 0.2): lambda 0.4) on 40 stratified subsets, and c4 #60
           (range 1, lambda 0.0125) on 48 stratified subsets.  ~40 min of oracle time on 16
           cores.
  grids    the WHOLE parameter grid on EVERY subset at c3 (1,600 subsets) and c4 (10,000
           subsets, k up to ~2,000): one representative of each bit-distinct (range, lambda)
           of the grid -- every factorization a whole-grid call executes (R26) -- with the
           global losses.  ~30 min of oracle time on 16 cores.
  c5_corner c5 at the grid's worst-conditioned corner (#120 = (2, 2, 0.05): range 2, lambda
           0.025, kappa ~ 1e5) over ALL 2,500 subsets with the global loss.  ~35 min of oracle.
Any entry beyond 1e-9 is adjudicated with the long-double (x87 80-bit) oracle and reported
with ||e||, m and a kappa estimate; the bar is never loosened."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1912_13132_b200 as pg  # noqa: E402
import workloads  # noqa: E402

THREADS = os.cpu_count() or 8
RTOL = 1e-9


def strat(k, m, n, seed):
    """min-k, max-k, first and last subset, then seeded random subsets with validation data."""
    rng = np.random.default_rng(seed)
    has = np.nonzero(m > 0)[0]
    pick = {int(has[np.argmin(k[has])]), int(has[np.argmax(k[has])]), int(has[0]), int(has[-1])}
    pick |= set(rng.choice(np.setdiff1d(has, list(pick)), size=max(0, n - len(pick)), replace=False).tolist())
    return np.array(sorted(pick))


def _kappa(w, ref_part, s, prm):
    """2-norm condition number of Sigma + lambda I for subset s (numpy eigvalsh; report only)."""
    ti = ref_part.train(s)
    tx, ty = w.x[ti], w.y[ti]
    d = np.sqrt((tx[:, None] - tx[None, :]) ** 2 + (ty[:, None] - ty[None, :]) ** 2)
    a = np.exp(-d / prm[0])
    a[np.diag_indices_from(a)] += prm[2] / prm[1]
    ev = np.linalg.eigvalsh(a)
    return float(ev[-1] / ev[0])


def _adjudicate(w, ref_part, s, prm, g, o):
    ti, vi = ref_part.train(s), ref_part.val(s)
    ld = oracle.subset_cv(w.x[ti], w.y[ti], w.value[ti], w.x[vi], w.y[vi], w.value[vi], *prm, long_double=True)
    return {"subset": int(s), "config": [float(v) for v in prm], "gpu": g, "oracle": o, "oracle_long_double": ld,
            "rel_gpu_vs_ld": abs(g - ld) / abs(ld), "rel_oracle_vs_ld": abs(o - ld) / abs(ld),
            "norm_e": float(np.sqrt(o)), "m": int(vi.size), "k": int(ti.size), "kappa": _kappa(w, ref_part, s, prm)}


def compare(w, ref_part, res, ref, rows, params):
    g, o = res.subset_loss[rows], ref.subset_loss[rows]
    nz = o != 0
    rel = np.where(nz, np.abs(g - o) / np.where(nz, np.abs(o), 1.0), 0.0)
    entry = {"subsets_checked": int(len(rows)), "configs_checked": int(len(params)),
             "entries_checked": int(g.size), "exact_zero_entries_match": bool(np.all(g[~nz] == 0.0)),
             "max_rel_err_subset": float(rel.max()) if rel.size else 0.0,
             "entries_beyond_1e-9": int((rel > RTOL).sum())}
    bad = np.argwhere(rel > RTOL)
    entry["adjudicated"] = [_adjudicate(w, ref_part, int(rows[i]), params[c], float(g[i, c]), float(o[i, c]))
                            for i, c in bad[:10]]
    return entry


def _part(ctx, w):
    if w.depth is None:
        ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
        ref_part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
    else:
        ctx.partition_bisect(w.x, w.y, w.value, w.role, w.domain, w.depth, w.delta, w.shell_cap, w.cap_seed)
        _, rects = oracle.bisect(w.x, w.y, w.role, w.domain, w.depth, w.delta)
        ref_part = oracle.cap_shells(oracle.partition_rects(w.x, w.y, w.role, w.domain, rects, w.delta),
                                     w.x, w.y, w.domain, w.shell_cap, w.cap_seed)
    toff, tidx, voff, vidx = ctx.partition_export()
    member_ok = bool(np.array_equal(toff, ref_part.train_off) and np.array_equal(tidx, ref_part.train_idx)
                     and np.array_equal(voff, ref_part.val_off) and np.array_equal(vidx, ref_part.val_idx))
    return ref_part, member_ok


def plan_sampled(ctx, out):
    plan = {"c1": (None, None), "c2": (None, None), "c3": ([0, 13, 26], None), "c4": ([0, 60, 63], 24),
            "c5": ([4, 62, 120], 8), "c6": ([62], 3)}
    for name, (cfg_idx, nsub) in plan.items():
        t0 = time.time()
        w = workloads.make(name, device="cuda")
        ref_part, member_ok = _part(ctx, w)
        params = w.params if cfg_idx is None else w.params[cfg_idx]
        res = ctx.cv_loss(params)
        sub = None if nsub is None else strat(ref_part.k(), ref_part.m(), nsub, 7)
        ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, params, subsets=sub, threads=THREADS)
        rows = np.arange(ref_part.n_subsets) if sub is None else sub
        entry = {"membership_bit_exact": member_ok, "subsets": int(ref_part.n_subsets),
                 "config_indices": cfg_idx if cfg_idx is not None else "all",
                 **compare(w, ref_part, res, ref, rows, params),
                 "k_range": [int(ref_part.k().min()), int(ref_part.k().max())]}
        if sub is None:
            entry["max_rel_err_global"] = float(np.max(np.abs(res.loss - ref.loss) / np.abs(ref.loss)))
        entry["seconds"] = round(time.time() - t0, 1)
        out["configs"][name] = entry
        print(name, json.dumps(entry), file=sys.stderr, flush=True)


def plan_c5_full(ctx, out):
    w = workloads.make("c5", device="cuda")
    ref_part, member_ok = _part(ctx, w)
    k, m = ref_part.k(), ref_part.m()
    # (a) all 2,500 subsets at the truth, and the global loss
    t0 = time.time()
    p = w.params[[62]]
    res = ctx.cv_loss(p)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, p, threads=THREADS)
    e = {"membership_bit_exact": member_ok, "config_index": 62, "config": p[0].tolist(),
         **compare(w, ref_part, res, ref, np.arange(ref_part.n_subsets), p),
         "loss_gpu": float(res.loss[0]), "loss_oracle": float(ref.loss[0]),
         "rel_err_global": float(abs(res.loss[0] - ref.loss[0]) / abs(ref.loss[0])),
         "k_range": [int(k.min()), int(k.max())], "m_range": [int(m.min()), int(m.max())],
         "seconds": round(time.time() - t0, 1)}
    out["configs"]["c5_truth_all_subsets"] = e
    print("c5 all", json.dumps(e), file=sys.stderr, flush=True)
    # (b) conditioning extremes of the c5 grid on 40 stratified subsets
    t0 = time.time()
    idx = [4, 120]
    p = w.params[idx]
    res = ctx.cv_loss(p)
    sub = strat(k, m, 40, 11)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, p, subsets=sub, threads=THREADS)
    e = {"config_indices": idx, "configs": p.tolist(), **compare(w, ref_part, res, ref, sub, p),
         "kappa_max_k_subset": {str(i): _kappa(w, ref_part, int(sub[np.argmax(k[sub])]), p[j])
                                for j, i in enumerate(idx)},
         "seconds": round(time.time() - t0, 1)}
    out["configs"]["c5_extremes_40_subsets"] = e
    print("c5 extremes", json.dumps(e), file=sys.stderr, flush=True)
    # (c) c4's worst corner on 48 stratified subsets (and the empty-validation zeros)
    t0 = time.time()
    w4 = workloads.make("c4", device="cuda")
    rp4, ok4 = _part(ctx, w4)
    p = w4.params[[60]]
    res = ctx.cv_loss(p)
    sub = strat(rp4.k(), rp4.m(), 48, 13)
    ref = oracle.cv_loss(w4.x, w4.y, w4.value, rp4, p, subsets=sub, threads=THREADS)
    e = {"membership_bit_exact": ok4, "config_index": 60, "config": p[0].tolist(),
         **compare(w4, rp4, res, ref, sub, p),
         "empty_validation_zeros": bool(np.all(res.subset_loss[rp4.m() == 0] == 0.0)),
         "seconds": round(time.time() - t0, 1)}
    out["configs"]["c4_cfg60_48_subsets"] = e
    print("c4 #60", json.dumps(e), file=sys.stderr, flush=True)


def plan_c5_corner(ctx, out):
    w = workloads.make("c5", device="cuda")
    ref_part, member_ok = _part(ctx, w)
    k, m = ref_part.k(), ref_part.m()
    t0 = time.time()
    p = w.params[[120]]
    res = ctx.cv_loss(p)
    ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, p, threads=THREADS)
    big = int(np.argmax(k))
    e = {"membership_bit_exact": member_ok, "config_index": 120, "config": p[0].tolist(),
         **compare(w, ref_part, res, ref, np.arange(ref_part.n_subsets), p),
         "loss_gpu": float(res.loss[0]), "loss_oracle": float(ref.loss[0]),
         "rel_err_global": float(abs(res.loss[0] - ref.loss[0]) / abs(ref.loss[0])),
         "kappa_max_k_subset": _kappa(w, ref_part, big, p[0]),
         "k_range": [int(k.min()), int(k.max())], "m_range": [int(m.min()), int(m.max())],
         "seconds": round(time.time() - t0, 1)}
    out["configs"]["c5_cfg120_all_subsets"] = e
    print("c5 #120 all", json.dumps(e), file=sys.stderr, flush=True)


def plan_grids(ctx, out):
    for name in ("c3", "c4"):
        t0 = time.time()
        w = workloads.make(name, device="cuda")
        ref_part, member_ok = _part(ctx, w)
        # one representative per bit-distinct (range, lambda = nugget / sigma2) (R26)
        zeta = np.stack([w.params[:, 0], w.params[:, 2] / w.params[:, 1]], axis=1)
        _, rep = np.unique(zeta, axis=0, return_index=True)
        rep = np.sort(rep)
        params = np.ascontiguousarray(w.params[rep])
        res = ctx.cv_loss(params)
        ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, params, threads=THREADS)
        lam = params[:, 2] / params[:, 1]
        entry = {"membership_bit_exact": member_ok, "subsets": int(ref_part.n_subsets),
                 "grid_configs": int(len(w.params)), "distinct_range_lambda": int(len(rep)),
                 "config_indices": rep.tolist(),
                 "range_minmax": [float(params[:, 0].min()), float(params[:, 0].max())],
                 "lambda_minmax": [float(lam.min()), float(lam.max())],
                 **compare(w, ref_part, res, ref, np.arange(ref_part.n_subsets), params),
                 "max_rel_err_global": float(np.max(np.abs(res.loss - ref.loss) / np.abs(ref.loss))),
                 "status_all_ok": bool(np.all(res.status == -1)),
                 "k_range": [int(ref_part.k().min()), int(ref_part.k().max())],
                 "seconds": round(time.time() - t0, 1)}
        out["configs"][name + "_whole_grid_all_subsets"] = entry
        print(name, json.dumps(entry), file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="sampled", choices=["sampled", "c5_full", "grids", "c5_corner"])
    args = ap.parse_args()
    out = {"tolerance": "per-subset and global loss |g - o| <= 1e-9 |o|; membership bit-exact",
           "plan": args.plan, "oracle_threads": THREADS, "configs": {}}
    with pg.Context(0) as ctx:
        {"c5_full": plan_c5_full, "grids": plan_grids, "c5_corner": plan_c5_corner, "sampled": plan_sampled}[args.plan](ctx, out)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
