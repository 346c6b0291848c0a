#!/usr/bin/env python
"""Parity report ("a parity JSON per config"): GPU path through the C ABI vs the
CPU oracle on c1..c6 -- membership bit-exactness and the max relative error of per-subset and
global CV losses (full where the oracle is fast, stratified samples at c4-c6).  Writes one
JSON object to stdout.  Needs a GPU; the oracle runs on the host cores."""
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


def strat(k, m, n, seed):
    rng = np.random.default_rng(seed)
    has = np.nonzero(m > 0)[0]
    pick = {int(has[np.argmin(k[has])]), int(has[np.argmax(k[has])])}
    pick |= set(rng.choice(has, size=max(0, n - len(pick)), replace=False).tolist())
    return np.array(sorted(pick))


def main():
    out = {"tolerance": "per-subset and global loss |g - o| <= 1e-9 |o|; membership bit-exact", "configs": {}}
    plan = {"c1": (None, None), "c2": (None, None), "c3": ([0, 13, 26], None), "c4": ([0, 63], 24),
            "c5": ([62], 8), "c6": ([62], 3)}
    with pg.Context(0) as ctx:
        for name, (cfg_idx, nsub) in plan.items():
            t0 = time.time()
            w = workloads.make(name, device="cuda")
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
            params = w.params if cfg_idx is None else w.params[cfg_idx]
            res = ctx.cv_loss(params)
            sub = None if nsub is None else strat(ref_part.k(), ref_part.m(), nsub, 7)
            ref = oracle.cv_loss(w.x, w.y, w.value, ref_part, params, subsets=sub, threads=THREADS)
            rows = np.arange(ref_part.n_subsets) if sub is None else sub
            g, o = res.subset_loss[rows], ref.subset_loss[rows]
            nz = o != 0
            rel = np.abs(g[nz] - o[nz]) / np.abs(o[nz])
            entry = {"membership_bit_exact": member_ok, "subsets": int(ref_part.n_subsets),
                     "configs_checked": int(len(params)), "subsets_checked": int(len(rows)),
                     "entries_checked": int(g.size), "exact_zero_entries_match": bool(np.all(g[~nz] == 0.0)),
                     "max_rel_err_subset": float(rel.max()) if rel.size else 0.0,
                     "k_range": [int(ref_part.k().min()), int(ref_part.k().max())], "seconds": round(time.time() - t0, 1)}
            if sub is None:
                entry["max_rel_err_global"] = float(np.max(np.abs(res.loss - ref.loss) / np.abs(ref.loss)))
            out["configs"][name] = entry
            print(name, json.dumps(entry), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
