"""P3 -- do the two CTAs of an SM leave the update at the same time?  Runs one c5
configuration through the diagnostic timeline build (probes/libpgpcv_timeline.so:
-DPGPCV_PHASE_PROFILE -DPGPCV_TIMELINE; thread 0 of every CTA logs each switch between the
DMMA update and everything else, on the SM clock) and reports, per SM, the share of time
with both / one / no CTA in the update next to what independent CTAs would give."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LEN = 1 << 15

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import paper_1912_13132_b200 as pg
    import workloads
    w = workloads.make(sys.argv[2], device="cuda")
    with pg.Context(0) as ctx:
        ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
        ctx.cv_loss(np.array([[1.0, 1.0, 0.1]]), want_subset_loss=False)
    sys.exit(0)

wname = sys.argv[1] if len(sys.argv) > 1 else "c5"
lib = os.path.join(ROOT, "probes", "libpgpcv_timeline.so")
if not os.path.exists(lib):
    sys.path.insert(0, ROOT)
    from paper_1912_13132_b200 import _build
    _build.build(force=True, defines=["PGPCV_PHASE_PROFILE", "PGPCV_TIMELINE"], out=lib)
path = "/tmp/pgpcv_timeline.bin"
env = dict(os.environ, PGPCV_LIB=lib, PGPCV_TIMELINE_FILE=path)
r = subprocess.run([sys.executable, __file__, "child", wname], env=env, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
raw = np.fromfile(path, np.uint64).reshape(-1, LEN)
by_sm = {}
for cta, row in enumerate(raw):
    n = int(row[1])
    if n < 4:
        continue
    ev = row[2:2 + n]
    by_sm.setdefault(int(row[0]), []).append(((ev >> np.uint64(1)).astype(np.int64), (ev & np.uint64(1)).astype(np.int8)))
stats = []
for sm, ctas in sorted(by_sm.items()):
    if len(ctas) != 2:
        continue
    t0 = max(c[0][0] for c in ctas)
    t1 = min(c[0][-1] for c in ctas)
    if t1 <= t0:
        continue
    grid = np.linspace(t0, t1, 200_000)
    states = []
    for times, st in ctas:
        idx = np.searchsorted(times, grid, side="right") - 1
        states.append(st[np.clip(idx, 0, len(st) - 1)])
    a, b = states
    p_a, p_b = a.mean(), b.mean()
    stats.append({"sm": sm, "gemm_share_cta0": float(p_a), "gemm_share_cta1": float(p_b),
                  "both_in_update": float(np.mean(a & b)), "neither": float(np.mean((1 - a) & (1 - b))),
                  "neither_if_independent": float((1 - p_a) * (1 - p_b))})
agg = {k: float(np.mean([s[k] for s in stats])) for k in stats[0] if k != "sm"} if stats else {}
print(json.dumps({"workload": wname, "sms_analysed": len(stats), "mean": agg, "per_sm": stats[:8]}, indent=1))
