"""P2 -- where the cv_kernel's time goes: runs one c5 (or c6) configuration through the
diagnostic build libpgpcv_phases.so (-DPGPCV_PHASE_PROFILE: thread 0 of every CTA
attributes its clock64() time to 15 phases) and prints the phase shares per kernel variant
as JSON.  Usage: python probes/p2_phases.py [c2..c6] [lib]  (PGPCV_SMALL_K selects the split)."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["item_setup", "column_setup", "A_generation", "gemm_issue", "gemm_operand_wait",
         "tile0_barrier", "diag_factor", "diag_store", "trsm_store", "column_end_fence",
         "back_substitution", "predict_outputs", "diag_setup", "diag_panel_warp0", "diag_trailing"]

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1912_13132_b200 as pg
    import workloads
    wname = sys.argv[2]
    w = workloads.make(wname, device="cuda")
    with pg.Context(0) as ctx:
        if w.depth is None:
            ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
        else:
            ctx.partition_bisect(w.x, w.y, w.value, w.role, w.domain, w.depth, w.delta, w.shell_cap, w.cap_seed)
        # P2_STEP=1: the bench's first step (5 grid configs: one range, several lambda --
        # the per-range covariance reuse applies); default one config
        params = w.params[0:5] if os.environ.get("P2_STEP") else np.array([[1.0, 1.0, 0.1]])
        ctx.cv_loss(params, want_subset_loss=False)
        t = ctx.last_timing()
        print("TIMING", json.dumps(t), flush=True)
    sys.exit(0)

wname = sys.argv[1] if len(sys.argv) > 1 else "c5"
lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_1912_13132_b200", "libpgpcv_phases.so")
if not os.path.exists(lib):  # the diagnostic build (not part of __graft_entry__.build())
    sys.path.insert(0, ROOT)
    from paper_1912_13132_b200 import _build
    _build.build(force=True, defines=["PGPCV_PHASE_PROFILE"], out=lib)
env = dict(os.environ, PGPCV_LIB=lib)
r = subprocess.run([sys.executable, __file__, "child", wname], env=env, capture_output=True, text=True)
ms = re.findall(r"PGPCV_PHASES (\{.*\})", r.stderr)
t = re.search(r"TIMING (\{.*\})", r.stdout)
if not ms:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
out = {"workload": wname, "lib": os.path.basename(lib), "timing": json.loads(t.group(1)) if t else None,
       "variants": {}}
for m in ms:  # one line per kernel variant launched (0 large, 1 small)
    d = json.loads(m)
    cyc = d["cycles"]
    tot = sum(cyc)
    out["variants"][{0: "large", 1: "small"}.get(d.get("variant", 0))] = {
        "slots": d["slots"], "share": {n: round(c / tot, 4) for n, c in zip(NAMES, cyc)}}
print(json.dumps(out))
