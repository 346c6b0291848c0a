"""Repeat the full c2 grid on the GPU and count disagreements with the oracle (race hunt)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads, oracle
import paper_1912_13132_b200 as pg
w = workloads.make('c2')
part = oracle.partition(w.x, w.y, w.role, w.domain, w.kx, w.ky, w.delta)
ref = oracle.cv_loss(w.x, w.y, w.value, part, w.params, threads=os.cpu_count())
ctx = pg.Context(0)
ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for r in range(reps):
    res = ctx.cv_loss(w.params)
    bad = ~(np.abs(res.subset_loss - ref.subset_loss) <= 1e-9 * np.abs(ref.subset_loss))
    print(f"rep {r}: bad {int(bad.sum())} nan {int(np.isnan(res.subset_loss).sum())} "
          f"max rel {np.nanmax(np.abs(res.subset_loss - ref.subset_loss) / np.abs(ref.subset_loss)):.2e} "
          f"ms {ctx.last_timing()['kernel_ms']:.2f}", flush=True)
    k = part.k(); m = part.m()
    for (si, ci) in np.argwhere(bad)[:12]:
        print(f"   s={si} c={ci} k={k[si]} m={m[si]} ld={((k[si]+1+15)//16)*16} gpu={res.subset_loss[si,ci]:.6g} ref={ref.subset_loss[si,ci]:.6g}", flush=True)
