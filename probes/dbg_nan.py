import os, sys, numpy as np
sys.path.insert(0, '.')
import workloads, oracle
w = workloads.make('c2')
import subprocess
for slots in sys.argv[1:]:
    os.environ['PGPCV_MAX_SLOTS'] = slots
    import paper_1912_13132_b200 as pg
    ctx = pg.Context(0)
    ctx.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    r = ctx.cv_loss(w.params[:3])
    print('slots', slots, 'nan', np.isnan(r.subset_loss).sum(), 'status', r.status, 'code', r.code, 'timing', ctx.last_timing(), flush=True)
    print(r.subset_loss[:6].tolist(), flush=True)
    ctx.close()
