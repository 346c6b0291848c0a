# GPU: compute-sanitizer (memcheck / racecheck / synccheck) on small runs through the C ABI,
# and the parity report
set -x
cat > /tmp/san_run.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1912_13132_b200 as pg, workloads
w = workloads.make("c2", n=3000)
with pg.Context(0) as c:
    c.partition(w.x, w.y, w.value, w.role, w.domain, w.kx, w.ky, w.delta)
    r = c.evaluate(w.params[:2], nll=True, subset_nll=True)
    c.select(); c.predict(w.params[:1], target_role=pg.ROLE_VALIDATION)
    c.partition_bisect(w.x, w.y, w.value, w.role, w.domain, 3, 0.05, 20, 7)
    c.cv_loss(w.params[:1])
    X = np.stack([np.ones(w.n), w.x], 1); c.gls(X, w.params[0])
    x, y, v, role = workloads.random_points(5, 200, frac_val=0.1)
    c.partition(x, y, v, role, (0, 1, 0, 1), 1, 1, 0.0); c.cv_loss([[0.2, 1.0, 0.1]])
print("ran", float(r.loss[0]))
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_run.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "rc $?" >> gpurun_out/sanitizer_$tool.log
done
timeout 2400 python scripts/parity_report.py > gpurun_out/parity.json 2> gpurun_out/parity.err
echo done
