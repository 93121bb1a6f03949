"""Dev: per-kernel timing on the C2 workload (CUDA events), for iteration."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G
from paper_2301_03047_b200 import workloads, _native as N, _device as D
from paper_2301_03047_b200.solvers import GapRunner

cfgname = sys.argv[1] if len(sys.argv) > 1 else 'C2'
wl = workloads.make(cfgname)
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
x = r.xa
r.dop.adjoint(y, x)
eng = r.eng
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
t_ref = timeit(lambda: eng.refresh(x), 2)
print('n exemplars', eng.n)
h, w, c = wl.shape
out = {'refresh_ms': t_ref}
out['wnnm_scatter_ms'] = timeit(lambda: eng.regularize(x, 0.05), 3)
out['gap_ms'] = timeit(lambda: r.dop.gap_update(eng.acc, eng.cnt, eng.frac, x, y, -0.5, 1.5, r.xb, r.resid_sq[:1], eng.gap_ws))
s = D.stream()
out['corner_resp_ms'] = timeit(lambda: N.call("glr_corner_response", x.data_ptr(), h, w, c, eng.resp.data_ptr(), eng.ws_corner.data_ptr(), s))
out['corners_ms'] = timeit(lambda: N.call("glr_corners", eng.resp.data_ptr(), h, w, wl.match.max_corners, wl.match.nms, 0.01, eng.corners.data_ptr(), eng.n_corners.data_ptr(), eng.ws_nms.data_ptr(), eng.ws_nms.numel(), s))
out['match_ms'] = timeit(lambda: eng.match_shard(), 2)
print(json.dumps(out, indent=1))
