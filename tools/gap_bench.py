"""Dev: time the fused GAP projection kernel on C2 (CUDA events)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402
wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else 'C2')
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
x = r.xa
r.dop.init_x(y, x)
eng = r.eng
eng.refresh(x)
eng.regularize(x, 0.05)
f = lambda: r.dop.gap_update(eng.acc, eng.cnt, eng.frac, x, y, -0.5, 1.5, r.xb, r.resid_sq[:1], eng.gap_ws)  # noqa
for _ in range(3):
    f()
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    f()
b.record(); torch.cuda.synchronize()
print('gap_update ms', a.elapsed_time(b) / 20)
