import sys
import torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G
from paper_2301_03047_b200 import workloads
from paper_2301_03047_b200.solvers import GapRunner
name = sys.argv[1] if len(sys.argv) > 1 else 'C4'
wl = workloads.make(name)
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
snaps = []
def on_iter(it, x):
    snaps.append((x.data_ptr(), float(x.double().abs().sum()), float((x.double() ** 2).sum())))
xf = r.run(y, on_iter=on_iter)
torch.cuda.synchronize()
for i, s in enumerate(snaps):
    print(i, s)
print('resid', r.resid_sq[:wl.max_iters].tolist())
print('scene', wl.scene.shape, 'x', tuple(xf.shape), 'cfg.init', cfg.init)
