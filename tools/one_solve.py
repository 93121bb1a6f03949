"""Dev: exactly one solve of a configuration (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G
from paper_2301_03047_b200 import workloads
from paper_2301_03047_b200.solvers import GapRunner
name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
wl = workloads.make(name)
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
r.run(y)
torch.cuda.synchronize()
