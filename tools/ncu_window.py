"""Dev: run one C2 solve with the CUDA profiler range opened around a plain
warm iteration (6) and a refresh iteration (10), for
`ncu --profile-from-start off --set full ...`."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
wl = workloads.make(name)
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
rt = torch.cuda.cudart()


def on_iter(it, x):
    if it in (5, 9):
        torch.cuda.synchronize()
        rt.cudaProfilerStart()
    if it in (6, 10):
        torch.cuda.synchronize()
        rt.cudaProfilerStop()


r.run(y, on_iter=on_iter)
torch.cuda.synchronize()
print('done')
