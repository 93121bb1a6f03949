"""Dev: how often the top-K cut falls below L (needs GLR_NVCC_EXTRA=-DGLR_TOPK_STATS)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _native as N, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402
wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else 'C2')
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
r.run(y)
torch.cuda.synchronize()
buf = (C.c_uint * 4)()
fn = N.load().glr_debug_topk_stats
fn.argtypes = [C.c_void_p]
fn(buf)
print('rows', buf[0], 'fallback below L', buf[1], 'mean count>=L', buf[2] / max(buf[0], 1), 'max', buf[3])
