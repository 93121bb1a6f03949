"""Dev: per-phase cycles of topk_kernel over one solve (needs
GLR_NVCC_EXTRA=-DGLR_TOPK_PHASES)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
from paper_2301_03047_b200 import _native as N, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402
wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else 'C4')
r = GapRunner(workloads.operator_for(wl), wl.solver_config())
y = r.dop.upload_y(wl.y)
fn = N.load().glr_debug_topk_phases
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8)()
r.run(y)
torch.cuda.synchronize()
fn(buf, 1)
r.run(y)
torch.cuda.synchronize()
fn(buf, 0)
v = [int(x) for x in buf[:6]]
tot = sum(v)
names = ["sampled floor", "row pass (ring)", "cut search", "collection", "sort A", "greedy walk + output"]
for nm, c in zip(names, v):
    print(f"{nm:24s} {100.0 * c / max(tot, 1):5.1f} %")
