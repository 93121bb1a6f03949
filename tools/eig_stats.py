"""Dev: Jacobi sweep-count histogram per iteration of one C2 solve
(needs a build with GLR_NVCC_EXTRA=-DGLR_EIG_STATS)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _native as N, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
wl = workloads.make(name)
cfg = wl.solver_config()
r = GapRunner(workloads.operator_for(wl), cfg)
y = r.dop.upload_y(wl.y)
lib = N.load()
fn = lib.glr_debug_eig_hist
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_uint * 146)()
fn(buf, 1)


def on_iter(it, x):
    torch.cuda.synchronize()
    fn(buf, 1)
    h = np.array(buf[:64])
    cold = {i: int(v) for i, v in enumerate(h[:32]) if v}
    warm = {i: int(v) for i, v in enumerate(h[32:]) if v}
    tot = h[:32] @ np.arange(32) + h[32:] @ np.arange(32)
    rk = np.array(buf[64:129])
    cum = np.cumsum(rk) / max(rk.sum(), 1)
    q = [int(np.searchsorted(cum, f)) for f in (0.1, 0.5, 0.9, 0.99)]
    res = np.frombuffer(bytes(buf), dtype=np.uint64, count=8, offset=130 * 4)
    ng = max(int(res[0]), 1)
    rs = ' '.join(f'{int(v) / ng:.1f}' for v in res[1:7])
    print(f"it {it:2d} pairs/group above 1e-4..1e-9: {rs}  lines/warm group {int(res[7]) / ng:.1f}")
    print(f"it {it:2d} mean sweeps {tot / max(h.sum(), 1):.2f} cold {cold} warm {warm} "
          f"kept-rank mean {rk @ np.arange(65) / max(rk.sum(), 1):.1f} p10/50/90/99 {q}")


r.run(y, on_iter=on_iter)
