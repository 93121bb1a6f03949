"""Dev: fallback reasons of the fused heat + top-K list path on one refresh
(needs a build with GLR_NVCC_EXTRA=-DGLR_TOPK_STATS)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _device as D, _native as N, workloads  # noqa: E402
from paper_2301_03047_b200.engine import DeviceOperator, GlrEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
if name.startswith("C5"):
    wl = workloads.make("C5")
    mc = G.MatchConfig(patch_size=int(name[3:] or 8), group_size=64, max_corners=1024,
                       exemplar_stride=4096)
    x_d = D.f64(wl.scene)
else:
    wl = workloads.make(name)
    mc = wl.match
    dop = DeviceOperator(workloads.operator_for(wl))
    x_d = D.zeros(wl.shape, D.torch().float64)
    dop.init_x(dop.upload_y(wl.y), x_d)
eng = GlrEngine(wl.shape, mc, low_memory_match=True)
lib = N.load()
buf = (C.c_uint * 10)()
lib.glr_debug_topk_stats(buf)
before = np.array(buf[:])
eng.refresh(x_d)
D.torch().cuda.synchronize()
lib.glr_debug_topk_stats(buf)
d = np.array(buf[:]) - before
print(name, "cap", eng.cand_cap, "rows", d[4], "overflow", d[5], "short", d[6], "ties", d[7],
      "mean list", d[8] / max(d[4], 1), "max list", buf[9], "fallback", eng.n_fallback)
