"""Dev: one C5 refresh (2048^2, P, N exemplars) inside a profiler range, for
`ncu --profile-from-start off` (dense or fused heat + top-K)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _device as D, workloads  # noqa: E402
from paper_2301_03047_b200.engine import GlrEngine  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
wl = workloads.make("C5")
mc = G.MatchConfig(patch_size=p, group_size=64, max_corners=n, exemplar_stride=4096)
eng = GlrEngine(wl.shape, mc, low_memory_match=fused)
x = D.f64(wl.scene)
eng.refresh(x)
torch.cuda.synchronize()
rt = torch.cuda.cudart()
rt.cudaProfilerStart()
eng.refresh(x)
torch.cuda.synchronize()
rt.cudaProfilerStop()
print("done", eng.n, eng.n_fallback)
