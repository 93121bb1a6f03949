"""Dev: per-iteration statistics of the iterate of one solve."""
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
prev = [None]
ref = torch.as_tensor(wl.scene, device='cuda', dtype=torch.float64).reshape(-1)


def on_iter(it, x):
    xf = x.reshape(-1)
    d = float((xf - prev[0]).abs().max()) if prev[0] is not None else float('nan')
    prev[0] = xf.clone()
    mse = float(((xf.clamp(0, 1) - ref) ** 2).mean()) if ref.numel() == xf.numel() else float('nan')
    print(f"it {it:2d} sigma {cfg.sigma_at(it):.4f} mean {float(xf.mean()):.6f} std {float(xf.std()):.6f} "
          f"max|dx| {d:.3e} mse {mse:.3e} finite {bool(torch.isfinite(xf).all())}")


r.run(y, on_iter=on_iter)
