"""Dev: wall-clock breakdown of the public gap_solve path on C2 (host inputs)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _device as D, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402

wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else 'C2')
cfg = wl.solver_config()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
op = workloads.operator_for(wl)
op.meta["masks"] = pin(op.meta["masks"])
op.gram_diag = pin(op.gram_diag)
y = pin(wl.y)
G.gap_solve(op, y, cfg)
for rep in range(2):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    r = GapRunner(op, cfg)
    torch.cuda.synchronize(); T.append(time.perf_counter())
    yd = r.dop.upload_y(y)
    torch.cuda.synchronize(); T.append(time.perf_counter())
    x = r.run(yd, events=True)
    torch.cuda.synchronize(); T.append(time.perf_counter())
    res = D.host(r.resid_sq)
    T.append(time.perf_counter())
    out = D.host(x).copy()
    T.append(time.perf_counter())
    out = np.clip(out, 0.0, 1.0)
    T.append(time.perf_counter())
    names = ['runner init', 'upload y', 'run', 'resid d2h', 'x d2h+copy', 'clip']
    print(' '.join(f'{n}={1e3 * (T[i + 1] - T[i]):.1f}ms' for i, n in enumerate(names)))
    t0 = time.perf_counter()
    G.gap_solve(op, y, cfg)
    print('gap_solve total', 1e3 * (time.perf_counter() - t0))
