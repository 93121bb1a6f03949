"""Dev: how many groups keep the same anchor AND identical positions across refreshes."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G
from paper_2301_03047_b200 import workloads
from paper_2301_03047_b200.solvers import GapRunner
for name in sys.argv[1:]:
    wl = workloads.make(name)
    cfg = wl.solver_config()
    r = GapRunner(workloads.operator_for(wl), cfg)
    y = r.dop.upload_y(wl.y)
    trace = []
    r.run(y, trace=trace)
    for j in range(1, len(trace)):
        a0, p0 = trace[j - 1]; a1, p1 = trace[j]
        d0 = {tuple(a): i for i, a in enumerate(a0)}
        same_anchor = same_pos = same_set = 0
        for i, a in enumerate(a1):
            k = d0.get(tuple(a))
            if k is None: continue
            same_anchor += 1
            if p0[k] == p1[i]: same_pos += 1
            if set(map(tuple, p0[k])) == set(map(tuple, p1[i])): same_set += 1
        print(name, j, len(a1), 'same anchor', same_anchor, 'same positions', same_pos, 'same set', same_set, flush=True)
