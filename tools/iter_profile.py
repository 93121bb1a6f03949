"""Dev: per-iteration kernel times of one full solve (CUDA events)."""
import sys
import numpy as np
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
r.eng.timing = []
r.run(y, events=True)
torch.cuda.synchronize()
w = [a.elapsed_time(b) for (n, _), a, b in r.eng.timing if n == 'wnnm_scatter']
h = [a.elapsed_time(b) for (n, _), a, b in r.eng.timing if n in ('heat_map', 'heat_topk')]
print(name, 'wnnm per iteration (ms):', ' '.join(f'{v:.1f}' for v in w))
print('heat per refresh (ms):', ' '.join(f'{v:.1f}' for v in h))
names = sorted({n for (n, _), a, b in r.eng.timing})
for nm in names:
    if nm in ('wnnm_scatter', 'heat_map', 'heat_topk'):
        continue
    v = [a.elapsed_time(b) for (n, _), a, b in r.eng.timing if n == nm]
    print(f'{nm}: n={len(v)} mean {sum(v) / len(v):.3f} ms total {sum(v):.1f} ms')
it = [(e[0].elapsed_time(e[3])) for e in r.events]
print('iteration ms:', ' '.join(f'{v:.1f}' for v in it))
print('total', sum(it), 'fallback exemplars (last refresh):', r.eng.n_fallback)
