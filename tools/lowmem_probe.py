"""Dev: dense (heat map + top-K) vs fused low-memory (glr_heat_topk) matching
on C2: per-refresh times and fallback counts."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import workloads, _device as D  # noqa: E402
from paper_2301_03047_b200.engine import GlrEngine  # noqa: E402

wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else 'C2')
x = D.f64(wl.scene)
for lm in (False, True):
    eng = GlrEngine(wl.shape, wl.match, low_memory_match=lm)
    for rep in range(3):
        eng.timing = []
        eng.refresh(x)
        torch.cuda.synchronize()
        t = {}
        for (name, nb), a, b in eng.timing:
            t[name] = t.get(name, 0.0) + a.elapsed_time(b)
        eng.timing = None
    pos = D.host(eng.positions[:eng.n]).copy()
    print('low_memory' if lm else 'dense', {k: round(v, 3) for k, v in t.items()},
          'fallback', eng.n_fallback, flush=True)
    if lm:
        print('positions identical to dense:', (pos == pos_dense).all())
    else:
        pos_dense = pos
    del eng
    torch.cuda.empty_cache()
