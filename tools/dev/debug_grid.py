import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1506_06039_b200 import Plan
from tests import paper_forms as pf
cases = [(128, 64, 1, 9, 4096), (96, 64, 0, 20, 4096), (80, 96, 0, 32, 4096), (64, 64, 1, 16, 4096), (128,128,0,30,16384)]
for (m, n, levels, w, hi) in cases:
    rng = np.random.default_rng(m * 1000 + n + levels + w)
    T = 3
    bits = 16 if hi > 16384 else (14 if hi > 4096 else 12)
    fr = rng.integers(0, hi, size=(T, m, n)).astype(np.uint16)
    tp = rng.integers(0, hi, size=(m, n)).astype(np.uint16)
    fr[1] = pf.translate_zero_fill(tp, 3, -2)
    B = oracle.pyramid(tp, levels)[levels]
    for rep in range(3):
        p = Plan(m, n, w, levels, "u16", bits, device=0, algo="tc")
        p.set_template(torch.from_numpy(tp).cuda())
        g = p.score_grid(torch.from_numpy(fr).cuda()).cpu().numpy()
        bad = 0
        for k in range(T):
            A = oracle.pyramid(fr[k], levels)[levels]
            ref = oracle.objective_grid(A, B, w)
            d = np.argwhere(g[k] != ref)
            bad += len(d)
            if len(d): print((m,n,levels,w), 'rep', rep, 'frame', k, 'nbad', len(d), 'first', d[:6].tolist(), 'rel', float(np.max(np.abs(g[k]-ref)/ref)))
        print((m,n,levels,w), 'rep', rep, 'bad', bad, flush=True)
