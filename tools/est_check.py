"""Dev tool: GPU estimate_batch (HQL) vs oracle on random instances."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2205_11226_b200 import estimators as est, Layer
from oracle import oracle
rng = np.random.default_rng(5)
ts, cs = [], []
for m, n in [(2, 1), (3, 2), (5, 4), (9, 8), (17, 16), (40, 20), (100, 32), (300, 31), (700, 12), (1849, 32), (1500, 24), (64, 32), (33, 32), (34, 33 - 1)]:
    y0 = rng.uniform(0, 255, n)
    ts.append(est.TargetContext((0, 0), np.ones(32, bool), y0, n))
    cs.append(est.CandidateSet(np.round(rng.uniform(0, 255, (m, 4))), np.round(rng.uniform(0, 255, (m, n)))))
got = est.estimate_batch(Layer.HQL, ts, cs)
for t, c, g in zip(ts, cs, got):
    vals, info = oracle.hql(t.y0, c.x, c.y)
    print(c.x.shape[0], t.n_y, g.layer.value, info['layer'], 'beta', g.diagnostics.bandwidth.beta if g.diagnostics.bandwidth else None, info['beta'],
          'alpha', g.diagnostics.bandwidth.alpha if g.diagnostics.bandwidth else None, info['alpha'], 'maxdiff', np.max(np.abs(g.values - vals)), 'gap', info['beta_gap'])
