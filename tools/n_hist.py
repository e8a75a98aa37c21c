import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
for cfg, nf, prof in ((5, 24, 'efficient'), (4, 1, 'sentinel')):
    px, st = make_config(cfg, frames=nf)
    p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
    tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
    r = conceal_batch(tp, ts, p, records=True)
    rec = r.records
    s = rec[rec['layer'] == 2]
    n = s['n_y'].astype(int); cyc = s['cycles'].astype(float)
    print(f"cfg{cfg}: HQL patches {len(s)}")
    for v in np.unique(n):
        sel = n == v
        print(f"  n={v:2d}: {sel.mean():.3f} of HQL patches, {cyc[sel].sum() / cyc.sum():.3f} of HQL cycles, mean cycles {cyc[sel].mean():.0f}, k={v+1}, last tile rows {(v+1) % 8 or 8}")
