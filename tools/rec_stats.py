"""Dev tool: per-patch statistics from the decision records (m, n_y, cycles by layer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
cfg, nf, prof = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
px, st = make_config(cfg, frames=nf)
p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
conceal_batch(tp, ts, p)
r = conceal_batch(tp, ts, p, records=True)
rec = r.records
print(r.summary)
tot = rec['cycles'].astype(np.float64).sum()
for lay, name in ((0, 'BRL'), (1, 'IDL'), (2, 'HQL')):
    s = rec[rec['layer'] == lay]
    if len(s) == 0:
        continue
    cyc = s['cycles'].astype(np.float64)
    m = s['m_candidates'].astype(np.float64)
    print(f"{name}: {len(s)} patches, cycles mean {cyc.mean():.0f} p50 {np.median(cyc):.0f} p90 {np.percentile(cyc, 90):.0f}, "
          f"share {cyc.sum() / tot:.3f}; m mean {m.mean():.1f} p50 {np.median(m):.0f} p90 {np.percentile(m, 90):.0f}; "
          f"n_y mean {s['n_y'].mean():.1f}; rings mean {s['rings_used'].mean():.1f}")
    if lay >= 1:
        edges = [0, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
        h = np.digitize(m, edges)
        for b in np.unique(h):
            sel = h == b
            print(f"   m in [{edges[b-1]},{edges[b] if b < len(edges) else 'inf'}): {sel.sum():8d}  cycles mean {cyc[sel].mean():8.0f}  "
                  f"share {cyc[sel].sum() / tot:.3f}")
    if lay == 2:
        for ny in (8, 16, 24, 32):
            sel = (s['n_y'] > ny - 8) & (s['n_y'] <= ny)
            print(f"   n_y in ({ny-8},{ny}]: {sel.sum():8d} cycles mean {cyc[sel].mean() if sel.any() else 0:8.0f}")
