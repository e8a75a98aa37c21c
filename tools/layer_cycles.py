"""Dev tool: per-layer share of SM cycles (bm_patch_record.cycles) on a workload subset."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
cfg = int(sys.argv[1]); nf = int(sys.argv[2]); prof = sys.argv[3]
px, st = make_config(cfg, frames=nf)
p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
r = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), p, records=True)
rec = r.records
tot = rec['cycles'].astype(np.float64).sum()
for L, name in [(0, 'BRL'), (1, 'IDL'), (2, 'HQL'), (-1, 'deferred')]:
    sel = rec['layer'] == L
    if sel.any():
        c = rec['cycles'][sel].astype(np.float64)
        print(f"{name}: n={sel.sum()} share={c.sum()/tot:.3f} mean_cycles={c.mean():.0f} p50={np.median(c):.0f} p99={np.percentile(c,99):.0f} meanM={rec['m_candidates'][sel].mean():.0f}")
hq = rec['layer'] == 2
if hq.any():
    m = rec['m_candidates'][hq]; c = rec['cycles'][hq]
    for lo, hi in [(0, 500), (500, 1000), (1000, 1500), (1500, 2100)]:
        s = (m >= lo) & (m < hi)
        if s.any(): print(f"  HQL M in [{lo},{hi}): n={s.sum()} mean_cycles={c[s].mean():.0f}")
print(r.summary)
