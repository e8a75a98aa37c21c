"""Dev tool: per-cell cost from the records (sum of per-patch cycles) and the
critical chain of a config (cfg3 slices are bound by row chains)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200 import _native
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
cfg, nf, prof = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
px, st = make_config(cfg, frames=nf)
p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
conceal_batch(tp, ts, p)
r = conceal_batch(tp, ts, p, records=True, time_kernel=True)
rec = r.records
khz = _native.lib().bm_device_clock_khz()
cell = (rec['frame'].astype(np.int64) * 1000 + (rec['row'] // 16)) * 1000 + rec['col'] // 16
u, inv = np.unique(cell, return_inverse=True)
cyc = np.bincount(inv, weights=rec['cycles'].astype(np.float64))
print('kernel ms', _native.kernel_times_ms()[-1], 'cells', len(u), 'summary', r.summary)
print('cell cycles: mean %.0f p50 %.0f p90 %.0f max %.0f  (ms at %d kHz: mean %.3f max %.3f)' % (
    cyc.mean(), np.median(cyc), np.percentile(cyc, 90), cyc.max(), khz, cyc.mean() / khz, cyc.max() / khz))
# chain estimate: per frame, per lost row of cells, sum of cell cycles along the row
fr = u // 1000000; rr = (u // 1000) % 1000
tot = {}
for f_, r_, c_ in zip(fr, rr, cyc):
    tot[(f_, r_)] = tot.get((f_, r_), 0) + c_
best = max(tot.values())
print('max row-chain cycles %.3e = %.1f ms' % (best, best / khz))
