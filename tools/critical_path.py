"""Critical-path anatomy of a workload (dev tool): conceal with records, sum
the per-patch SM cycles of every cell, and follow the longest chain of the
cross-cell dependency DAG (each cell waits for its earlier-raster lost
8-neighbours).  Prints the chain's length in cells and cycles, its layer
mix, and what the per-cell cost is made of.

    python tools/critical_path.py cfg3 [--build 256|512]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import WORKLOADS, profile_of  # noqa: E402
from paper_2205_11226_b200 import conceal_batch  # noqa: E402
from paper_2205_11226_b200.synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--build", type=int, default=None)
ap.add_argument("--frames", type=int, default=None)
a = ap.parse_args()
cfg, prof_name, forced = WORKLOADS[a.workload]
px, st = make_config(cfg, frames=a.frames)
prof = profile_of(prof_name)
tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
conceal_batch(tp, ts, prof, forced_layer=forced, kernel_build=a.build)  # warm-up
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
res = conceal_batch(tp, ts, prof, forced_layer=forced, records=True, kernel_build=a.build)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1)
rec = res.records
khz = int(torch.cuda.get_device_properties(0).clock_rate) if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1965000
B, H, W = px.shape
GR, GC = H // 16, W // 16
cell = (rec["frame"].astype(np.int64) * GR + rec["row"] // 16) * GC + rec["col"] // 16
cyc = rec["cycles"].astype(np.float64)
ncell = B * GR * GC
cost = np.bincount(cell, weights=cyc, minlength=ncell)
npatch = np.bincount(cell, minlength=ncell)
lost = npatch > 0
by_layer = {}
for k, name in ((-1, "deferred"), (0, "BRL"), (1, "IDL"), (2, "HQL")):
    sel = rec["layer"] == k
    by_layer[name] = np.bincount(cell[sel], weights=cyc[sel], minlength=ncell)
# longest path (cycles) per frame in raster order
best = np.zeros(ncell)
prev = np.full(ncell, -1)
for f in range(B):
    for r in range(GR):
        for c in range(GC):
            i = (f * GR + r) * GC + c
            if not lost[i]:
                continue
            b, p = 0.0, -1
            for dr, dc in ((-1, -1), (-1, 0), (-1, 1), (0, -1)):
                rr, cc = r + dr, c + dc
                if 0 <= rr and 0 <= cc < GC:
                    j = (f * GR + rr) * GC + cc
                    if lost[j] and best[j] > b:
                        b, p = best[j], j
            best[i] = b + cost[i]
            prev[i] = p
end = int(np.argmax(best))
chain = []
while end >= 0:
    chain.append(end)
    end = prev[end]
chain = chain[::-1]
hz = 1.965e9
print(f"{a.workload}: {B} frames, {lost.sum()} lost cells, {len(rec)} patches, launch {ms:.1f} ms, "
      f"dag depth {res.summary['max_level']}")
print(f"critical chain: {len(chain)} cells, {best[chain[-1]]:.3e} cycles = {best[chain[-1]] / hz * 1e3:.1f} ms at 1965 MHz")
ch = np.array(chain)
pp = npatch[ch].sum()
print(f"  patches on chain {pp}, mean {cost[ch].sum() / pp:.0f} cycles/patch")
for name, v in by_layer.items():
    n = int(np.isin(cell, ch)[rec["layer"] == {"deferred": -1, "BRL": 0, "IDL": 1, "HQL": 2}[name]].sum()) if False else None
    print(f"  {name:8s} {v[ch].sum() / cost[ch].sum() * 100:5.1f}% of chain cycles")
layer_of = rec["layer"]
onchain = np.isin(cell, ch)
for k, name in ((0, "BRL"), (1, "IDL"), (2, "HQL")):
    sel = onchain & (layer_of == k)
    if sel.any():
        print(f"  {name}: {sel.sum()} patches, mean {cyc[sel].mean():.0f} cycles, median {np.median(cyc[sel]):.0f}, "
              f"p90 {np.percentile(cyc[sel], 90):.0f}; m mean {rec['m_candidates'][sel].mean():.0f}, "
              f"rings mean {rec['rings_used'][sel].mean():.1f}")
allsel = layer_of >= 0
print("whole batch per layer:")
for k, name in ((0, "BRL"), (1, "IDL"), (2, "HQL")):
    sel = layer_of == k
    if sel.any():
        print(f"  {name}: {sel.sum()} patches, mean {cyc[sel].mean():.0f} cycles, m mean {rec['m_candidates'][sel].mean():.0f}")
