"""Dev tool: one conceal_batch of a config subset (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
cfg, nf, prof = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
px, st = make_config(cfg, frames=nf)
p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
for _ in range(2):
    r = conceal_batch(tp, ts, p)
print(r.summary)
