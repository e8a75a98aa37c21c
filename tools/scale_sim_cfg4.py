import sys, os
sys.path.insert(0, '/root/repo')
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
prof = bm.Profile.sentinel()
px_all, st_all = make_config(4, frames=8)
for nf in (1, 2, 4, 8):
    tp = torch.from_numpy(px_all[:nf]).cuda(); ts = torch.from_numpy(st_all[:nf]).cuda()
    for build in (None, 256, 512):
        conceal_batch(tp, ts, prof, forced_layer=bm.Layer.HQL, kernel_build=build)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = conceal_batch(tp, ts, prof, forced_layer=bm.Layer.HQL, kernel_build=build, sync=False); e1.record(); e1.synchronize()
        print(f"cfg4 frames {nf} build {build}: {e0.elapsed_time(e1):.1f} ms", flush=True)
