"""Dev tool: per-GPU share of cfg5 at N = 8/4/2/1 GPUs (32/64/128/256 frames)
on one GPU, per kernel build: the time a rank of the N-GPU run needs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config

prof = bm.Profile.named("efficient")
frames = [int(a) for a in sys.argv[1:]] or [32, 64, 128, 256]
px_all, st_all = make_config(5, frames=max(frames))
for nf in frames:
    tp = torch.from_numpy(px_all[:nf]).cuda()
    ts = torch.from_numpy(st_all[:nf]).cuda()
    for build in (None, 256, 512, "cluster"):
        conceal_batch(tp, ts, prof, kernel_build=build)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(2):
            e0.record()
            r = conceal_batch(tp, ts, prof, kernel_build=build, sync=False)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        cells = r.summary["lost_cells"] if r.summary else 0
        print(f"frames {nf:4d} build {str(build):7s}: {min(ms):8.1f} ms  ({cells / (min(ms) / 1e3):9.0f} cells/s per GPU)", flush=True)
