"""Dump one full frame's GPU result (lost-pixel values + records) for offline
parity forensics against the oracle / reference (dev tool).

    python tools/dump_frame.py <cfg> <frame> <profile|sentinel> <forced|-> <out.npz> [--build N]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2205_11226_b200 import Profile, conceal_batch  # noqa: E402
from paper_2205_11226_b200.synth import make_config  # noqa: E402

cfg, frame, prof_name, forced, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
build = int(sys.argv[7]) if len(sys.argv) > 7 else None
prof = Profile.sentinel() if prof_name == "sentinel" else Profile.named(prof_name)
forced = None if forced == "-" else forced
px, st = make_config(cfg, frames=1, first=frame)
res = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof, forced_layer=forced,
                    want_f64=True, records=True, kernel_build=build)
v = res.recon_f64[0].cpu().numpy()
np.savez_compressed(out, lost_values=v[st[0] == 1], records=res.records)
print("dumped", out, len(res.records))
