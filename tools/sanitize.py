"""compute-sanitizer driver: one conceal_batch on a cfg5 crop
(3 frames, one of each mask kind: dispersed / slice / random) plus a narrow
slice crop, both kernel builds, checked against the CPU oracle afterwards so
the run also proves the sanitized launch computed the right thing.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import parity  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2205_11226_b200 import Profile, conceal_batch  # noqa: E402
from paper_2205_11226_b200.synth import make_config  # noqa: E402

crop = tuple(int(v) for v in os.environ.get("BM_SAN_CROP", "96,128").split(","))
prof = Profile.named("efficient")
px, st = make_config(5, frames=3, crop=crop)
ok = True
for build in (256, 512):
    res = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof, want_f64=True, records=True,
                        kernel_build=build)
    torch.cuda.synchronize()
    g = res.recon_f64.cpu().numpy()
    for f in range(px.shape[0]):
        o_out, o_rec, status, cells = oracle.conceal(px[f].astype(np.float64), st[f], prof.t_phi, prof.t_nu)
        sel = res.records[res.records["frame"] == f]
        r = parity.compare(o_out, o_rec, g[f], sel, st[f], prof.t_phi, prof.t_nu)
        print(f"build {build} frame {f}: cells {cells} {r.summary()}", flush=True)
        ok &= r.ok
print("SANITIZE_PARITY", "OK" if ok else "FAIL", flush=True)
sys.exit(0 if ok else 1)
