"""Dev tool: bitwise comparison of two native build variants on a workload
(FP64 outputs and records), e.g. for changes meant to be bit-identical.

    python tools/bitcmp.py <variantA|base> <variantB|base> [cfg frames build]
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(variant, cfg, frames, build, out):
    code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import numpy as np, torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.synth import make_config
from bench import WORKLOADS, profile_of
cfgn, prof, forced = WORKLOADS['cfg{cfg}']
px, st = make_config(cfgn, frames={frames})
kb = None if {build!r} == 'auto' else ({build!r} if not {build!r}.isdigit() else int({build!r}))
r = bm.conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), profile_of(prof),
                     forced_layer=None if forced is None else bm.Layer[forced], want_f64=True, records=True, kernel_build=kb)
np.savez({out!r}, f64=r.recon_f64.cpu().numpy(), rec=r.records, build=str(r.summary.get('kernel_build')))
"""
    env = dict(os.environ)
    env.pop("BM_NATIVE_VARIANT", None)
    if variant != "base":
        env["BM_NATIVE_VARIANT"] = variant
    subprocess.run([sys.executable, "-c", code], check=True, env=env)


a, b = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "5"
frames = int(sys.argv[4]) if len(sys.argv) > 4 else 8
build = sys.argv[5] if len(sys.argv) > 5 else "auto"
run(a, cfg, frames, build, "/tmp/bitcmp_a.npz")
run(b, cfg, frames, build, "/tmp/bitcmp_b.npz")
A, B = np.load("/tmp/bitcmp_a.npz"), np.load("/tmp/bitcmp_b.npz")
same_f = np.array_equal(A["f64"].view(np.uint64), B["f64"].view(np.uint64))
ra, rb = A["rec"], B["rec"]
keys = [k for k in ra.dtype.names if k != "cycles"]
same_r = len(ra) == len(rb) and all(np.array_equal(ra[k], rb[k], equal_nan=ra[k].dtype.kind == "f") for k in keys)
nd = int((A["f64"] != B["f64"]).sum())
print(f"cfg{cfg} frames {frames} build {A['build']}/{B['build']}: {a} vs {b}: f64 bit-identical {same_f} "
      f"({nd} values differ), records identical {same_r}")
