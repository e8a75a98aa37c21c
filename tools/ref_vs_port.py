"""Speed of the reference's own Python path against the plain-C FP64 port
(oracle/) on identical inputs, single process each (build container only:
/root/reference does not travel to the GPU box).  The bench's CPU baseline and
reference arm run the port on the GPU box's host; this ratio states how that
port relates to the reference itself.

    python tools/ref_vs_port.py > profiles/ref_vs_port_r02.txt
"""
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import blockmend as ref  # noqa: E402

from bench import cpu_jobs  # noqa: E402
from oracle import oracle  # noqa: E402

jobs, cores, crop = cpu_jobs("cfg5", crop=384)
sel = jobs[:6]
tot_ref = tot_port = cells_tot = 0.0
print(f"# reference blockmend.conceal_image (Python {sys.version.split()[0]}, numpy {np.__version__}, 1 BLAS thread) "
      f"vs the C port oracle.conceal, one process, the bench's cfg5 CPU-sample crops ({crop}x{crop}, efficient)")
for i, (px, st, t_phi, t_nu, forced) in enumerate(sel):
    prof = ref.Profile.custom(t_phi, t_nu)
    t0 = time.perf_counter()
    _, rep = ref.conceal_image(ref.ImageBuffer(px.astype(np.float64)), ref.LossMask(st), prof)
    t1 = time.perf_counter()
    _, _, status, cells = oracle.conceal(px.astype(np.float64), st, t_phi, t_nu)
    t2 = time.perf_counter()
    tot_ref += t1 - t0
    tot_port += t2 - t1
    cells_tot += cells
    print(f"crop {i}: {cells} lost cells, {rep.patches} patches {rep.layer_counts}: reference {t1 - t0:7.2f} s, "
          f"C port {t2 - t1:6.3f} s, ratio {(t1 - t0) / (t2 - t1):5.1f}x")
print(f"total: {int(cells_tot)} cells; reference {cells_tot / tot_ref:.2f} cells/s, C port {cells_tot / tot_port:.2f} "
      f"cells/s per core; the C port is {tot_ref / tot_port:.1f}x faster than the reference")
