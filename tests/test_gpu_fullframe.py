"""Full-size parity at the configs' real dependency depth:
whole BASELINE frames concealed on the GPU against the CPU oracle, with the
oracle's cells of each dependency level run concurrently on every host core
(oracle.conceal_dag: the same result as the serial raster order).

Frames: one 1080p slice frame (cfg3, ~120-level chains), one 3840x2160 frame
with 20% random 8x8 losses under forced HQL and under forced IDL (cfg4,
~370-400 levels), and one 1080p frame of each cfg5 mask kind (dispersed,
slice, random 16x16).  The parity bar is tests/parity.py's; the all-pixel
figures (every lost pixel, excused cells included) are printed and bounded.
"""

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_11226_b200 import Profile, conceal_batch
from paper_2205_11226_b200.synth import make_config

pytestmark = pytest.mark.gpu

CASES = [
    # (id, cfg, frame, profile, forced layer)
    ("cfg3_slice_frame", 3, 0, "efficient", None),
    ("cfg4_4k_hql_frame", 4, 0, "sentinel", "HQL"),
    ("cfg4_4k_idl_frame", 4, 0, "sentinel", "IDL"),
    ("cfg5_dispersed_frame", 5, 0, "efficient", None),
    ("cfg5_slice_frame", 5, 1, "efficient", None),
    ("cfg5_random_frame", 5, 2, "efficient", None),
]
# measured excused divergences (threshold decisions + reference beta ties) per frame
EXCUSED_MAX = {"cfg4_4k_hql_frame": 8}


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_full_frame_parity(native, case):
    import torch

    name, cfg, frame, prof_name, forced = case
    prof = Profile.sentinel() if prof_name == "sentinel" else Profile.named(prof_name)
    fcode = -1 if forced is None else {"BRL": 0, "IDL": 1, "HQL": 2}[forced]
    px, st = make_config(cfg, frames=1, first=frame)
    res = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof, forced_layer=forced,
                        want_f64=True, records=True)
    o_out, o_rec, status, cells = oracle.conceal_dag(px[0].astype(np.float64), st[0], prof.t_phi, prof.t_nu,
                                                     10.0, fcode)
    assert status == 0 and cells == res.summary["lost_cells"]
    pr = parity.compare(o_out, o_rec, res.recon_f64[0].cpu().numpy(), res.records, st[0], prof.t_phi, prof.t_nu)
    print(f"{name}: depth {res.summary['max_level']} cells {cells} patches {len(o_rec)} {pr.summary()}")
    assert pr.ok, pr.problems[:5]
    assert len(pr.allowed) + len(pr.beta_ties) <= EXCUSED_MAX.get(name, 0), (pr.allowed, pr.beta_ties)
    # even counting excused cells, u8 stays within +-1 LSB on <= 0.1% of the lost pixels
    # unless a rounding-decided beta tie propagated (reported above)
    if not pr.beta_ties:
        assert pr.max_u8_all <= 1 and pr.u8_off_all <= 0.001 * pr.lost_pixels
