"""bm_patch_record (include/blockmend_b200.h) as a numpy dtype, and its
conversion to the reference's LayerDecision (profiles.py:81-95)."""

from __future__ import annotations

import numpy as np

RECORD_DTYPE = np.dtype(
    [
        ("frame", "<i4"),
        ("row", "<i4"),
        ("col", "<i4"),
        ("layer", "i1"),
        ("flags", "u1"),
        ("n_y", "u1"),
        ("rings_used", "u1"),
        ("m_candidates", "<i4"),
        ("cycles", "<u4"),
        ("beta_gap", "<f4"),
        ("pad", "<u4"),
        ("phi", "<f8"),
        ("nu", "<f8"),
        ("beta", "<f8"),
        ("alpha", "<f8"),
    ]
)
assert RECORD_DTYPE.itemsize == 64

REC_FALLBACK, REC_DEFERRED, REC_HAS_NU, REC_HAS_PHI, REC_HAS_BW, REC_HAS_M = 1, 2, 4, 8, 16, 32


def decode_flags(r) -> dict:
    f = int(r["flags"])
    return {
        "fallback": bool(f & REC_FALLBACK),
        "deferred": bool(f & REC_DEFERRED),
        "has_nu": bool(f & REC_HAS_NU),
        "has_phi": bool(f & REC_HAS_PHI),
        "has_bw": bool(f & REC_HAS_BW),
        "has_m": bool(f & REC_HAS_M),
    }
