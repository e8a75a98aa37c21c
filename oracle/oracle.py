"""ctypes wrapper of the CPU oracle (oracle/bm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, never by the product
package.  The oracle is a plain-C FP64 restatement of the reference
``blockmend`` concealment path; its pin against the reference lives in
tests/test_oracle_golden.py (golden vectors from tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libbm_oracle.so")

# numpy view of bm_patch_record (include/blockmend_b200.h)
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


class _Info(ctypes.Structure):
    _fields_ = [
        ("layer", ctypes.c_int),
        ("fallback", ctypes.c_int),
        ("m", ctypes.c_int),
        ("has_nu", ctypes.c_int),
        ("beta", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("nu", ctypes.c_double),
        ("gap", ctypes.c_double),
    ]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        _lib.orc_conceal.restype = ctypes.c_int
        _lib.orc_conceal.argtypes = [
            ctypes.c_int, ctypes.c_int, dp, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_int, dp, ctypes.c_void_p, ctypes.c_long,
            ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long),
        ]
        _lib.orc_conceal_dag.restype = ctypes.c_int
        _lib.orc_conceal_dag.argtypes = _lib.orc_conceal.argtypes + [ctypes.c_int]
        _lib.orc_hql.argtypes = [dp, ctypes.c_int, dp, dp, ctypes.c_int, ctypes.c_double, dp,
                                 ctypes.POINTER(_Info)]
        _lib.orc_idl.argtypes = [dp, ctypes.c_int, dp, dp, ctypes.c_int, ctypes.c_double, dp, dp]
        _lib.orc_brl.argtypes = [dp, ctypes.c_int, dp]
        _lib.orc_pairwise_sum.restype = ctypes.c_double
        _lib.orc_pairwise_sum.argtypes = [dp, ctypes.c_long]
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def conceal(pixels, states, t_phi, t_nu, sigma2=10.0, forced_layer=-1):
    """Oracle conceal_image on one frame -> (out float64, records, status, lost_cells)."""
    px = np.ascontiguousarray(pixels, dtype=np.float64)
    st = np.ascontiguousarray(states, dtype=np.uint8)
    h, w = px.shape
    out = np.empty_like(px)
    cap = (h // 16) * (w // 16) * 64 + 1
    recs = np.zeros(cap, dtype=RECORD_DTYPE)
    nrec = ctypes.c_long(0)
    cells = ctypes.c_long(0)
    status = lib().orc_conceal(
        h, w, _dp(px), st.ctypes.data, float(t_phi), float(t_nu), float(sigma2), int(forced_layer),
        _dp(out), recs.ctypes.data, cap, ctypes.byref(nrec), ctypes.byref(cells),
    )
    return out, recs[: nrec.value].copy(), status, cells.value


def conceal_dag(pixels, states, t_phi, t_nu, sigma2=10.0, forced_layer=-1, threads=None):
    """conceal() with the cells of each dependency level concurrent on
    `threads` threads (same result as the serial raster order); for
    full-size parity frames."""
    px = np.ascontiguousarray(pixels, dtype=np.float64)
    st = np.ascontiguousarray(states, dtype=np.uint8)
    h, w = px.shape
    out = np.empty_like(px)
    cap = (h // 16) * (w // 16) * 64 + 1
    recs = np.zeros(cap, dtype=RECORD_DTYPE)
    nrec = ctypes.c_long(0)
    cells = ctypes.c_long(0)
    if threads is None:
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    status = lib().orc_conceal_dag(
        h, w, _dp(px), st.ctypes.data, float(t_phi), float(t_nu), float(sigma2), int(forced_layer),
        _dp(out), recs.ctypes.data, cap, ctypes.byref(nrec), ctypes.byref(cells), int(threads),
    )
    return out, recs[: nrec.value].copy(), status, cells.value


def _dense(y0, x, y):
    y0 = np.asarray(y0, dtype=np.float64)
    n = y0.shape[0]
    x = np.asarray(x, dtype=np.float64).reshape(-1, 4)
    m = x.shape[0]
    yy = np.zeros((max(m, 1), 32))
    yy[:m, :n] = np.asarray(y, dtype=np.float64).reshape(m, n)
    y0p = np.zeros(32)
    y0p[:n] = y0
    return y0p, n, np.ascontiguousarray(x if m else np.zeros((1, 4))), yy, m


def hql(y0, x, y, sigma2=10.0):
    y0p, n, xx, yy, m = _dense(y0, x, y)
    out = np.zeros(4)
    info = _Info()
    lib().orc_hql(_dp(y0p), n, _dp(xx), _dp(yy), m, sigma2, _dp(out), ctypes.byref(info))
    return out, {"layer": info.layer, "fallback": bool(info.fallback), "beta": info.beta,
                 "alpha": info.alpha, "nu": info.nu if info.has_nu else None, "beta_gap": info.gap}


def idl(y0, x, y, sigma2=10.0):
    y0p, n, xx, yy, m = _dense(y0, x, y)
    out = np.zeros(4)
    raw = ctypes.c_double(0.0)
    rc = lib().orc_idl(_dp(y0p), n, _dp(xx), _dp(yy), m, sigma2, _dp(out), ctypes.byref(raw))
    return (None if rc else out), raw.value


def pairwise_sum(a):
    """The oracle's restatement of NumPy's pairwise summation (test hook)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_pairwise_sum(_dp(a), a.size)


def brl(y0):
    y0 = np.ascontiguousarray(y0, dtype=np.float64)
    out = np.zeros(4)
    lib().orc_brl(_dp(y0), y0.shape[0], _dp(out))
    return out
