"""Loader and ctypes bindings of the sm_100a extension (_blockmend_b200.so).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute call raises NativeUnavailableError.
`build()` compiles csrc/ in-tree with nvcc for sm_100a.
"""

from __future__ import annotations

import ctypes
import glob
import os
import subprocess

from .errors import DimensionMismatchError, NativeUnavailableError

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "_blockmend_b200.so")
SOURCES = [os.path.join(PKG_DIR, "csrc", f)
           for f in ("bm_conceal.cu", "bm_conceal_wide.cu", "bm_conceal_cluster.cu", "bm_aux.cu", "bm_api.cu")]
HEADERS = sorted(glob.glob(os.path.join(PKG_DIR, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG_DIR, "csrc", "*.h"))) + [
    os.path.join(os.path.dirname(PKG_DIR), "include", "blockmend_b200.h")
]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

BM_FLAG_TIME_KERNEL = 1
BM_FLAG_BUILD_256, BM_FLAG_BUILD_512, BM_FLAG_BUILD_CLUSTER, BM_FLAG_NARROW_512 = 2, 4, 8, 16
BM_OK, BM_ERR_ARGS, BM_ERR_LOST_LEFT, BM_ERR_CUDA, BM_ERR_WORKSPACE, BM_ERR_STATES = 0, 1, 2, 3, 4, 5


class Params(ctypes.Structure):
    _fields_ = [
        ("frames", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("pixel_dtype", ctypes.c_int32),
        ("t_phi", ctypes.c_double),
        ("t_nu", ctypes.c_double),
        ("sigma2", ctypes.c_double),
        ("forced_layer", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class Summary(ctypes.Structure):
    _fields_ = [
        ("lost_cells", ctypes.c_int64),
        ("patches", ctypes.c_int64),
        ("layer_counts", ctypes.c_int64 * 3),
        ("deferred_fills", ctypes.c_int64),
        ("lost_left", ctypes.c_int64),
        ("max_level", ctypes.c_int32),
        ("bad_states", ctypes.c_int32),
        ("flop64", ctypes.c_int64),
        ("flop32", ctypes.c_int64),
        ("hql_patches", ctypes.c_int64),
        ("gate_candidates", ctypes.c_int64),
        ("kernel_build", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


SUMMARY_BYTES = ctypes.sizeof(Summary)
EXPORTS = [
    "bm_abi_version", "bm_status_string", "bm_workspace_bytes", "bm_max_records", "bm_device_clock_khz",
    "bm_kernel_times_ms", "bm_kernel_times_reset", "bm_debug_phase_cycles",
    "bm_conceal", "bm_compact_records", "bm_conceal_host", "bm_estimate_batch",
    "bm_sqdiff_batch", "bm_ssim_batch", "bm_gen_masks",
    "bm_select_and_estimate", "bm_extract_targets", "bm_collect", "bm_patch_scores", "bm_build_schedule",
    "bm_expansion_maps", "bm_estimator_stages",
]


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> _blockmend_b200.so (in-tree)."""
    if not force and not needs_build():
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    cmd = ["nvcc", *NVCC_FLAGS, "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    """The loaded extension; raises NativeUnavailableError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    # BM_NATIVE_VARIANT=<tag> loads an in-tree build variant _blockmend_b200.<tag>.so
    # (tools/ A/B experiments); the default is the product build.
    tag = os.environ.get("BM_NATIVE_VARIANT")
    path = LIB_PATH.replace(".so", f".{tag}.so") if tag else LIB_PATH
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing: build it with paper_2205_11226_b200._native.build() "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.bm_abi_version.restype = ctypes.c_int
    L.bm_status_string.restype = ctypes.c_char_p
    L.bm_status_string.argtypes = [ctypes.c_int]
    L.bm_workspace_bytes.restype = ctypes.c_size_t
    L.bm_workspace_bytes.argtypes = [ctypes.POINTER(Params)]
    L.bm_max_records.restype = i64
    L.bm_max_records.argtypes = [ctypes.POINTER(Params)]
    L.bm_device_clock_khz.restype = ctypes.c_int
    L.bm_kernel_times_ms.restype = ctypes.c_int
    L.bm_kernel_times_ms.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    L.bm_kernel_times_reset.restype = None
    L.bm_debug_phase_cycles.restype = ctypes.c_int
    L.bm_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.bm_conceal.restype = ctypes.c_int
    L.bm_conceal.argtypes = [ctypes.POINTER(Params), vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.bm_compact_records.restype = ctypes.c_int
    L.bm_compact_records.argtypes = [ctypes.POINTER(Params), vp, vp, vp, ctypes.POINTER(i64), vp]
    L.bm_conceal_host.restype = ctypes.c_int
    L.bm_conceal_host.argtypes = [ctypes.POINTER(Params), vp, vp, vp, vp, vp, ctypes.POINTER(i64), ctypes.POINTER(Summary)]
    L.bm_estimate_batch.restype = ctypes.c_int
    L.bm_estimate_batch.argtypes = [i32, i32, i32, ctypes.c_double, vp, vp, vp, vp, vp, vp, vp, vp]
    L.bm_sqdiff_batch.restype = ctypes.c_int
    L.bm_sqdiff_batch.argtypes = [vp, vp, i32, vp, i32, i32, i32, vp, vp, vp]
    L.bm_ssim_batch.restype = ctypes.c_int
    L.bm_ssim_batch.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp]
    L.bm_gen_masks.restype = ctypes.c_int
    L.bm_gen_masks.argtypes = [i32, i32, i32, i32, i32, i32, vp, vp, vp]
    L.bm_select_and_estimate.restype = ctypes.c_int
    L.bm_select_and_estimate.argtypes = [ctypes.POINTER(Params), vp, vp, i32, vp, vp, vp, vp, vp, vp]
    L.bm_extract_targets.restype = ctypes.c_int
    L.bm_extract_targets.argtypes = [i32, i32, vp, vp, i32, vp, vp, vp, vp, vp]
    L.bm_collect.restype = ctypes.c_int
    L.bm_collect.argtypes = [i32, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.bm_patch_scores.restype = ctypes.c_int
    L.bm_patch_scores.argtypes = [i32, i32, vp, i32, vp, vp, vp, vp]
    L.bm_build_schedule.restype = ctypes.c_int
    L.bm_build_schedule.argtypes = [i32, i32, vp, i32, vp, vp, vp, vp, vp]
    L.bm_expansion_maps.restype = ctypes.c_int
    L.bm_expansion_maps.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp]
    L.bm_estimator_stages.restype = ctypes.c_int
    L.bm_estimator_stages.argtypes = [i32, i32, i32, ctypes.c_double, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    _lib = L
    return L


def check(status: int) -> None:
    """Map a C-ABI status onto the reference's exceptions."""
    if status == BM_OK:
        return
    msg = lib().bm_status_string(status).decode()
    if status == BM_ERR_LOST_LEFT:
        raise AssertionError(msg)  # profiles.py:305
    if status == BM_ERR_STATES:
        raise ValueError(msg)  # image.py:69-70
    if status == BM_ERR_ARGS:
        raise DimensionMismatchError(msg)
    raise NativeUnavailableError(msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def kernel_times_ms() -> list[float]:
    """Durations of the timed concealment-kernel launches since the last reset."""
    buf = (ctypes.c_float * 256)()
    n = lib().bm_kernel_times_ms(buf, 256)
    return [float(buf[i]) for i in range(n)]


def kernel_times_reset() -> None:
    lib().bm_kernel_times_reset()


PHASES = ["gate", "means", "covariance", "cholesky", "linv", "quadforms", "dmin", "beta", "nearest", "staging",
          "e2_done", "loo", "alpha", "chol_only", "patch_idl", "patch_hql",
          "idl_pick", "idl_gather", "idl_estimate", "idl_writeback", "dep_wait", "patch_brl", "cta_life", "ctas",
          "sidl_setup", "sidl_screen", "sidl_ringsums", "sidl_scan", "sidl_dist_max", "sidl_exp_sum", "sidl_final", "sidl_count",
          "beta_loop_t0", "beta_loop_reduce", "loo_loops_t0", "nn_sorted", "nn_warp_merged", "nn_all_merged", "chol_linv", "chol_linv_stored",
          "load_tile", "load_tile_cells", "load_tile_nbufs", "gate2_first", "gate2_rest", "gate2_sums", "gate2_scan", "gate2_count"]


def phase_cycles(reset: bool = True) -> dict:
    buf = (ctypes.c_uint64 * 48)()
    check(lib().bm_debug_phase_cycles(buf, int(reset)))
    return {name: int(buf[i]) for i, name in enumerate(PHASES)}
