"""Host-side logic of the package (no GPU): loss generators, sharding,
records, API validation, ABI header/library consistency."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2205_11226_b200 import (
    BlockGrid, DimensionMismatchError, ImageBuffer, LossMask, Profile, gen_dispersed_mask, gen_random_mask,
)
from paper_2205_11226_b200.loss import SplitMix64, fisher_yates
from paper_2205_11226_b200.parallel import shard_range
from paper_2205_11226_b200.records import RECORD_DTYPE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def scalar_splitmix(seed, n):
    m = (1 << 64) - 1
    s = seed & m
    out = []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & m
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        out.append(z ^ (z >> 31))
    return out


def test_splitmix_vectorised_matches_scalar():
    for seed in (0, 1, 424242, 2**63 + 5):
        a = SplitMix64(seed).draws(50)
        assert [int(v) for v in a] == scalar_splitmix(seed, 50)
        g = SplitMix64(seed)
        assert [g.next_u64() for _ in range(5)] == scalar_splitmix(seed, 5)


def test_splitmix_known_answer():
    # first outputs of splitmix64(seed=0) (Steele et al. reference values)
    assert scalar_splitmix(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_fisher_yates_is_a_permutation():
    p = fisher_yates(1000, SplitMix64(7))
    assert sorted(p) == list(range(1000))


def test_masks():
    d = gen_dispersed_mask(BlockGrid(64, 64)).states
    assert d.sum() == 4 * 256
    r = gen_random_mask(BlockGrid(64, 48), 0.5, 3).states
    assert (r == 1).sum() == 6 * 256  # round(0.5 * 12) blocks


def test_shard_range_partitions():
    for n in (1, 7, 16, 256):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_types_validate_like_reference():
    with pytest.raises(ValueError):
        LossMask(np.full((4, 4), 3, np.uint8))
    with pytest.raises(ValueError):
        Profile.custom(-1.0, 0.5)
    with pytest.raises(ValueError):
        Profile.custom(10.0, 0.0)
    with pytest.raises(ValueError):
        Profile.named("turbo")
    assert Profile.sentinel().t_nu == float("inf")
    img = ImageBuffer(np.array([[-3.0, 0.5, 254.5, 300.0]]))
    assert img.quantized().tolist() == [[0, 1, 255, 255]]


def test_conceal_image_shape_mismatch():
    from paper_2205_11226_b200 import conceal_image

    with pytest.raises(DimensionMismatchError):
        conceal_image(ImageBuffer(np.zeros((16, 16))), LossMask(np.zeros((16, 17), np.uint8)), Profile.named("express"))


def test_record_dtype_matches_header():
    h = open(os.path.join(ROOT, "include", "blockmend_b200.h")).read()
    assert "64 bytes" in h
    assert RECORD_DTYPE.itemsize == 64


def _header_symbols():
    h = open(os.path.join(ROOT, "include", "blockmend_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(bm_\w+)\(", h, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2205_11226_b200 import _native

    _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)
    # queries that need no device
    lib.bm_abi_version.restype = ctypes.c_int
    assert lib.bm_abi_version() == 1
    lib.bm_status_string.restype = ctypes.c_char_p
    assert b"LOST" in lib.bm_status_string(2)


def test_product_path_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2205_11226_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("no oracle", "").lower() or f == "__init__.py", f
