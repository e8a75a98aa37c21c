"""Patch geometry, scheduling, context extraction and the masked candidate
gather (drop-in for blockmend/framework.py).

Conventions follow the reference (framework.py:1-18): a patch is the 2x2
pixel group at `patch_origin`; its 6x6 window has origin patch_origin - 2;
the context layout is the 32 window offsets outside the patch, row-major;
the support area is the 3x3 block neighbourhood of the patch's block,
clipped to the image; candidate windows are grouped in Chebyshev rings.

The functions that read pixels or states run on the GPU through the C ABI
(csrc/bm_api.cu): extract_target -> bm_extract_targets, the masked gather of
gather_candidates / expand_support -> bm_collect, patch_scores ->
bm_patch_scores, build_schedule -> bm_build_schedule, build_expansion_map ->
bm_expansion_maps.  Only integer bookkeeping (support bounds, pending-patch
lists, ring slicing) stays on the host.  The fused concealment kernel runs
the same semantics per cell without materialising any of these objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import EmptyContextError
from .image import BLOCK_SIZE, BlockGrid, ImageBuffer, LossMask, PixelState

WINDOW = 6
PATCH = 2
PATCH_OFFSETS = np.array([(2, 2), (2, 3), (3, 2), (3, 3)], dtype=np.intp)
CONTEXT_OFFSETS = np.array(
    [(r, c) for r in range(WINDOW) for c in range(WINDOW) if not (2 <= r <= 3 and 2 <= c <= 3)], dtype=np.intp
)
N_CONTEXT = len(CONTEXT_OFFSETS)  # 32
N_PATCH = len(PATCH_OFFSETS)  # 4
MAX_MAP = 2048  # >= 43 * 43 window origins of one support area


def _pixels(img) -> np.ndarray:
    return img.pixels if isinstance(img, ImageBuffer) else np.asarray(img)


def _states(mask) -> np.ndarray:
    return mask.states if isinstance(mask, LossMask) else np.asarray(mask)


@dataclass(frozen=True)
class PatchJob:
    """One 2x2 patch to conceal, with its scheduling score (framework.py:52-57)."""

    patch_origin: tuple[int, int]
    block_id: tuple[int, int]
    reliability: int


@dataclass
class TargetContext:
    """The missing patch plus its usable 6x6 context (framework.py:60-77)."""

    patch_origin: tuple[int, int]
    layout_usable: np.ndarray  # bool per CONTEXT_OFFSETS entry
    y0: np.ndarray  # usable context samples, layout order
    n_y: int
    n_x: int = N_PATCH
    _used_offsets: np.ndarray | None = field(default=None, repr=False)

    def used_offsets(self) -> np.ndarray:
        """Window offsets read for each candidate: usable context, then patch."""
        if self._used_offsets is None:
            self._used_offsets = np.vstack([CONTEXT_OFFSETS[np.asarray(self.layout_usable, bool)], PATCH_OFFSETS])
        return self._used_offsets

    def layout_bits(self) -> int:
        """The usable layout as a 32-bit mask (bit k = CONTEXT_OFFSETS[k]), the C-ABI form."""
        lay = np.asarray(self.layout_usable, bool)
        return sum(1 << k for k in range(N_CONTEXT) if lay[k])


@dataclass
class CandidateSet:
    """Prototype/context pairs gathered from the support area (framework.py:80-91)."""

    x: np.ndarray  # (M', 4)
    y: np.ndarray  # (M', N_y)
    ring_index: int = 0
    exhausted: bool = True

    @property
    def m_current(self) -> int:
        return self.x.shape[0]


@dataclass(frozen=True)
class ExpansionMap:
    """Candidate window origins ordered by (ring, raster position) (framework.py:94-111)."""

    origins: np.ndarray  # (K, 2), sorted
    rings: np.ndarray  # (K,), ascending

    @property
    def max_ring(self) -> int:
        return int(self.rings[-1]) if len(self.rings) else 0

    def ring_slice(self, ring: int) -> tuple[int, int]:
        lo = int(np.searchsorted(self.rings, ring, side="left"))
        hi = int(np.searchsorted(self.rings, ring, side="right"))
        return lo, hi

    def prefix_end(self, rings: int) -> int:
        return int(np.searchsorted(self.rings, rings, side="right"))


def block_origin_of(patch_origin: tuple[int, int]) -> tuple[int, int]:
    r, c = patch_origin
    return (r // BLOCK_SIZE) * BLOCK_SIZE, (c // BLOCK_SIZE) * BLOCK_SIZE


def support_bounds(shape: tuple[int, int], patch_origin: tuple[int, int]):
    """Pixel bounds (r0, r1, c0, c1) of the clipped 3x3 block support (framework.py:119-127)."""
    h, w = shape
    br, bc = block_origin_of(patch_origin)
    return max(0, br - BLOCK_SIZE), min(h, br + 2 * BLOCK_SIZE), max(0, bc - BLOCK_SIZE), min(w, bc + 2 * BLOCK_SIZE)


# ------------------------------------------------------------ device helpers


class _Dev:
    """The current CUDA device, and numpy <-> device copies for one call."""

    def __init__(self):
        self.torch = _native.require_cuda()
        self.dev = self.torch.device("cuda", self.torch.cuda.current_device())
        self.lib = _native.lib()

    def put(self, arr, dtype):
        return self.torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype)).to(self.dev)

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.dev)

    @property
    def stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream


def _image_on_device(d: _Dev, img, mask):
    pixels = np.asarray(_pixels(img), dtype=np.float64)
    states = np.asarray(_states(mask))
    if pixels.shape != states.shape:
        from .errors import DimensionMismatchError

        raise DimensionMismatchError(f"shape mismatch: {pixels.shape} vs {states.shape}")
    return d.put(pixels, np.float64), d.put(states, np.uint8), states.shape


# ------------------------------------------------------------------ geometry


def build_expansion_maps(shape: tuple[int, int], patch_origins) -> list[ExpansionMap]:
    """build_expansion_map for many patch origins in one device call."""
    origins = np.asarray(patch_origins, dtype=np.int32).reshape(-1, 2)
    if len(origins) == 0:
        return []
    h, w = int(shape[0]), int(shape[1])
    d = _Dev()
    t_o = d.put(origins, np.int32)
    k = d.empty((len(origins),), d.torch.int32)
    o = d.empty((len(origins), MAX_MAP, 2), d.torch.int32)
    r = d.empty((len(origins), MAX_MAP), d.torch.int32)
    _native.check(d.lib.bm_expansion_maps(h, w, len(origins), t_o.data_ptr(), k.data_ptr(), o.data_ptr(),
                                          r.data_ptr(), d.stream))
    k, o, r = k.cpu().numpy(), o.cpu().numpy(), r.cpu().numpy()
    return [ExpansionMap(o[i, : k[i]].astype(np.intp), r[i, : k[i]].astype(np.intp)) for i in range(len(origins))]


def build_expansion_map(shape: tuple[int, int], patch_origin: tuple[int, int]) -> ExpansionMap:
    """Window origins of the clipped support in (ring, row, col) order (framework.py:130-148)."""
    return build_expansion_maps(shape, [patch_origin])[0]


# ------------------------------------------------------------------ targets


def extract_targets(img, mask, patch_origins) -> list[TargetContext | None]:
    """extract_target for many patches in one device call; None where the
    context is empty (the single-patch form raises EmptyContextError)."""
    origins = np.asarray(patch_origins, dtype=np.int32).reshape(-1, 2)
    if len(origins) == 0:
        return []
    d = _Dev()
    px, st, (h, w) = _image_on_device(d, img, mask)
    t_o = d.put(origins, np.int32)
    lay = d.empty((len(origins),), d.torch.int32)
    ny = d.empty((len(origins),), d.torch.int32)
    y0 = d.torch.zeros((len(origins), 32), dtype=d.torch.float64, device=d.dev)
    _native.check(d.lib.bm_extract_targets(h, w, px.data_ptr(), st.data_ptr(), len(origins), t_o.data_ptr(),
                                           lay.data_ptr(), ny.data_ptr(), y0.data_ptr(), d.stream))
    lay = lay.cpu().numpy().view(np.uint32)
    ny, y0 = ny.cpu().numpy(), y0.cpu().numpy()
    out = []
    for i in range(len(origins)):
        if ny[i] == 0:
            out.append(None)
            continue
        usable = ((int(lay[i]) >> np.arange(N_CONTEXT)) & 1).astype(bool)
        out.append(TargetContext((int(origins[i, 0]), int(origins[i, 1])), usable, y0[i, : ny[i]].copy(), int(ny[i])))
    return out


def extract_target(img, mask, patch_origin: tuple[int, int]) -> TargetContext:
    """Read the usable context around a patch (framework.py:151-168);
    EmptyContextError if none."""
    t = extract_targets(img, mask, [patch_origin])[0]
    if t is None:
        raise EmptyContextError(f"no usable context around patch {tuple(patch_origin)}")
    return t


# ------------------------------------------------------------------- gather


def _collect_many(img, mask, requests):
    """_collect (framework.py:171-183) for several (target, window origins)
    requests in one bm_collect call; returns [(x, y)] per request."""
    if not requests:
        return []
    counts = np.array([len(o) for _, o in requests], dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    total = int(counts.sum())
    out = []
    if total == 0:
        return [(np.empty((0, N_PATCH)), np.empty((0, t.n_y))) for t, _ in requests]
    d = _Dev()
    px, st, (h, w) = _image_on_device(d, img, mask)
    allo = np.concatenate([np.asarray(o, dtype=np.int32).reshape(-1, 2) for _, o in requests])
    lays = np.array([t.layout_bits() for t, _ in requests], dtype=np.uint32)
    t_o, t_off, t_cnt = d.put(allo, np.int32), d.put(offs, np.int32), d.put(counts, np.int32)
    t_lay = d.put(lays.view(np.int32), np.int32)
    x = d.empty((total, 4), d.torch.float64)
    y = d.empty((total, 32), d.torch.float64)
    m = d.empty((len(requests),), d.torch.int32)
    _native.check(d.lib.bm_collect(h, w, px.data_ptr(), st.data_ptr(), len(requests), t_o.data_ptr(),
                                   t_off.data_ptr(), t_cnt.data_ptr(), t_lay.data_ptr(), x.data_ptr(), y.data_ptr(),
                                   m.data_ptr(), d.stream))
    m, x, y = m.cpu().numpy(), x.cpu().numpy(), y.cpu().numpy()
    for q, (t, _) in enumerate(requests):
        lo = offs[q]
        out.append((x[lo : lo + m[q]].copy(), y[lo : lo + m[q], : t.n_y].copy()))
    return out


def _collect(pixels, states, target: TargetContext, origins: np.ndarray):
    return _collect_many(pixels, states, [(target, origins)])[0]


def gather_candidates(img, mask, target: TargetContext, emap: ExpansionMap, rings: int) -> CandidateSet:
    """All candidates whose window origin lies in rings 1..rings (framework.py:186-195)."""
    if rings < 1:
        raise ValueError("rings must be >= 1")
    end = emap.prefix_end(rings)
    x, y = _collect(img, mask, target, emap.origins[:end])
    reached = min(rings, emap.max_ring)
    return CandidateSet(x, y, ring_index=reached, exhausted=reached >= emap.max_ring)


def expand_support(img, mask, target: TargetContext, emap: ExpansionMap, cset: CandidateSet) -> CandidateSet:
    """Append the next ring's candidates; no-op when already exhausted (framework.py:198-207)."""
    if cset.exhausted:
        return cset
    ring = cset.ring_index + 1
    lo, hi = emap.ring_slice(ring)
    x_new, y_new = _collect(img, mask, target, emap.origins[lo:hi])
    x = np.concatenate([cset.x, x_new]) if cset.m_current else x_new
    y = np.concatenate([cset.y, y_new]) if cset.m_current else y_new
    return CandidateSet(x, y, ring_index=ring, exhausted=ring >= emap.max_ring)


def empty_candidate_set(target: TargetContext, emap: ExpansionMap) -> CandidateSet:
    return CandidateSet(np.empty((0, N_PATCH), dtype=np.float64), np.empty((0, target.n_y), dtype=np.float64),
                        ring_index=0, exhausted=emap.max_ring == 0)


# ----------------------------------------------------------------- schedule


def lost_patch_origins(states: np.ndarray, block_origin: tuple[int, int]) -> list[tuple[int, int]]:
    """Origins of the block's 2x2 patches that still contain a LOST pixel (framework.py:219-227)."""
    states = _states(states)
    br, bc = block_origin
    sub = states[br : br + BLOCK_SIZE, bc : bc + BLOCK_SIZE] == PixelState.LOST
    out = []
    for r in range(0, BLOCK_SIZE, PATCH):
        for c in range(0, BLOCK_SIZE, PATCH):
            if sub[r : r + PATCH, c : c + PATCH].any():
                out.append((br + r, bc + c))
    return out


def patch_scores(states: np.ndarray, pending: list[tuple[int, int]]):
    """(available_count, usable_count) of each pending patch's context (framework.py:230-240)."""
    states = np.asarray(_states(states))
    origins = np.asarray(pending, dtype=np.int32).reshape(-1, 2)
    if len(origins) == 0:
        return np.zeros(0, np.intp), np.zeros(0, np.intp)
    d = _Dev()
    st = d.put(states, np.uint8)
    t_o = d.put(origins, np.int32)
    a = d.empty((len(origins),), d.torch.int32)
    u = d.empty((len(origins),), d.torch.int32)
    _native.check(d.lib.bm_patch_scores(states.shape[0], states.shape[1], st.data_ptr(), len(origins),
                                        t_o.data_ptr(), a.data_ptr(), u.data_ptr(), d.stream))
    return a.cpu().numpy().astype(np.intp), u.cpu().numpy().astype(np.intp)


def pick_next_patch(states: np.ndarray, pending: list[tuple[int, int]]):
    """Most reliable pending patch: max available context, then max usable,
    then raster order (framework.py:243-250)."""
    states = np.asarray(_states(states))
    avail, usable = patch_scores(states, pending)
    origins = np.asarray(pending, dtype=np.intp)
    raster = origins[:, 0] * states.shape[1] + origins[:, 1]
    best = np.lexsort((raster, -usable, -avail))[0]
    return pending[best], int(avail[best])


def build_schedules(mask, block_ids) -> list[list[PatchJob]]:
    """build_schedule for many blocks in one device call (bm_build_schedule)."""
    states = np.asarray(_states(mask))
    grid = BlockGrid(states.shape[1], states.shape[0])
    blocks = [tuple(int(v) for v in b) for b in block_ids]
    for b in blocks:
        grid.block_origin(b)  # validates the block id
    if not blocks:
        return []
    d = _Dev()
    st = d.put(states, np.uint8)
    t_b = d.put(np.asarray(blocks, dtype=np.int32), np.int32)
    n = d.empty((len(blocks),), d.torch.int32)
    o = d.empty((len(blocks), 64, 2), d.torch.int32)
    rel = d.empty((len(blocks), 64), d.torch.int32)
    _native.check(d.lib.bm_build_schedule(states.shape[0], states.shape[1], st.data_ptr(), len(blocks),
                                          t_b.data_ptr(), n.data_ptr(), o.data_ptr(), rel.data_ptr(), d.stream))
    n, o, rel = n.cpu().numpy(), o.cpu().numpy(), rel.cpu().numpy()
    return [[PatchJob((int(o[i, k, 0]), int(o[i, k, 1])), blocks[i], int(rel[i, k])) for k in range(n[i])]
            for i in range(len(blocks))]


def build_schedule(mask, block_id: tuple[int, int]) -> list[PatchJob]:
    """Simulated filling order of one block's lost patches (framework.py:253-274):
    reliability recomputed after each simulated completion, no deferral."""
    return build_schedules(mask, [block_id])[0]
