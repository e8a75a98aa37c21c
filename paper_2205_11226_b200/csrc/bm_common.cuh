// bm_common.cuh — constants, geometry and warp/CTA reduction helpers for the
// sm_100a concealment kernels.  Geometry follows the reference's framework.py
// (WINDOW/PATCH 28-29, CONTEXT_OFFSETS 33-36, support_bounds 119-127,
// build_expansion_map 130-148).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bm {

constexpr int NT = 256;          // threads per concealment CTA (2 CTAs = 2 cells per SM, 128 regs)
constexpr int NWARP = NT / 32;
constexpr int BS = 16;           // BLOCK_SIZE (image.py:18)
constexpr int TILE = 48;         // 3x3-cell support area (framework.py:119-127)
constexpr int TS = 52;           // tile row stride (elements); 52 = 4 mod 16 spreads 6x6 windows over banks
constexpr int MAXCAND = 2048;    // >= 43*43 = 1849 window origins per support
constexpr int MAXRING = 27;      // rings 1..26 (+ sentinel)
constexpr int NBETA = 21;        // BETA_GRID = 2^-8 .. 2^12 (estimators.py:32)
constexpr int KMAX = 33;         // min(N_y + 1, M') nearest for alpha (estimators.py:221)
constexpr uint8_t ST_AV = 0, ST_LO = 1, ST_RE = 2;  // PixelState (image.py:21-24)
constexpr unsigned FULL = 0xffffffffu;

// CONTEXT_OFFSETS (framework.py:33-36): row-major 6x6 minus the 2x2 patch.
__host__ __device__ constexpr int ctx_r(int k) {
  return k < 14 ? (k < 6 ? 0 : (k < 12 ? 1 : 2)) : (k < 18 ? (k < 16 ? 2 : 3) : (k < 20 ? 3 : (k < 26 ? 4 : 5)));
}
__host__ __device__ constexpr int ctx_c(int k) {
  // rows 0,1: 6 each; row 2: cols 0,1,4,5; row 3: cols 0,1,4,5; rows 4,5: 6 each
  return k < 12 ? k % 6
                : (k < 16 ? ((k - 12) < 2 ? (k - 12) : (k - 12) + 2)
                          : (k < 20 ? ((k - 16) < 2 ? (k - 16) : (k - 16) + 2) : (k - 20) % 6));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_minf(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ int warp_sumi(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Transposing warp reduction: every lane holds v[0..31]; afterwards lane l
// holds sum over lanes of v[l] (31 shuffles instead of 32*5).  Fixed order,
// hence deterministic.
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const bool hi = lane & 16;
    double send = hi ? v[i] : v[i + 16];
    double keep = hi ? v[i + 16] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const bool hi = lane & 8;
    double send = hi ? v[i] : v[i + 8];
    double keep = hi ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const bool hi = lane & 4;
    double send = hi ? v[i] : v[i + 4];
    double keep = hi ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 4);
  }
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const bool hi = lane & 2;
    double send = hi ? v[i] : v[i + 2];
    double keep = hi ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  {
    const bool hi = lane & 1;
    double send = hi ? v[0] : v[1];
    double keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(FULL, send, 1);
  }
  return v[0];
}

// NumPy's pairwise summation order for n <= 128 elements (the order of
// ndarray.sum along a contiguous axis), so BRL means and Euclidean distances
// are bit-identical to the reference for any inputs.
template <typename F>
__device__ __forceinline__ double pairwise_sum_n(int n, F a) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res += a(i);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = a(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] += a(i + j);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a(i);
  return res;
}

// Chebyshev ring geometry of one patch's expansion map (framework.py:130-148),
// in closed form: ring 1 = candidate patch origins within distance 3, ring r>1
// = the square annulus at distance r+2, each ordered raster-wise and clipped
// to the support rectangle [A0,A1]x[B0,B1] of candidate patch origins.
struct RingGeom {
  int pr, pc;          // target patch origin (absolute)
  int A0, A1, B0, B1;  // candidate patch-origin bounds (absolute, inclusive)
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ int ring_count(const RingGeom& g, int r) {
  if (g.A0 > g.A1 || g.B0 > g.B1) return 0;
  if (r == 1) {
    int a0 = max(g.A0, g.pr - 3), a1 = min(g.A1, g.pr + 3);
    int b0 = max(g.B0, g.pc - 3), b1 = min(g.B1, g.pc + 3);
    return (a1 >= a0 && b1 >= b0) ? (a1 - a0 + 1) * (b1 - b0 + 1) : 0;
  }
  const int d = r + 2;
  int b0 = max(g.B0, g.pc - d), b1 = min(g.B1, g.pc + d);
  int lc = b1 >= b0 ? b1 - b0 + 1 : 0;
  int top = (g.pr - d >= g.A0 && g.pr - d <= g.A1) ? lc : 0;
  int bot = (g.pr + d >= g.A0 && g.pr + d <= g.A1) ? lc : 0;
  int m0 = max(g.A0, g.pr - d + 1), m1 = min(g.A1, g.pr + d - 1);
  int nm = m1 >= m0 ? m1 - m0 + 1 : 0;
  int lv = (g.pc - d >= g.B0 && g.pc - d <= g.B1);
  int rv = (g.pc + d >= g.B0 && g.pc + d <= g.B1);
  return top + nm * (lv + rv) + bot;
}

// i-th (raster-ordered) candidate patch origin of ring r.
__device__ __forceinline__ void ring_entry(const RingGeom& g, int r, int i, int& a, int& b) {
  if (r == 1) {
    int a0 = max(g.A0, g.pr - 3);
    int b0 = max(g.B0, g.pc - 3), b1 = min(g.B1, g.pc + 3);
    int w = b1 - b0 + 1;
    a = a0 + i / w;
    b = b0 + i % w;
    return;
  }
  const int d = r + 2;
  int b0 = max(g.B0, g.pc - d), b1 = min(g.B1, g.pc + d);
  int lc = b1 >= b0 ? b1 - b0 + 1 : 0;
  int top = (g.pr - d >= g.A0 && g.pr - d <= g.A1) ? lc : 0;
  if (i < top) {
    a = g.pr - d;
    b = b0 + i;
    return;
  }
  i -= top;
  int m0 = max(g.A0, g.pr - d + 1), m1 = min(g.A1, g.pr + d - 1);
  int nm = m1 >= m0 ? m1 - m0 + 1 : 0;
  int lv = (g.pc - d >= g.B0 && g.pc - d <= g.B1);
  int rv = (g.pc + d >= g.B0 && g.pc + d <= g.B1);
  int per = lv + rv;
  if (i < nm * per) {
    a = m0 + i / per;
    int j = i % per;
    b = (lv && j == 0) ? g.pc - d : g.pc + d;
    return;
  }
  i -= nm * per;
  a = g.pr + d;
  b = b0 + i;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace bm
