// bm_common.cuh — constants, geometry and warp/CTA reduction helpers for the
// sm_100a concealment kernels.  Geometry follows the reference's framework.py
// (WINDOW/PATCH 28-29, CONTEXT_OFFSETS 33-36, support_bounds 119-127,
// build_expansion_map 130-148).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef BM_NS
#define BM_NS bm  // bm_conceal_wide.cu compiles the kernels again as bmw with BM_NT=512
#endif

namespace BM_NS {

#ifndef BM_NT
#define BM_NT 256
#endif
constexpr int NT = BM_NT;        // threads per concealment CTA (2 CTAs = 2 cells per SM, 128 regs)
constexpr int NWARP = NT / 32;
#ifndef BM_CS
#define BM_CS 1
#endif
// CTAs per thread-block cluster that share one cell (bm_conceal_cluster.cu):
// every CTA of the cluster runs the cell's control flow on identical data, the
// candidate loops of the HQL pipeline are split over the cluster's warps
// (global warp index rank * NWARP + warp) and the partial results are
// combined over distributed shared memory in rank order, so every CTA holds
// the same bits.  1 = no cluster.
constexpr int CS = BM_CS;
constexpr int GWARPS = CS * NWARP;  // warps sharing a cell's candidate loops
constexpr int BS = 16;           // BLOCK_SIZE (image.py:18)
constexpr int TILE = 48;         // 3x3-cell support area (framework.py:119-127)
#ifndef BM_TS
#define BM_TS 53
#endif
constexpr int TS = BM_TS;        // tile row stride (elements); odd: fewer bank conflicts in the window gathers (A/B 52..60)
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
// Exact warp max / min of doubles with two redux.sync steps on an
// order-preserving 64-bit key (hi word, then lo word) instead of a 5-round
// shuffle butterfly.  NaN lanes are ignored (like fmax / fmin).
__device__ __forceinline__ unsigned long long f64_key(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double f64_unkey(unsigned hi, unsigned lo) {
  const unsigned long long k = ((unsigned long long)hi << 32) | lo;
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}
__device__ __forceinline__ double warp_max(double v) {
  const unsigned long long k = f64_key(v != v ? -INFINITY : v);
  const unsigned h = __reduce_max_sync(FULL, (unsigned)(k >> 32));
  const unsigned l = __reduce_max_sync(FULL, (unsigned)(k >> 32) == h ? (unsigned)k : 0u);
  return f64_unkey(h, l);
}
__device__ __forceinline__ double warp_min(double v) {
  const unsigned long long k = f64_key(v != v ? INFINITY : v);
  const unsigned h = __reduce_min_sync(FULL, (unsigned)(k >> 32));
  const unsigned l = __reduce_min_sync(FULL, (unsigned)(k >> 32) == h ? (unsigned)k : 0xFFFFFFFFu);
  return f64_unkey(h, l);
}
__device__ __forceinline__ float warp_minf(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ int warp_sumi(int v) {
  return (int)__reduce_add_sync(FULL, (unsigned)v);
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

// NumPy's pairwise summation order (numpy/_core/src/umath/loops_utils.h.src
// pairwise_sum: the order of ndarray.sum along a contiguous axis), so BRL
// means, Euclidean distances and the alpha sums are bit-identical to the
// reference for any inputs.  Blocks of <= 128 elements use eight strided
// accumulators; longer runs split at n/2 rounded down to a multiple of 8
// (pairwise_sum_long: one level, n <= 256).
template <typename F>
__device__ __forceinline__ double pairwise_block(int lo, int n, F a) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res += a(lo + i);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = a(lo + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] += a(lo + i + j);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a(lo + i);
  return res;
}
template <typename F>
__device__ __forceinline__ double pairwise_sum_n(int n, F a) {  // n <= 128
  return pairwise_block(0, n, a);
}
template <typename F>
__device__ __forceinline__ double pairwise_sum_long(int n, F a) {  // n <= 256
  if (n <= 128) return pairwise_block(0, n, a);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_block(0, n2, a) + pairwise_block(n2, n - n2, a);
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

// i-th (raster-ordered) candidate patch origin of ring r, branch-free: ring 1
// is the clipped 7x7 square (rows of width w); ring r > 1 is the clipped
// square annulus at Chebyshev distance d = r + 2: its top row, then per middle
// row the left and/or right side entries, then its bottom row.
__device__ __forceinline__ void ring_entry(const RingGeom& g, int r, int i, int& a, int& b) {
  const bool first = r == 1;
  const int d = first ? 3 : r + 2;
  const int b0 = max(g.B0, g.pc - d), b1 = min(g.B1, g.pc + d);
  const int lc0 = max(b1 - b0 + 1, 0), lc = max(lc0, 1);  // row width (lc >= 1 for the division)
  // ring 1: rows of the square
  const int q1 = i / lc;
  const int a_sq = max(g.A0, g.pr - 3) + q1, b_sq = b0 + (i - q1 * lc);
  // annulus
  const int top = (g.pr - d >= g.A0 && g.pr - d <= g.A1) ? lc0 : 0;
  const int m0 = max(g.A0, g.pr - d + 1), m1 = min(g.A1, g.pr + d - 1);
  const int nm = max(m1 - m0 + 1, 0);
  const int lv = (g.pc - d >= g.B0 && g.pc - d <= g.B1), rv = (g.pc + d >= g.B0 && g.pc + d <= g.B1);
  const int per = lv + rv, sh = per >> 1;  // 2 side entries per row: i2 >> 1, i2 & 1
  const int i2 = i - top, i3 = i2 - nm * per;
  const int a_side = m0 + (i2 >> sh), b_side = (lv && (i2 & sh) == 0) ? g.pc - d : g.pc + d;
  a = first ? a_sq : (i2 < 0 ? g.pr - d : (i3 < 0 ? a_side : g.pr + d));
  b = first ? b_sq : (i2 < 0 ? b0 + i : (i3 < 0 ? b_side : b0 + i3));
}

// ---- thread-block cluster / distributed shared memory (CS > 1) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_rank() {
  if constexpr (CS == 1) {
    return 0;
  } else {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
  }
}
// every thread of every CTA of the cluster; release / acquire at cluster scope
__device__ __forceinline__ void cluster_sync_all() {
  if constexpr (CS > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}
// shared::cluster address of `p` (a shared-memory object of this CTA) in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(const void* p, unsigned rank) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(smem_u32(p)), "r"(rank));
  return o;
}
__device__ __forceinline__ double ld_dsmem_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int ld_dsmem_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// exp(a) for the weight kernels (IDL, beta grid, LOO): a = (64k' + j) ln2/64 + r,
// |r| <= ln2/128; e^a = 2^k' * T_j * e^r with T_j = 2^(j/64) as a hi + lo pair
// (80-digit values) and e^r = 1 + q, q a degree-5 Estrin polynomial
// (truncation < 0.3 ulp): T_j e^r = hi + fma(hi, q, lo), ~0.5-1 ulp, ~10 FP64
// ops, no branches.  Arguments below -708 return 0: every weight sum this
// feeds holds a term >= e^-20, so those terms are below half an ulp of it.
__device__ const double g_exp2_64[128] = {  // (hi, lo) pairs; copied to shared memory (EstSmem::exptab)
    0x1.0000000000000p+0, 0x0.0p+0, 0x1.02c9a3e778061p+0, -0x1.19083535b085dp-56,
    0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55, 0x1.0874518759bc8p+0, 0x1.186be4bb284ffp-57,
    0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54, 0x1.0e3ec32d3d1a2p+0, 0x1.03a1727c57b53p-59,
    0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54, 0x1.1429aaea92de0p+0, -0x1.32fbf9af1369ep-54,
    0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55, 0x1.1a35beb6fcb75p+0, 0x1.e5b4c7b4968e4p-55,
    0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54, 0x1.2063b88628cd6p+0, 0x1.dc775814a8495p-55,
    0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54, 0x1.26b4565e27cddp+0, 0x1.2bd339940e9d9p-55,
    0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55, 0x1.2d285a6e4030bp+0, 0x1.0024754db41d5p-54,
    0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55, 0x1.33c08b26416ffp+0, 0x1.32721843659a6p-54,
    0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54, 0x1.3a7db34e59ff7p+0, -0x1.5e436d661f5e3p-56,
    0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55, 0x1.4160a21f72e2ap+0, -0x1.ef3691c309278p-58,
    0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59, 0x1.486a2b5c13cd0p+0, 0x1.3c1a3b69062f0p-56,
    0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56, 0x1.4f9b2769d2ca7p+0, -0x1.4b309d25957e3p-54,
    0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55, 0x1.56f4736b527dap+0, 0x1.9bb2c011d93adp-54,
    0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54, 0x1.5e76f15ad2148p+0, 0x1.ba6f93080e65ep-54,
    0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54, 0x1.6623882552225p+0, -0x1.bb60987591c34p-54,
    0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54, 0x1.6dfb23c651a2fp+0, -0x1.bbe3a683c88abp-57,
    0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55, 0x1.75feb564267c9p+0, -0x1.0245957316dd3p-54,
    0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55, 0x1.7e2f336cf4e62p+0, 0x1.05d02ba15797ep-56,
    0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54, 0x1.868d99b4492edp+0, -0x1.fc6f89bd4f6bap-54,
    0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54, 0x1.8f1ae99157736p+0, 0x1.5cc13a2e3976cp-55,
    0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57, 0x1.97d829fde4e50p+0, -0x1.d185b7c1b85d1p-54,
    0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56, 0x1.a0c667b5de565p+0, -0x1.359495d1cd533p-54,
    0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54, 0x1.a9e6b5579fdbfp+0, 0x1.0fac90ef7fd31p-54,
    0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54, 0x1.b33a2b84f15fbp+0, -0x1.2805e3084d708p-57,
    0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56, 0x1.bcc1e904bc1d2p+0, 0x1.23dd07a2d9e84p-55,
    0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55, 0x1.c67f12e57d14bp+0, 0x1.2884dff483cadp-54,
    0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56, 0x1.d072d4a07897cp+0, -0x1.cbc3743797a9cp-54,
    0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55, 0x1.da9e603db3285p+0, 0x1.c2300696db532p-54,
    0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54, 0x1.e502ee78b3ff6p+0, 0x1.39e8980a9cc8fp-55,
    0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54, 0x1.efa1bee615a27p+0, 0x1.dc7f486a4b6b0p-54,
    0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54, 0x1.fa7c1819e90d8p+0, 0x1.74853f3a5931ep-55,
};
// coefficients in the constant bank (direct DFMA operands, no register moves)
__device__ __constant__ double c_expw[6] = {
    0x1.71547652b82fep+6,                        // 64 / ln2
    0x1.62e4200000000p-7, 0x1.fdf473de6af28p-28,  // ln2 / 64 = hi + lo (hi * k exact for |k| < 2^20)
    0x1.5555555555555p-3, 0x1.1111111111111p-7, 0x1.5555555555555p-5};  // 1/6, 1/120, 1/24
// a <= 709 and a not NaN (the weight arguments in the beta grid and LOO,
// <= 20 by construction); a < -708 -> 0.  tab: the 128 doubles of g_exp2_64
// in shared memory (16-byte aligned).
__device__ __forceinline__ double exp_wn(double a, const double* __restrict__ tab) {
  const double ac = a < -708.0 ? -708.0 : a;
  const double t = fma(ac, c_expw[0], 0x1.8p52);  // round(a * 64 / ln2) in the low word
  const int ki = __double2loint(t);
  const double kd = t - 0x1.8p52;
  double r = fma(kd, -c_expw[1], ac);
  r = fma(kd, -c_expw[2], r);
  const double r2 = r * r;
  const double p23 = fma(r, c_expw[3], 0.5);
  const double p45 = fma(r, c_expw[4], c_expw[5]);
  const double q = fma(r2, fma(r2, p45, p23), r);  // e^r - 1
  const double2 tj = reinterpret_cast<const double2*>(tab)[ki & 63];
  const double v = tj.x + fma(tj.x, q, tj.y);  // in [0.99, 2)
  const double res = __hiloint2double(__double2hiint(v) + ((ki >> 6) << 20), __double2loint(v));  // * 2^(ki>>6)
  return a >= -708.0 ? res : 0.0;
}
// exp_wn without the FP64 compares: the argument clamp and the underflow test
// run on the integer pipe (the rounded exponent k = round(a 64/ln2) is the
// 64-bit difference of t and the shifter, exact while |k| < 2^51); k below
// -1021*64 (a < ~-707.6) -> 0, and so are a = -inf and any a < -2^44.  For
// a <= 25 or -inf; a = +inf / NaN give garbage (callers select them away).
__device__ __forceinline__ double exp_wf(double a, const double* __restrict__ tab) {
  const double t = fma(a, c_expw[0], 0x1.8p52);
  const long long kb = __double_as_longlong(t) - 0x4338000000000000ll;
  const int ki = (int)kb;
  const double kd = t - 0x1.8p52;
  double r = fma(kd, -c_expw[1], a);
  r = fma(kd, -c_expw[2], r);
  const double r2 = r * r;
  const double p23 = fma(r, c_expw[3], 0.5);
  const double p45 = fma(r, c_expw[4], c_expw[5]);
  const double q = fma(r2, fma(r2, p45, p23), r);  // e^r - 1
  const double2 tj = reinterpret_cast<const double2*>(tab)[ki & 63];
  const double v = tj.x + fma(tj.x, q, tj.y);
  const double res = __hiloint2double(__double2hiint(v) + ((ki >> 6) << 20), __double2loint(v));
  return kb >= -1021ll * 64 ? res : 0.0;
}
// general version: NaN stays NaN, overflow -> inf
__device__ __forceinline__ double exp_w(double a, const double* __restrict__ tab) {
  const double res = exp_wn(a, tab);
  return a <= 709.0 ? res : a * INFINITY;
}

}  // namespace BM_NS
