// bm_hql.cuh — the FP64 high-quality layer (hql_estimate, estimators.py:248-286)
// on B200 FP64 tensor cores (mma.sync.m8n8k4.f64, "DMMA").
//
// Every candidate-sized contraction of the reference is a small GEMM with
// K = the candidate count M' (<= 1849):
//   covariance    C   = Zc^T Zc                 (40 x 40, K = M')   estimators.py:140-142
//   quadforms     V   = L^-1 (y0 - Y)^T, d = |V_j|^2 (32 x M')       estimators.py:154-158
//                 (V is consumed in registers; only d leaves the stage)
//   beta grid     P   = W_beta [Y|X|1]          (24 x 40, K = M')   estimators.py:197-206
//   alpha Gram    G   = U_near (y0 - Y)^T, U = C^-1 (y0 - y_near)    estimators.py:225-229
//                 (= V_near^T V), q = d_i + d_j - 2G  (40 x M')
//   LOO sums      Zp  = W_loo [Y|X|1]           (40 x 40, K = M')   estimators.py:231-238
// Warps own disjoint candidate slices (no barrier inside a pass), keep all
// output tiles of their slice in registers, and combine them with one
// fixed-order 3-round tree reduction -> deterministic results.
// The exponentials of the weight matrices are computed in the A-fragment
// registers (each (row, candidate) weight exactly once).
#pragma once
#include "bm_common.cuh"
#include "bm_estimators.cuh"

namespace BM_NS {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Candidate loaders.  Column col of candidate j: columns 0..31 = y (N_y used),
// 32..35 = x, 36 = 1 (sums), 37..39 unused.  A lane resolves its columns once
// into Refs; a fragment element is then one IMAD + one load.

__device__ __forceinline__ double ld_shared_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifndef BM_CNEAR
#define BM_CNEAR 1  // compact (rolled) per-patch code paths; 0 = the unrolled versions (A/B)
#endif
#ifndef BM_BETA_UNROLL
#define BM_BETA_UNROLL 2
#endif
#ifndef BM_COV_UNROLL
#define BM_COV_UNROLL 1
#endif
#ifndef BM_QF_UNROLL
#define BM_QF_UNROLL 1
#endif
#ifndef BM_CTREE
#define BM_CTREE 1
#endif
#ifndef BM_CBETA
#define BM_CBETA 1
#endif
#ifndef BM_LOO_UNROLL
#define BM_LOO_UNROLL 1
#endif
constexpr int kBetaUnroll = BM_BETA_UNROLL, kCovUnroll = BM_COV_UNROLL, kQfUnroll = BM_QF_UNROLL,
              kLooUnroll = BM_LOO_UNROLL;
constexpr int LS = 36;  // stride of Linv / Un: conflict-free A-fragment loads (36 = 4 mod 16)
#ifndef BM_LOO_FAST
#define BM_LOO_FAST 1  // LOO / beta weights: integer-pipe exp underflow and clamp, fused x - xref (A/B)
#endif
#ifndef BM_COV1P
#define BM_COV1P 0  // one-pass covariance about a sampled shift (no means pass) (A/B)
#endif
#ifndef BM_LOO_ROW1
#define BM_LOO_ROW1 0  // LOO: a last row tile holding one real row runs as a SIMT pass (A/B)
#endif
#ifndef BM_NEAR2
#define BM_NEAR2 1  // nearest-set distances two candidates per pass (bit-identical) (A/B)
#endif
#ifndef BM_LINV_N
#define BM_LINV_N 1  // L^-1 substitution stops at row n (bit-identical) (A/B)
#endif
#ifndef BM_LINV_ROLL
#define BM_LINV_ROLL 1  // L^-1 substitution rolled over the rows, columns kept in shared memory (bit-identical) (A/B)
#endif
#ifndef BM_ALPHA_PAR
#define BM_ALPHA_PAR 1  // alpha den / num pairwise sums on 8-lane groups (bit-identical) (A/B)
#endif
#ifndef BM_BETA_PAR
#define BM_BETA_PAR 1  // beta epilogue: the 21 x n residual divisions on all threads (bit-identical) (A/B)
#endif
#ifndef BM_COV_PAR
#define BM_COV_PAR 1  // covariance epilogue: the divisions by m - 1 on all threads (bit-identical) (A/B)
#endif
#ifndef BM_CHOL_TRIM
#define BM_CHOL_TRIM 1  // Cholesky: ridge on the lanes, incremental trailing-block indices, no dead L fill (bit-identical) (A/B)
#endif
#ifndef BM_QF_HOIST
#define BM_QF_HOIST 1  // quadforms: L^-1 A fragments held in registers over the column tiles (N_y <= 24) (A/B)
#endif
#ifndef BM_LOO_HOIST
#define BM_LOO_HOIST 1  // LOO: the pass's U A fragments / nearest index / d_i held in registers over the column tiles (A/B)
#endif
#ifndef BM_CHOL_UNR
#define BM_CHOL_UNR 1  // Cholesky column: the block's dot product unrolled (loads together, same fma order) (A/B)
#endif
#ifndef BM_LINV_PAIR
#define BM_LINV_PAIR 1  // L^-1 substitution two rows per step (shared loads, four chains; bit-identical) (A/B)
#endif
#ifndef BM_TSTAGE
#define BM_TSTAGE 1  // Gram staging / alpha: nearest rows on the lanes, transposed Wt / Vt / R / u (bit-identical) (A/B)
#endif
#ifndef LOO_RR
#define LOO_RR 1  // 8-row tiles of the nearest set per LOO pass over the candidates
#endif

constexpr int RED_HALF = NWARP / 2;
constexpr int RED_CHUNK = 15;                         // tree reductions in chunks of <= 15 values
constexpr int ZP_OFF = RED_HALF * 10 * 32;             // Zp rows after the LOO's 10-value partials
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int R1_SIZE = cmax(cmax(ZP_OFF + KMAX * 40, 2 * 32 * 33), cmax(RED_HALF * RED_CHUNK * 32, MAXCAND));

static_assert(R1_SIZE >= MAXCAND, "HqlSmem::R1 doubles as the IDL exponent buffer");

struct HqlSmem {
  int16_t coff[40];
  double mean[40];
  double Linv[32 * LS];
  double Bm[4 * 32];     // C_XY L^-T
  double cxy[4 * 32];
  double R1[R1_SIZE];    // tree-reduction partials / cyy+L / [ZP_OFF..): Zp rows < 33 / u
  double R2[1600];       // P (24x40) / Un (40x36)
  double wmin[NWARP][40];
  double rdiag[32];
  double dn[40];
  int near[40];
  double cmat[4 * KMAX], rmat[4 * KMAX];
  double xt[4], yt[32];
  double redmin[2][NWARP];
  int redidx[2][NWARP];
  int gbest;
  int fail;
  double nearv[40];                      // the CTA's k-nearest distances (cluster merge)
  double xb[CS > 1 ? 2 * 1024 : 1];      // DSMEM exchange, double-buffered (CS > 1)
};

constexpr int XB_HALF = 1024;

// Cluster-wide fixed-order sum of warp 0's per-lane values v[0..N) (CS > 1):
// each CTA publishes its partial in its exchange buffer, one cluster barrier,
// then warp 0 of every CTA adds the CS partials in rank order over DSMEM, so
// every CTA gets the same bits.  Called by all threads of every CTA; the
// exchange buffer alternates (ph), so one barrier per exchange suffices.
template <int N>
__device__ __forceinline__ void cluster_sum_w0(double (&v)[N], HqlSmem& H, int& ph) {
  static_assert(N * 32 <= XB_HALF, "exchange fits the buffer");
  if constexpr (CS > 1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* b = H.xb + ph * XB_HALF;
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < N; i++) b[i * 32 + lane] = v[i];
    }
    cluster_sync_all();
    if (warp == 0) {
      uint32_t base[CS];
#pragma unroll
      for (int r = 0; r < CS; r++) base[r] = map_rank(b, r) + lane * 8u;
#pragma unroll
      for (int i = 0; i < N; i++) {
        double t = ld_dsmem_f64(base[0] + i * 256u);
#pragma unroll
        for (int r = 1; r < CS; r++) t += ld_dsmem_f64(base[r] + i * 256u);
        v[i] = t;
      }
    }
    ph ^= 1;
  }
}

// per-CTA global scratch (doubles)
constexpr size_t HQL_Z = 0;                                   // dense Z [MAXCAND][40] (estimator API only)
constexpr size_t HQL_SCRATCH_FUSED = 0;                       // the fused kernel needs none
constexpr size_t HQL_SCRATCH_DENSE = HQL_Z + (size_t)MAXCAND * 40;

// Dispatch on the number of 8-wide column tiles that hold the n used context
// values (NA = ceil(n/8), 2..4; n <= 8 runs as 2): the DMMA loops skip the
// tiles that only see zero padding (exact: their products are zeros or feed
// outputs nobody reads), ~30% fewer DMMAs at the typical n = 12..24.
template <int V>
struct IntC {
  static constexpr int value = V;
};
template <class F>
__device__ __forceinline__ void with_na(int n, F&& f) {
  const int na = (n + 7) >> 3;
  if (na <= 2) f(IntC<2>{});
  else if (na == 3) f(IntC<3>{});
  else f(IntC<4>{});
}

// Warp-wide minimum of (v, j) pairs, v >= 0 or +inf (no NaN), ties to the
// smaller j: three redux.sync steps on the order-preserving bit pattern
// (hi word, lo word, index) instead of a 5-round shuffle butterfly.  Returns v
// and the winning j (all lanes).
__device__ __forceinline__ double warp_argmin_key(double v, int j, int& jmin) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned mh = __reduce_min_sync(FULL, hi);
  const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xFFFFFFFFu);
  jmin = (int)__reduce_min_sync(FULL, (hi == mh && lo == ml) ? (unsigned)j : 0x7FFFFFFFu);
  return __hiloint2double((int)mh, (int)ml);
}

// Fixed-order tree reduction of per-warp register tiles (NWARP warps -> warp 0)
// in chunks of C values; red must hold (NWARP/2) * C * 32 doubles.
template <int N, int C = N>
__device__ __forceinline__ void tree_reduce(double (&acc)[N], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += C) {
#if BM_CTREE
#pragma unroll 1  // rolled over the levels: one copy of the chunk code
#else
#pragma unroll
#endif
    for (int half = NWARP / 2; half >= 1; half >>= 1) {
      __syncthreads();
      if (warp >= half && warp < 2 * half) {
#pragma unroll
        for (int i = 0; i < C; i++)
          if (c0 + i < N) red[((warp - half) * C + i) * 32 + lane] = acc[c0 + i];
      }
      __syncthreads();
      if (warp < half) {
#pragma unroll
        for (int i = 0; i < C; i++)
          if (c0 + i < N) acc[c0 + i] += red[(warp * C + i) * 32 + lane];
      }
    }
  }
}

// Fused kernel: candidates are window origins cand[j] in the shared support tile.
struct TileLoader {
  const double* tile;    // shared
  const uint16_t* cand;  // shared
  __device__ __forceinline__ int base(int j) const { return cand[j]; }
  // shared-space byte address of the column at window origin 0 (1 register).
  // Constant columns (y beyond n, the ones column 36, 37..39) alias a real
  // tile column: every consumer either ignores those outputs, multiplies
  // them by exact zeros (U / L^-1 vanish beyond n), or substitutes the ones
  // column itself (ONES_COL).
  using Ref = uint32_t;
  __device__ __forceinline__ Ref ref(const HqlSmem& H, int col) const {
    const int off = H.coff[col];
    return smem_addr(tile + (off >= 0 ? off : 0));
  }
  __device__ __forceinline__ double at(Ref r, int b) const {
    return *(const double*)__cvta_shared_to_generic((size_t)(r + (uint32_t)b * 8u));
  }
};
constexpr int ONES_COL = 36;  // Z column of ones: its weighted sum is the weight total

// Estimator API: dense Z [m][40] in global memory (all 40 columns stored).
struct DenseLoader {
  const double* Z;
  __device__ __forceinline__ int base(int j) const { return j * 40; }
  using Ref = const double*;
  __device__ __forceinline__ Ref ref(const HqlSmem&, int col) const { return Z + col; }
  __device__ __forceinline__ double at(Ref r, int b) const { return r[b]; }
};

// Column table of the Z view for target layout n (uoff: tile offsets of the
// n usable context positions; nullptr for the dense layout).
__device__ __forceinline__ void hql_columns(HqlSmem& H, int n, const int16_t* uoff) {
  const int t = threadIdx.x;
  if (t < 40) {
    int16_t off = -1;
    if (t < n) off = uoff ? uoff[t] : (int16_t)t;
    else if (t >= 32 && t < 36) {
      const int q = t - 32;
      off = uoff ? (int16_t)((2 + (q >> 1)) * TS + 2 + (q & 1)) : (int16_t)t;
    }
    H.coff[t] = off;
  }
}

// The HQL pipeline for one patch.  Inputs: zv (candidates), m >= 2, n, y0
// (shared, [32]).  Outputs in H/out: ok, vals[4], beta, alpha, gap.
// Per-phase cycle accounting of the HQL pipeline and the patch loop (thread 0,
// after barriers); read back with bm_debug_phase_cycles.  Phase 0 =
// everything before HQL.  Compiled in only for diagnostic builds
// (-DBM_DIAG=1: tools/build_variant.sh + BM_NATIVE_VARIANT); the product
// build carries no per-patch global atomics.
__device__ unsigned long long g_phase_cycles[48];
#if BM_DIAG
#define BM_DIAG_ADD(k, v) atomicAdd(&g_phase_cycles[k], (unsigned long long)(v))
#define BM_PHASE(k)                                 \
  do {                                              \
    if (threadIdx.x == 0) {                         \
      const long long now_ = clock64();             \
      BM_DIAG_ADD(k, now_ - ph_t);                  \
      ph_t = now_;                                  \
    }                                               \
  } while (0)
#else
#define BM_DIAG_ADD(k, v) ((void)0)
#define BM_PHASE(k) ((void)0)
#endif

struct HqlOut {
  double vals[4];
  double beta, alpha;
  float gap;
  int ok;
};

template <class ZL>
__device__ void hql_mma(const ZL& zv, int m, int n, const double* y0, HqlSmem& H, double* __restrict__ gs,
                        HqlOut& out, const double* exptab, double* dS) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  long long ph_t = clock64();
  const int nks = (m + 3) >> 2;  // k-steps of 4 candidates
  const int nct = (m + 7) >> 3;  // column tiles of 8 candidates
  // candidate loops run over the cluster's warps (CS = 1: this CTA's warps)
  const unsigned rank = cluster_rank();
  const int gw = (int)rank * NWARP + warp;
  int xph = 0;  // exchange-buffer phase (cluster_sum_w0)

  // ---------------------------------------------------------------- means
#if BM_COV1P
  // one-pass covariance (below) about a shift s: the mean of the first
  // min(m, 32) candidates (warp 0; every CTA of a cluster gets the same bits).
  // C = (D - S S^T / m) / (m - 1) with D = sum (z - s)(z - s)^T and S =
  // sum (z - s) from the same DMMA pass; |mean - s| is a fraction of the
  // spread, so the correction does not cancel digits.
  if (warp == 0) {
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    const typename ZL::Ref c0 = zv.ref(H, lane), c1 = zv.ref(H, lane < 8 ? 32 + lane : 37);
    const int ms = min(m, 32);
    for (int j = 0; j < ms; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        if (j + u < ms) {
          const int b = zv.base(j + u);
          a0[u] += zv.at(c0, b);
          a1[u] += zv.at(c1, b);
        }
      }
    }
    H.mean[lane] = ((a0[0] + a0[1]) + (a0[2] + a0[3])) / ms;
    if (lane < 8) H.mean[32 + lane] = ((a1[0] + a1[1]) + (a1[2] + a1[3])) / ms;
  }
  __syncthreads();
  BM_PHASE(1);
#else
  {
    // 4 independent accumulator pairs per lane (loads overlap), fixed-order combine
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    const typename ZL::Ref c0 = zv.ref(H, lane), c1 = zv.ref(H, lane < 8 ? 32 + lane : 37);
    int j = gw;
    for (; j + 3 * GWARPS < m; j += 4 * GWARPS) {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int b = zv.base(j + u * GWARPS);
        a0[u] += zv.at(c0, b);
        a1[u] += zv.at(c1, b);
      }
    }
#pragma unroll
    for (int u = 0; u < 3; u++) {  // tail: j + 3 GWARPS >= m
      if (j + u * GWARPS < m) {
        const int b = zv.base(j + u * GWARPS);
        a0[u] += zv.at(c0, b);
        a1[u] += zv.at(c1, b);
      }
    }
    a0[0] = (a0[0] + a0[1]) + (a0[2] + a0[3]);
    a1[0] = (a1[0] + a1[1]) + (a1[2] + a1[3]);
    H.wmin[warp][lane] = a0[0];
    if (lane < 8) H.wmin[warp][32 + lane] = a1[0];
    __syncthreads();
    if constexpr (CS == 1) {
      if (tid < 40) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NWARP; w++) s += H.wmin[w][tid];
        H.mean[tid] = s / m;  // z.mean(axis=0)
      }
    } else {
      double v[2] = {0.0, 0.0};  // warp 0: columns lane and 32 + lane
      if (warp == 0) {
#pragma unroll
        for (int w = 0; w < NWARP; w++) {
          v[0] += H.wmin[w][lane];
          if (lane < 8) v[1] += H.wmin[w][32 + lane];
        }
      }
      cluster_sum_w0<2>(v, H, xph);
      if (warp == 0) {
        H.mean[lane] = v[0] / m;
        if (lane < 8) H.mean[32 + lane] = v[1] / m;
      }
    }
    __syncthreads();
    BM_PHASE(1);
  }

#endif

  // ------------------------------------------------- covariance (DMMA)
  {
    typename ZL::Ref cr[5];
    double mu[5];
#pragma unroll
    for (int tl = 0; tl < 5; tl++) {
      const int col = 8 * tl + g;
      cr[tl] = zv.ref(H, col);
      mu[tl] = H.mean[col];
    }
    constexpr int NCACC = BM_COV1P ? 30 : 28;  // (+ the (x|1, x|1) tile: the sums S of the x columns)
    double acc[NCACC];
#pragma unroll
    for (int i = 0; i < NCACC; i++) acc[i] = 0.0;
    // software pipeline: the next k-step's fragments load during this step's MMAs
    with_na(n, [&](auto NAc) {
    constexpr int NA = decltype(NAc)::value;
    double f[5], fn[5];
    auto load_f = [&](int s, double(&o)[5]) {
      const int j = 4 * s + t4;
      const bool valid = j < m;
      const int b = zv.base(min(j, m - 1));  // clamped: branch-free loads
#pragma unroll
      for (int tl = 0; tl < 5; tl++) {
        if (tl >= NA && tl < 4) {
          o[tl] = 0.0;
          continue;
        }
        const double raw = zv.at(cr[tl], b);
        o[tl] = valid ? raw - mu[tl] : 0.0;
      }
      if (BM_COV1P && g == ONES_COL - 32) o[4] = valid ? 1.0 : 0.0;  // column of ones: S = sum (z - s)
    };
    load_f(gw, f);
#pragma unroll kCovUnroll
    for (int s = gw; s < nks; s += GWARPS) {
      load_f(s + GWARPS, fn);
      int idx = 0;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int bb = a; bb < 5; bb++) {
          if (a < NA && (bb < NA || bb == 4)) dmma(acc[2 * idx], acc[2 * idx + 1], f[a], f[bb]);
          idx++;
        }
      if (BM_COV1P) dmma(acc[NCACC - 2], acc[NCACC - 1], f[4], f[4]);
#pragma unroll
      for (int tl = 0; tl < 5; tl++) f[tl] = fn[tl];
    }
    });
    tree_reduce<NCACC, NCACC / 2>(acc, H.R1);
    cluster_sum_w0<NCACC>(acc, H, xph);
    double* cyy = H.R1 + R1_SIZE - 2 * 32 * 33;  // tail of R1 (partials no longer needed)
    double* L = cyy + 32 * 33;
#if BM_COV_PAR && !BM_COV1P
    // C = acc / (m - 1): warp 0 stages the 28 reduced tile halves, then all
    // threads do one division each and scatter into cyy / cxy (one more
    // barrier instead of 28 divisions per lane on warp 0)
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < NCACC; i++) H.R2[i * 32 + lane] = acc[i];  // (R2 is free until the nearest-set merge)
    }
    __syncthreads();
    for (int o = tid; o < NCACC * 32; o += NT) {
      const int vi = o >> 5, ln = o & 31;
      const int tile = vi >> 1, e = vi & 1;
      const int a = tile < 5 ? 0 : (tile < 9 ? 1 : (tile < 12 ? 2 : 3));
      const int bb = tile - (a == 0 ? 0 : (a == 1 ? 5 : (a == 2 ? 9 : 12))) + a;
      const int ra = 8 * a + (ln >> 2), cb = 8 * bb + 2 * (ln & 3) + e;
      const double v = H.R2[o] / (double)(m - 1);
      if (bb < 4) {
        if (ra < n && cb < n && ra <= cb) {
          cyy[ra * 33 + cb] = v;
          cyy[cb * 33 + ra] = v;
        }
      } else if (cb < 36 && ra < n) {
        H.cxy[(cb - 32) * 32 + ra] = v;
      }
    }
#else
    __syncwarp();
    if (warp == 0) {
      const double inv = 1.0 / (double)(m - 1);
#if BM_COV1P
      // S from the ones column (C column 36: lanes t4 == 2, element 0)
      double* Ssum = H.wmin[0];
      if (t4 == 2) {
        int id = 0;
#pragma unroll
        for (int a = 0; a < 4; a++) {
          id += 5 - a;  // tiles (a, a..4): idx of tile (a, 4) = id - 1
          Ssum[8 * a + g] = acc[2 * (id - 1)];
        }
        Ssum[32 + g] = acc[NCACC - 2];
      }
      __syncwarp();
#endif
      int idx = 0;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int bb = a; bb < 5; bb++) {
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int ra = 8 * a + g, cb = 8 * bb + 2 * t4 + e;
#if BM_COV1P
            const double v = fma(-Ssum[ra], Ssum[cb] / m, acc[2 * idx + e]) / (double)(m - 1);
#else
            const double v = acc[2 * idx + e] / (double)(m - 1);
#endif
            if (bb < 4) {
              if (ra < n && cb < n && ra <= cb) {
                cyy[ra * 33 + cb] = v;
                cyy[cb * 33 + ra] = v;
              }
            } else if (cb < 36 && ra < n) {
              H.cxy[(cb - 32) * 32 + ra] = v;
            }
          }
          idx++;
        }
      (void)inv;
    }
#endif
    __syncthreads();
    BM_PHASE(2);
    // ridge (estimators.py:148-150) and Cholesky (CovarianceBlocks._factor) on
    // warp 0; meanwhile warps 1..7 compute the Euclidean distances in NumPy's
    // order (optimize_alpha's nearest set, estimators.py:222)
    if (warp == 0) {
#if BM_CHOL_TRIM
      double ridge = 0.0;
      if (lane == 0) {
        const double tr = pairwise_sum_n(n, [&](int i) { return cyy[i * 33 + i]; });
        ridge = tr > 0.0 ? 1e-6 * tr / n : 1e-6;
      }
      ridge = __shfl_sync(FULL, ridge, 0);
      if (lane < n) cyy[lane * 33 + lane] += ridge;  // lane i: diagonal entry i
#else
      if (lane == 0) {
        const double tr = pairwise_sum_n(n, [&](int i) { return cyy[i * 33 + i]; });
        const double ridge = tr > 0.0 ? 1e-6 * tr / n : 1e-6;
        for (int i = 0; i < n; i++) cyy[i * 33 + i] += ridge;
      }
#endif
      __syncwarp();
      // Blocked right-looking Cholesky (8-column blocks) on warp 0: within a
      // block, lanes are rows and dot products run over the block's columns
      // only; the trailing update applies the block's rank-8 correction.
      bool fail = false;
      for (int c0 = 0; c0 < n && !fail; c0 += 8) {
        const int c1 = min(n, c0 + 8);
        for (int j = c0; j < c1; j++) {
          double t = 0.0;
          if (lane >= j && lane < n) {
            t = cyy[lane * 33 + j];
#if BM_CHOL_UNR
            // (the block's <= 7 earlier columns: loads issued together, the fma chain in the same order)
#pragma unroll
            for (int kk = 0; kk < 7; kk++)
              if (c0 + kk < j) t = fma(-L[lane * 33 + c0 + kk], L[j * 33 + c0 + kk], t);
#else
            for (int k = c0; k < j; k++) t = fma(-L[lane * 33 + k], L[j * 33 + k], t);
#endif
          }
          const double sd = __shfl_sync(FULL, t, j);
          if (!(sd > 0.0)) { fail = true; break; }
          const double rs = rsqrt(sd);  // 1 / L_jj
          if (lane == j) {
            L[j * 33 + j] = sd * rs;
            H.rdiag[j] = rs;
          }
          if (lane > j && lane < n) L[lane * 33 + j] = t * rs;
          __syncwarp();
        }
        if (fail) break;
        // trailing update A[i][jj] -= sum_{k in block} L[i][k] L[jj][k], c1 <= jj <= i < n
        const int rem = n - c1;
#if BM_CHOL_TRIM
        if (rem > 0) {
          // element e = lane + 32 s of the rem x rem trailing block: (row, col)
          // advanced incrementally (one division per block, not two per element)
          const int qd = 32 / rem, qm = 32 % rem;
          int ri = lane / rem, ci = lane % rem;
          for (int e = lane; e < rem * rem; e += 32) {
            if (ci <= ri) {
              const int i = c1 + ri, jj = c1 + ci;
              double t = cyy[i * 33 + jj];
#pragma unroll
              for (int k = 0; k < 8; k++)
                if (c0 + k < c1) t = fma(-L[i * 33 + c0 + k], L[jj * 33 + c0 + k], t);
              cyy[i * 33 + jj] = t;
            }
            ri += qd;
            ci += qm;
            if (ci >= rem) {
              ci -= rem;
              ri++;
            }
          }
        }
#else
        for (int e = lane; e < rem * rem; e += 32) {
          const int i = c1 + e / rem, jj = c1 + e % rem;
          if (jj > i) continue;
          double t = cyy[i * 33 + jj];
#pragma unroll
          for (int k = 0; k < 8; k++)
            if (c0 + k < c1) t = fma(-L[i * 33 + c0 + k], L[jj * 33 + c0 + k], t);
          cyy[i * 33 + jj] = t;
        }
#endif
        __syncwarp();
      }
#if !(BM_CHOL_TRIM && BM_LINV_ROLL)  // (the rolled L^-1 reads only L's lower triangle below row n)
      // the factor's lower triangle is complete; clear the upper part
      for (int j = 0; j < n; j++)
        if (lane < j) L[lane * 33 + j] = 0.0;
      // identity beyond n
      for (int j = n; j < 32; j++) {
        L[lane * 33 + j] = lane == j ? 1.0 : 0.0;
        if (lane == j) H.rdiag[j] = 1.0;
      }
      if (lane >= n)
        for (int j = 0; j < n; j++) L[lane * 33 + j] = 0.0;
#endif
      __syncwarp();
      if (lane == 0) {
        H.fail = fail;
        BM_DIAG_ADD(13, (clock64() - ph_t));  // Cholesky alone (diagnostic)
      }
      // L^-1 in registers: lane c builds column c by forward substitution
      // (L rows read as shared-memory broadcasts); identity beyond n
      // (rows i >= n are identity rows: they never feed rows < n and are
      // stored as zeros, so the substitution stops at n)
#if BM_LINV_ROLL
      // rolled over the rows: column `lane` lives in H.Linv itself (a lane
      // reads back only its own earlier stores), the even / odd partial sums
      // as in the unrolled form - the same bits in ~40 instructions instead
      // of ~1300 straight-line ones per patch (instruction fetch)
#if BM_LINV_PAIR
      // two rows per step (i even): rows i and i + 1 share the loads of the
      // earlier rows' entries x_k, k < i, and run four independent fma chains;
      // row i + 1 then adds its k = i term last, as the one-row loop does
      int i = 0;
#pragma unroll 1
      for (; i + 1 < n; i += 2) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 2
        for (int k = 0; k + 1 < i; k += 2) {
          const double x0 = H.Linv[k * LS + lane], x1 = H.Linv[(k + 1) * LS + lane];
          a0 = fma(L[i * 33 + k], x0, a0);
          a1 = fma(L[i * 33 + k + 1], x1, a1);
          b0 = fma(L[(i + 1) * 33 + k], x0, b0);
          b1 = fma(L[(i + 1) * 33 + k + 1], x1, b1);
        }
        const double rd0 = H.rdiag[i], rd1 = H.rdiag[i + 1];
        const double xi = lane > i ? 0.0 : (lane == i ? rd0 : -(a0 + a1) * rd0);
        H.Linv[i * LS + lane] = xi;
        b0 = fma(L[(i + 1) * 33 + i], xi, b0);
        H.Linv[(i + 1) * LS + lane] = lane > i + 1 ? 0.0 : (lane == i + 1 ? rd1 : -(b0 + b1) * rd1);
      }
      if (i < n) {  // the last row of an odd n (i even: its k < i terms pair up)
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 2
        for (int k = 0; k + 1 < i; k += 2) {
          s0 = fma(L[i * 33 + k], H.Linv[k * LS + lane], s0);
          s1 = fma(L[i * 33 + k + 1], H.Linv[(k + 1) * LS + lane], s1);
        }
        const double rdi = H.rdiag[i];
        H.Linv[i * LS + lane] = lane > i ? 0.0 : (lane == i ? rdi : -(s0 + s1) * rdi);
      }
#else
#pragma unroll 1
      for (int i = 0; i < n; i++) {
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
#pragma unroll 2
        for (; k + 1 < i; k += 2) {
          s0 = fma(L[i * 33 + k], H.Linv[k * LS + lane], s0);
          s1 = fma(L[i * 33 + k + 1], H.Linv[(k + 1) * LS + lane], s1);
        }
        if (k < i) s0 = fma(L[i * 33 + k], H.Linv[k * LS + lane], s0);
        const double rdi = H.rdiag[i];
        H.Linv[i * LS + lane] = lane > i ? 0.0 : (lane == i ? rdi : -(s0 + s1) * rdi);  // (lanes >= n: zeros)
      }
#endif
      if (lane == 0) BM_DIAG_ADD(38, (clock64() - ph_t));  // + L^-1 (diagnostic)
      for (int i = n; i < 32; i++) H.Linv[i * LS + lane] = 0.0;  // zero beyond n
      if (lane == 0) BM_DIAG_ADD(39, (clock64() - ph_t));  // + Linv stored (diagnostic)
#else
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; i++) {
        x[i] = 0.0;
        if (!BM_LINV_N || i < n) {  // warp-uniform
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int k = 0; k < i; k++) {
            const double lik = L[i * 33 + k];
            if (k & 1) s1 = fma(lik, x[k], s1);
            else s0 = fma(lik, x[k], s0);
          }
          const double rdi = H.rdiag[i];
          x[i] = lane > i ? 0.0 : (lane == i ? rdi : -(s0 + s1) * rdi);
        }
      }
      if (lane == 0) BM_DIAG_ADD(38, (clock64() - ph_t));  // + L^-1 (diagnostic)
#pragma unroll
      for (int i = 0; i < 32; i++) H.Linv[i * LS + lane] = (i < n && lane < n) ? x[i] : 0.0;  // zero beyond n
      if (lane == 0) BM_DIAG_ADD(39, (clock64() - ph_t));  // + Linv stored (diagnostic)
#endif
    } else {
      // warps 1..7: Euclidean distances in NumPy's order and the stable
      // k-nearest selection (optimize_alpha, estimators.py:221-223)
      // (CS > 1: this CTA takes the candidates j = l * CS + rank)
      constexpr int NW7 = NT - 32, PER = (MAXCAND / CS + NW7 - 1) / NW7;
      const int t7 = tid - 32, w7 = warp - 1;
      double ev[PER];
      // dist2 = ((y - y0) ** 2).sum(axis=1) in NumPy's pairwise order: eight
      // strided accumulators r[g] (dims g, g+8, ...) below n8 = n - n % 8, the
      // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree, then the tail dims in order
      // (n < 8: tail only).  One candidate per thread, read from the tile.
      // Column refs and y0 are shared-memory broadcasts.
      const int n8 = n - (n % 8);
#if BM_CNEAR && BM_NEAR2
      // two candidates per pass: the column offsets and y0 are loaded once
      // for both; each candidate keeps NumPy's order (the same operations as
      // the one-candidate form below, so the same bits)
#pragma unroll 1
      for (int i = 0; i < PER; i += 2) {
        const int ja = (t7 + i * NW7) * CS + (int)rank;
        const int jb = (t7 + (i + 1) * NW7) * CS + (int)rank;
        if (ja < m) {
          const bool hb = i + 1 < PER && jb < m;
          const int ba = zv.base(ja), bb = zv.base(hb ? jb : ja);
          double ra[8], rb[8];
#pragma unroll
          for (int q = 0; q < 8; q++) ra[q] = rb[q] = 0.0;
#pragma unroll 1
          for (int q0 = 0; q0 < n8; q0 += 8)
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const typename ZL::Ref rq = zv.ref(H, q0 + q);
              const double yq = y0[q0 + q];
              const double da = __dsub_rn(zv.at(rq, ba), yq), db = __dsub_rn(zv.at(rq, bb), yq);
              ra[q] = __dadd_rn(ra[q], __dmul_rn(da, da));
              rb[q] = __dadd_rn(rb[q], __dmul_rn(db, db));
            }
          double ea = __dadd_rn(__dadd_rn(__dadd_rn(ra[0], ra[1]), __dadd_rn(ra[2], ra[3])),
                                __dadd_rn(__dadd_rn(ra[4], ra[5]), __dadd_rn(ra[6], ra[7])));
          double eb = __dadd_rn(__dadd_rn(__dadd_rn(rb[0], rb[1]), __dadd_rn(rb[2], rb[3])),
                                __dadd_rn(__dadd_rn(rb[4], rb[5]), __dadd_rn(rb[6], rb[7])));
#pragma unroll 1
          for (int q = n8; q < n; q++) {
            const typename ZL::Ref rq = zv.ref(H, q);
            const double yq = y0[q];
            const double da = __dsub_rn(zv.at(rq, ba), yq), db = __dsub_rn(zv.at(rq, bb), yq);
            ea = __dadd_rn(ea, __dmul_rn(da, da));
            eb = __dadd_rn(eb, __dmul_rn(db, db));
          }
          dS[ja] = ea;
          if (hb) dS[jb] = eb;
        }
      }
#else
#if BM_CNEAR
      // rolled over the thread's candidates (compact code); each thread
      // stages its own distances in dS (free until the quadforms)
#pragma unroll 1
#else
#pragma unroll
#endif
      for (int i = 0; i < PER; i++) {
        const int j = (t7 + i * NW7) * CS + (int)rank;
#if !BM_CNEAR
        ev[i] = INFINITY;
#endif
        if (j < m) {
          const int b = zv.base(j);
          auto sq = [&](int q) {
            const double d = __dsub_rn(zv.at(zv.ref(H, q), b), y0[q]);
            return __dmul_rn(d, d);
          };
          double r[8];
#pragma unroll
          for (int q = 0; q < 8; q++) r[q] = 0.0;
#pragma unroll 1
          for (int q0 = 0; q0 < n8; q0 += 8)
#pragma unroll
            for (int q = 0; q < 8; q++) r[q] = __dadd_rn(r[q], sq(q0 + q));
          double e = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll 1
          for (int q = n8; q < n; q++) e = __dadd_rn(e, sq(q));
#if BM_CNEAR
          dS[j] = e;
#else
          ev[i] = e;
#endif
        }
      }
#endif  // BM_CNEAR && BM_NEAR2
#if BM_CNEAR
#pragma unroll
      for (int i = 0; i < PER; i++) {
        const int j = (t7 + i * NW7) * CS + (int)rank;
        ev[i] = j < m ? dS[j] : INFINITY;
      }
#endif
      const int k = min(n + 1, m);
      // (1) per-thread sort of its PER candidates by (e2, index)
      int ej[PER];
#pragma unroll
      for (int i = 0; i < PER; i++) ej[i] = (t7 + i * NW7) * CS + (int)rank;
#pragma unroll
      for (int pass = 0; pass < PER; pass++)
#pragma unroll
        for (int i = pass & 1; i + 1 < PER; i += 2) {
          const bool sw = ev[i + 1] < ev[i] || (ev[i + 1] == ev[i] && ej[i + 1] < ej[i]);
          const double lo_v = sw ? ev[i + 1] : ev[i], hi_v = sw ? ev[i] : ev[i + 1];  // branch-free swap
          const int lo_j = sw ? ej[i + 1] : ej[i], hi_j = sw ? ej[i] : ej[i + 1];
          ev[i] = lo_v;
          ev[i + 1] = hi_v;
          ej[i] = lo_j;
          ej[i + 1] = hi_j;
        }
      if (tid == 32) BM_DIAG_ADD(35, (clock64() - ph_t));  // sorted (diag)
      // (2) each warp merges its 32 sorted lanes into its k smallest
      double* lv = H.R2;                           // [NWARP-1][KMAX] values
      int* lj = reinterpret_cast<int*>(H.R2 + (NWARP - 1) * KMAX);  // [NWARP-1][KMAX] indices
      for (int it = 0; it < k; it++) {
        int bj;
        const double bv = warp_argmin_key(ev[0], ej[0], bj);
        if (lane == 0) {
          lv[w7 * KMAX + it] = bv;
          lj[w7 * KMAX + it] = bj;
        }
        if (ej[0] == bj) {  // pop the winner's head
#pragma unroll
          for (int i = 0; i + 1 < PER; i++) {
            ev[i] = ev[i + 1];
            ej[i] = ej[i + 1];
          }
          ev[PER - 1] = INFINITY;
          ej[PER - 1] = 0x7fffffff;
        }
      }
      if (tid == 32) BM_DIAG_ADD(36, (clock64() - ph_t));  // warp merged (diag)
      asm volatile("bar.sync 1, %0;" ::"r"(NW7) : "memory");  // warps 1..NWARP-1
      if (tid == 32) BM_DIAG_ADD(37, (clock64() - ph_t));  // all merged (diag)
      // (3) warp 1 merges the NWARP-1 sorted lists: lane w holds list w's head
      if (w7 == 0) {
        int ptr = 0;
        for (int it = 0; it < k; it++) {
          const double hv = (lane < NWARP - 1 && ptr < k) ? lv[lane * KMAX + ptr] : INFINITY;
          const int myj = (lane < NWARP - 1 && ptr < k) ? lj[lane * KMAX + ptr] : 0x7fffffff;
          int bj;
          const double bv = warp_argmin_key(hv, myj, bj);
          if (lane == 0) {
            H.near[it] = bj;
            H.nearv[it] = bv;
          }
          if (myj == bj && lane < NWARP - 1) ptr++;
        }
        if (lane == 0) BM_DIAG_ADD(8, (clock64() - ph_t));  // nearest side (diagnostic)
      }
    }
    __syncthreads();
    if constexpr (CS > 1) {
      // the cluster's k nearest: merge the CS CTAs' sorted (distance, index)
      // lists over DSMEM, identically in every CTA (ties -> smaller index)
      const int k = min(n + 1, m);
      double* b = H.xb + xph * XB_HALF;
      if (tid < k) {
        b[tid] = H.nearv[tid];
        b[KMAX + tid] = (double)H.near[tid];
      }
      cluster_sync_all();
      if (warp == 0) {
        // copy the CS sorted lists in one DSMEM round trip, then rank every
        // entry: its position in its own list + the entries of the other
        // lists that precede it in the (distance, index) order (a total
        // order: the lists hold disjoint candidates); the first k ranks are
        // the cluster's k nearest, the same set and order as a head-by-head
        // merge
        double* cv = H.R2;                                       // [CS][KMAX]
        int* cj = reinterpret_cast<int*>(H.R2 + CS * KMAX);       // [CS][KMAX]
#pragma unroll
        for (int r = 0; r < CS; r++) {
          const uint32_t base = map_rank(b, r);
          for (int e = lane; e < k; e += 32) {
            cv[r * KMAX + e] = ld_dsmem_f64(base + e * 8u);
            cj[r * KMAX + e] = (int)ld_dsmem_f64(base + (KMAX + e) * 8u);
          }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < CS; r++) {
          for (int e = lane; e < k; e += 32) {
            const double v = cv[r * KMAX + e];
            const int j = cj[r * KMAX + e];
            int rank = e;
#pragma unroll
            for (int o = 0; o < CS; o++) {
              if (o == r) continue;
              int lo = 0, hi = k;  // entries of list o before (v, j)
              while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                const double mv = cv[o * KMAX + mid];
                if (mv < v || (mv == v && cj[o * KMAX + mid] < j)) lo = mid + 1;
                else hi = mid;
              }
              rank += lo;
            }
            if (rank < k) H.near[rank] = j;
          }
        }
      }
      xph ^= 1;
      __syncthreads();
    }
    BM_PHASE(3);
    if (H.fail) {
      if (tid == 0) out.ok = 0;
      return;
    }
    __syncthreads();
    BM_PHASE(4);
    // Bm = C_XY L^-T : Bm[q][t] = sum_s C_XY[q][s] Linv[t][s]
    for (int o = tid; o < 128; o += NT) {
      const int q = o >> 5, t = o & 31;
      double s = 0.0;
      for (int k = 0; k < n; k++) s = fma(H.cxy[q * 32 + k], H.Linv[t * LS + k], s);
      H.Bm[q * 32 + t] = t < n ? s : 0.0;
    }
  }

  // ------------------------------ d_j = |L^-1 (y0 - y_j)|^2 (V in registers, DMMA)
  {
    double y0r[8];
    typename ZL::Ref ry[8];
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const int dim = 4 * kk + t4;
      y0r[kk] = dim < n ? y0[dim] : 0.0;
      ry[kk] = zv.ref(H, dim);
    }
    with_na(n, [&](auto NAc) {
    constexpr int NA = decltype(NAc)::value;
    double fb[8], fbn[8];
    // (L^-1 vanishes beyond n: the padding dims' B values only meet zeros)
    auto load_v = [&](int c, double(&o)[8]) {
      const int bB = zv.base(min(8 * c + g, m - 1));  // padding columns: d_j not stored
#pragma unroll
      for (int kk = 0; kk < 8; kk++) o[kk] = kk < 2 * NA ? y0r[kk] - zv.at(ry[kk], bB) : 0.0;
    };
    load_v(gw, fb);
    // The L^-1 A fragments do not change over the column tiles; the d_j
    // stores inside the loop keep the compiler from hoisting their loads, so
    // (N_y <= 24: 12 fragments) they are held in registers explicitly.
    constexpr bool HOIST = BM_QF_HOIST && NA <= 3;
    constexpr int NLA = HOIST ? NA * (NA + 1) : 1;
    double la[NLA];
    if constexpr (HOIST) {
      int q = 0;
#pragma unroll
      for (int r = 0; r < NA; r++)
#pragma unroll
        for (int kk = 0; kk < 2 * r + 2; kk++) la[q++] = H.Linv[(8 * r + g) * LS + 4 * kk + t4];
    }
#pragma unroll kQfUnroll
    for (int c = gw; c < nct; c += GWARPS) {
      load_v(c + GWARPS, fbn);
      double acc[8], acb[8];  // even / odd k-steps: two independent MMA chains
#pragma unroll
      for (int i = 0; i < 8; i++) acc[i] = acb[i] = 0.0;
      int q = 0;
#pragma unroll
      for (int r = 0; r < NA; r++)
#pragma unroll
        for (int kk = 0; kk < 2 * r + 2; kk++) {
          const double a = HOIST ? la[HOIST ? q : 0] : H.Linv[(8 * r + g) * LS + 4 * kk + t4];
          q++;
          if (kk & 1) dmma(acb[2 * r], acb[2 * r + 1], a, fb[kk]);
          else dmma(acc[2 * r], acc[2 * r + 1], a, fb[kk]);
        }
#pragma unroll
      for (int i = 0; i < 8; i++) acc[i] += acb[i];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) fb[kk] = fbn[kk];
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        s0 = fma(acc[2 * r], acc[2 * r], s0);
        s1 = fma(acc[2 * r + 1], acc[2 * r + 1], s1);
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(FULL, s0, o);
        s1 += __shfl_xor_sync(FULL, s1, o);
      }
      if (g == 0) {
        const int col = 8 * c + 2 * t4;
        if (col < m) dS[col] = s0;
        if (col + 1 < m) dS[col + 1] = s1;
        if constexpr (CS > 1) {  // every CTA of the cluster needs every d_j
#pragma unroll
          for (int r = 1; r < CS; r++) {
            const unsigned peer = (rank + r) % CS;
            if (col < m) st_dsmem_f64(map_rank(dS + col, peer), s0);
            if (col + 1 < m) st_dsmem_f64(map_rank(dS + col + 1, peer), s1);
          }
        }
      }
    }
    });
  }
  if constexpr (CS > 1) cluster_sync_all();
  else __syncthreads();
  BM_PHASE(5);
  double dmin;
  {
    double mn = INFINITY;
    for (int j = tid; j < m; j += NT) mn = fmin(mn, dS[j]);
    mn = warp_min(mn);
    if (lane == 0) H.redmin[0][warp] = mn;
    __syncthreads();
    BM_PHASE(6);
    dmin = H.redmin[0][0];
#pragma unroll
    for (int w = 1; w < NWARP; w++) dmin = fmin(dmin, H.redmin[0][w]);
  }

  // ------------------------------------------------ beta grid (DMMA)
  typename ZL::Ref crz[5];
#pragma unroll
  for (int ct = 0; ct < 5; ct++) crz[ct] = zv.ref(H, 8 * ct + g);
  {
    // MMA row 8r+g holds grid point beta_(3g+r): a lane's three betas are
    // consecutive, so one exp at beta_(3g+2) and two squarings give all three
    // (w(2^-1 beta) = w(beta)^2 exactly in real arithmetic; <= 4 ulp here)
    const double sc2 = ldexp(1.0, 7 - (3 * g + 2));  // 1/(2 beta_(3g+2))
    const bool brow = 3 * g + 2 < NBETA;
    double acc[30];
#pragma unroll
    for (int i = 0; i < 30; i++) acc[i] = 0.0;
    with_na(n, [&](auto NAc) {
    constexpr int NA = decltype(NAc)::value;
    // software pipeline: next k-step's d_j and B fragments load during this step
    double dl, dln, fb[5], fbn[5];
    auto load_b = [&](int s, double& d, double(&o)[5]) {
      const int j = 4 * s + t4;
      const bool valid = j < m;
      const int jc = min(j, m - 1);
      const int b = zv.base(jc);
      const double dd = dmin - dS[jc];
      d = valid ? dd : -INFINITY;  // -inf -> weight 0 for padding
#pragma unroll
      for (int ct = 0; ct < 5; ct++) o[ct] = (ct < NA || ct == 4) ? zv.at(crz[ct], b) : 0.0;  // weight 0 for padding
      if (g == ONES_COL - 32) o[4] = 1.0;
    };
    load_b(gw, dl, fb);
#pragma unroll kBetaUnroll
    for (int s = gw; s < nks; s += GWARPS) {
      load_b(s + GWARPS, dln, fbn);
      double fa[3];
#if BM_LOO_FAST
      const double e2w = brow ? exp_wf(dl * sc2, exptab) : 0.0;  // exp(expo - expo.max()); -inf -> 0
#else
      const double e2w = brow ? exp_wn(dl * sc2, exptab) : 0.0;  // exp(expo - expo.max()); -inf -> 0
#endif
      fa[2] = e2w;
      fa[1] = e2w * e2w;
      fa[0] = fa[1] * fa[1];
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int ct = 0; ct < 5; ct++)
          if (ct < NA || ct == 4) dmma(acc[2 * (r * 5 + ct)], acc[2 * (r * 5 + ct) + 1], fa[r], fb[ct]);
      dl = dln;
#pragma unroll
      for (int ct = 0; ct < 5; ct++) fb[ct] = fbn[ct];
    }
    });
    if (tid == 0) BM_DIAG_ADD(32, (clock64() - ph_t));  // beta loop (thread 0)
    tree_reduce<30, RED_CHUNK>(acc, H.R1);
    cluster_sum_w0<30>(acc, H, xph);
    if (tid == 0) BM_DIAG_ADD(33, (clock64() - ph_t));  // beta loop + reduce
    constexpr int PS = 41;  // row stride of P: conflict-free per-lane row reads
    double* P = H.R2;       // [24][PS]
    if (warp == 0) {
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          const int bi = 3 * g + r;  // grid index of MMA row 8r+g
          if (bi < 24) {
            P[bi * PS + 8 * ct + 2 * t4] = acc[2 * (r * 5 + ct)];
            P[bi * PS + 8 * ct + 2 * t4 + 1] = acc[2 * (r * 5 + ct) + 1];
          }
        }
    }
#if BM_BETA_PAR
    // the 21 x n squared residuals (y0 - y~0(beta_g))[t]^2, one division each,
    // on all threads (two barriers) instead of n divisions per lane on warp 0
    __syncthreads();
    for (int o = tid; o < NBETA * 32; o += NT) {
      const int gi = o >> 5, t = o & 31;
      if (t < n) {
        const double d = y0[t] - P[gi * PS + t] / P[gi * PS + ONES_COL];
        H.R1[gi * 33 + t] = __dmul_rn(d, d);
      }
    }
    __syncthreads();
#endif
    if (warp == 0) {
      __syncwarp();
      // eps_g = ||y0 - y~0(beta_g)||^2 in NumPy's pairwise order; strict < argmin
      double eps = INFINITY;
      if (lane < NBETA) {
        const double S = P[lane * PS + ONES_COL];
#if BM_BETA_PAR
        (void)S;
        const double* sq = H.R1 + lane * 33;
        eps = pairwise_sum_n(n, [&](int t) { return sq[t]; });
#elif BM_CBETA
        // squares staged per lane (R1 is free after the reduction): one copy
        // of the division code instead of one per unrolled pairwise term
        double* sq = H.R1 + lane * 33;
#pragma unroll 1
        for (int t = 0; t < n; t++) {
          const double d = y0[t] - P[lane * PS + t] / S;
          sq[t] = __dmul_rn(d, d);
        }
        eps = pairwise_sum_n(n, [&](int t) { return sq[t]; });
#else
        eps = pairwise_sum_n(n, [&](int t) {
          const double d = y0[t] - P[lane * PS + t] / S;
          return __dmul_rn(d, d);
        });
#endif
      }
      // first minimum (ties -> smaller beta; NaN never wins), butterfly over (key, index)
      double bv = eps != eps ? INFINITY : eps;
      int bi = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const int oi = __shfl_xor_sync(FULL, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      const int best = bv == INFINITY ? 0 : bi;
      const double best_eps = __shfl_sync(FULL, eps, best) != __shfl_sync(FULL, eps, best) ? INFINITY
                                                                                          : __shfl_sync(FULL, eps, best);
      double ya = lane < n ? fabs(y0[lane]) : 0.0;
      ya = warp_max(ya);
      const double dy = 1e-11 * ya;
      const double noise = 2.0 * sqrt(best_eps * n) * dy + n * dy * dy + 1e-300;
      double gap = (lane < NBETA && lane != best) ? fabs(eps - best_eps) / noise : INFINITY;
      gap = warp_min(gap);
      const double S = P[best * PS + ONES_COL];
      H.yt[lane] = lane < n ? P[best * PS + lane] / S : 0.0;
      if (lane < 4) H.xt[lane] = P[best * PS + 32 + lane] / S;
      if (lane == 0) {
        H.gbest = best;
        out.beta = ldexp(1.0, best - 8);
        out.gap = (float)gap;
      }
    }
    __syncthreads();
    BM_PHASE(7);
  }
  const double sb = ldexp(1.0, 7 - H.gbest);
  const int k = min(n + 1, m);

  // Rows of the Gram GEMM: U_i = C^-1 (y0 - y_near_i) = L^-T L^-1 (y0 - y_near_i),
  // so that v_i . v_j = U_i . (y0 - y_j) reads candidate j straight from the
  // shared support tile (V never goes through global memory).
  double* Un = H.R2;        // [40][LS]  A fragments of the Gram GEMM
#if BM_TSTAGE
  // Staging with the nearest rows on the lanes: Wt and Vt are kept transposed
  // ([32][WS], WS odd), a warp takes one dimension t (warp-uniform trip count
  // t + 1 or n - t instead of the longest lane's n), L^-1 entries are
  // broadcasts and the Wt / Vt reads are conflict-free (the [i][32] layout
  // with t on the lanes read L^-1 rows 8-way bank-conflicted).  Every output
  // keeps its fma order, so the same bits.
  constexpr int WS = 33;
  double* Vt = H.R1;            // [32][WS] (L^-1 (y0 - y_near_i))[t] at [t][i] (R1 head is free here)
  double* Wt = H.R1 + 32 * WS;  // [32][WS] (y0 - y_near_i)[q] at [q][i] (below Zp)
  static_assert(2 * 32 * WS <= ZP_OFF + KMAX * 40 && KMAX <= WS, "staging fits R1");
  for (int o = tid; o < k * 32; o += NT) {
    const int i = o >> 5, q = o & 31;
    Wt[q * WS + i] = q < n ? y0[q] - zv.at(zv.ref(H, q), zv.base(H.near[i])) : 0.0;
  }
  if (tid < 40) H.dn[tid] = tid < k ? dS[H.near[tid]] : 0.0;
  for (int o = tid; o < 40 * 32; o += NT) {  // Un vanishes beyond the k rows and n dimensions
    const int i = o >> 5, t = o & 31;
    if (i >= k || t >= n) Un[i * LS + t] = 0.0;
  }
  __syncthreads();
  const int nh = (k + 31) >> 5;  // lane groups of 32 nearest rows (2 only for k = 33)
  for (int row = warp; row < n * nh; row += NWARP) {
    const int t = row / nh, i = (row % nh) * 32 + lane;
    if (i < k) {
      double sv = 0.0;
      for (int q = 0; q <= t; q++) sv = fma(H.Linv[t * LS + q], Wt[q * WS + i], sv);
      Vt[t * WS + i] = sv;
    }
  }
  __syncthreads();
  for (int row = warp; row < n * nh; row += NWARP) {
    const int t = row / nh, i = (row % nh) * 32 + lane;
    if (i < k) {
      double su = 0.0;
      for (int q = t; q < n; q++) su = fma(H.Linv[q * LS + t], Vt[q * WS + i], su);
      Un[i * LS + t] = su;
    }
  }
  __syncthreads();
#else
  double* Vt = H.R1;             // [KMAX][32] L^-1 (y0 - y_near_i) (R1 head is free here)
  double* Wt = H.R1 + KMAX * 32;  // [KMAX][32] y0 - y_near_i (below Zp)
  static_assert(2 * KMAX * 32 <= ZP_OFF + KMAX * 40, "staging fits R1");
  for (int o = tid; o < k * 32; o += NT) {
    const int i = o >> 5, q = o & 31;
    Wt[o] = q < n ? y0[q] - zv.at(zv.ref(H, q), zv.base(H.near[i])) : 0.0;
  }
  if (tid < 40) H.dn[tid] = tid < k ? dS[H.near[tid]] : 0.0;
  __syncthreads();
  for (int o = tid; o < KMAX * 32; o += NT) {
    const int i = o >> 5, t = o & 31;
    double sv = 0.0;
    if (i < k && t < n)
      for (int q = 0; q <= t; q++) sv = fma(H.Linv[t * LS + q], Wt[i * 32 + q], sv);
    Vt[i * 32 + t] = sv;
  }
  __syncthreads();
  for (int o = tid; o < 40 * 32; o += NT) {
    const int i = o >> 5, t = o & 31;
    double su = 0.0;
    if (i < k && t < n)
      for (int q = t; q < n; q++) su = fma(H.Linv[q * LS + t], Vt[i * 32 + q], su);
    Un[i * LS + t] = su;
  }
  __syncthreads();
#endif
  BM_PHASE(9);

  // ---- fused Gram + leave-one-out sums (estimators.py:225-238), DMMA.
  // q_ij = d_i + d_j - 2 v_i.v_j (= (y_i-y_j)^T C^-1 (y_i-y_j)); the LOO
  // weights exp(x_ij - max_j x_ij), x = -q/(2 beta), are accumulated with a
  // lazily raised per-row reference max (rescale only when a new x exceeds it
  // by > 20, so w <= e^20): identical to the reference's shift after the final
  // normalisation, and q never round-trips through memory.  LOO_RR 8-row
  // tiles per pass bound registers; the Gram B fragments (y0 - y_j) are
  // re-read from the shared support tile each pass.
  double* Zp = H.R1 + ZP_OFF;  // [KMAX][40], after the <=20-tile tree-reduction partials
  // 8-row tiles of the nearest set on DMMA; with k = 8t + 1 (N_y = 16 / 24 /
  // 32), the last row runs as a SIMT pass below instead of a 1-of-8-rows tile
  const bool row1 = BM_LOO_ROW1 && CS == 1 && (k & 7) == 1 && k > 8;
  const int ntile = (k + 7 - (row1 ? 1 : 0)) >> 3;
  constexpr int RR = LOO_RR;       // row tiles per pass over the candidates
  double y0r[8];
  typename ZL::Ref ry[8];
#pragma unroll
  for (int kk = 0; kk < 8; kk++) {
    const int dim = 4 * kk + t4;
    y0r[kk] = dim < n ? y0[dim] : 0.0;
    ry[kk] = zv.ref(H, dim);
  }
  for (int r0 = 0; r0 < ntile; r0 += RR) {
    const long long t_pass = clock64();
    const int nrow = min(RR, ntile - r0);
    double xref[RR];
#pragma unroll
    for (int rr = 0; rr < RR; rr++) xref[rr] = -INFINITY;
    double acc[10 * RR];
#pragma unroll
    for (int i = 0; i < 10 * RR; i++) acc[i] = 0.0;
    with_na(n, [&](auto NAc) {
    constexpr int NA = decltype(NAc)::value;
#if BM_LOO_HOIST
    // (RR == 1) the pass's row tile: its U A fragments, nearest index and d_i
    // do not change over the column tiles; held in registers explicitly
    static_assert(LOO_RR == 1, "hoisted A fragments assume one row tile per pass");
    double ua[2 * NA];
#pragma unroll
    for (int kk = 0; kk < 2 * NA; kk++) ua[kk] = Un[(8 * r0 + g) * LS + 4 * kk + t4];
    const int hi_ = 8 * r0 + g;
    const int nri_h = hi_ < k ? H.near[hi_] : -2;
    const double dni_h = hi_ < k ? H.dn[hi_] : 0.0;
#endif
#pragma unroll kLooUnroll
    for (int c = gw; c < nct; c += GWARPS) {
      // Gram B fragment of column tile c: (y0 - y_j)[4kk + t4] for j = 8c + g
      // (U vanishes beyond n: the padding dims' values only meet zeros)
      double fv[8];
      {
        const int bB = zv.base(min(8 * c + g, m - 1));  // padding columns: clamped (their x is -inf)
#pragma unroll
        for (int kk = 0; kk < 2 * NA; kk++) fv[kk] = y0r[kk] - zv.at(ry[kk], bB);
      }
      const int col = 8 * c + 2 * t4;
      const double dv0 = dS[min(col, m - 1)], dv1 = dS[min(col + 1, m - 1)];
      // k-step 0 takes the tile's even candidates 8c + 2t4, k-step 1 the odd
      // ones: the Gram C fragment (row g, cols 2t4, 2t4+1) is then already the
      // A fragment of both k-steps, no shuffles
      const int b0 = zv.base(min(col, m - 1)), b1 = zv.base(min(col + 1, m - 1));
      const bool ones = g == ONES_COL - 32;
#pragma unroll
      for (int rr = 0; rr < RR; rr++) {
        if (rr >= nrow) break;
        const int r = r0 + rr;
        const int i = 8 * r + g;
#if BM_LOO_HOIST
        const int nri = nri_h;
        const double dni = dni_h;
        (void)i;
#else
        const int nri = i < k ? H.near[i] : -2;
        const double dni = i < k ? H.dn[i] : 0.0;
#endif
        double g0 = 0.0, g1 = 0.0, h0 = 0.0, h1 = 0.0;  // two independent MMA chains
#pragma unroll
        for (int kk = 0; kk < 2 * NA; kk += 2) {
#if BM_LOO_HOIST
          dmma(g0, g1, ua[kk], fv[kk]);
          dmma(h0, h1, ua[kk + 1], fv[kk + 1]);
#else
          dmma(g0, g1, Un[(8 * r + g) * LS + 4 * kk + t4], fv[kk]);
          dmma(h0, h1, Un[(8 * r + g) * LS + 4 * kk + 4 + t4], fv[kk + 1]);
#endif
        }
        g0 += h0;
        g1 += h1;
#if BM_LOO_FAST
        // -q_ij = 2 G_ij - (d_i + d_j); x = -q sb (sb a power of two) and
        // x - xref in one fma; the row-max vote compares bit patterns on the
        // integer pipe (a > 20 <=> bits(a) > bits(20) for non-NaN a)
        const bool v0 = nri >= 0 && col < m && col != nri, v1 = nri >= 0 && col + 1 < m && col + 1 != nri;
        const double u0 = fma(2.0, g0, -(dni + dv0)), u1 = fma(2.0, g1, -(dni + dv1));
        double a0 = fma(u0, sb, -xref[rr]), a1 = fma(u1, sb, -xref[rr]);
        constexpr long long B20 = 0x4034000000000000ll;  // bits of 20.0
        if (__any_sync(FULL, (v0 && __double_as_longlong(a0) > B20) || (v1 && __double_as_longlong(a1) > B20))) {
          // (rare) raise the row references, rescale the rows' partial sums
          double tmax = fmax(v0 ? u0 * sb : -INFINITY, v1 ? u1 * sb : -INFINITY);
          tmax = fmax(tmax, __shfl_xor_sync(FULL, tmax, 1));
          tmax = fmax(tmax, __shfl_xor_sync(FULL, tmax, 2));
          if (tmax > xref[rr] + 20.0) {
            const double f = xref[rr] == -INFINITY ? 0.0 : exp(xref[rr] - tmax);
#pragma unroll
            for (int q = 0; q < 10; q++) acc[rr * 10 + q] *= f;
            xref[rr] = tmax;
            a0 = fma(u0, sb, -tmax);
            a1 = fma(u1, sb, -tmax);
          }
        }
        const double e0 = exp_wf(a0, exptab), e1 = exp_wf(a1, exptab);
        const double w0 = v0 ? e0 : 0.0, w1 = v1 ? e1 : 0.0;  // (invalid: a may be +inf, e garbage)
#else
        double x0 = -INFINITY, x1 = -INFINITY;
        if (nri >= 0) {
          if (col < m && col != nri) x0 = -(dni + dv0 - 2.0 * g0) * sb;
          if (col + 1 < m && col + 1 != nri) x1 = -(dni + dv1 - 2.0 * g1) * sb;
        }
        if (__any_sync(FULL, fmax(x0, x1) > xref[rr] + 20.0)) {
          // (rare) raise the row references, rescale the rows' partial sums
          double tmax = fmax(x0, x1);
          tmax = fmax(tmax, __shfl_xor_sync(FULL, tmax, 1));
          tmax = fmax(tmax, __shfl_xor_sync(FULL, tmax, 2));
          if (tmax > xref[rr] + 20.0) {
            const double f = xref[rr] == -INFINITY ? 0.0 : exp(xref[rr] - tmax);
#pragma unroll
            for (int q = 0; q < 10; q++) acc[rr * 10 + q] *= f;
            xref[rr] = tmax;
          }
        }
        const double e0 = exp_wn(x0 - xref[rr], exptab), e1 = exp_wn(x1 - xref[rr], exptab);
        const double w0 = x0 == -INFINITY ? 0.0 : e0, w1 = x1 == -INFINITY ? 0.0 : e1;  // (xref may be -inf)
#endif
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          if (ct >= NA && ct < 4) continue;  // y columns beyond n: outputs unused
          const double z0 = ct == 4 && ones ? 1.0 : zv.at(crz[ct], b0);  // padding: weight 0
          const double z1 = ct == 4 && ones ? 1.0 : zv.at(crz[ct], b1);
          dmma(acc[rr * 10 + 2 * ct], acc[rr * 10 + 2 * ct + 1], w0, z0);
          dmma(acc[rr * 10 + 2 * ct], acc[rr * 10 + 2 * ct + 1], w1, z1);
        }
      }
    }
    });
    if (tid == 0) BM_DIAG_ADD(34, (clock64() - t_pass));  // LOO loops (thread 0)
    // combine the warps' partial sums at a common per-row reference
#pragma unroll
    for (int rr = 0; rr < RR; rr++)
      if (t4 == 0) H.wmin[warp][rr * 8 + g] = xref[rr];
    __syncthreads();
    double rowmx[RR];
#pragma unroll
    for (int rr = 0; rr < RR; rr++) {
      double mx = -INFINITY;
#pragma unroll
      for (int w = 0; w < NWARP; w++) mx = fmax(mx, H.wmin[w][rr * 8 + g]);
      rowmx[rr] = mx;
      const double f = (xref[rr] == -INFINITY) ? 0.0 : exp(xref[rr] - mx);
#pragma unroll
      for (int i = 0; i < 10; i++) acc[rr * 10 + i] *= f;
    }
#pragma unroll
    for (int rr = 0; rr < RR; rr++) {
      if (rr >= nrow) break;
      double a10[10];
#pragma unroll
      for (int i = 0; i < 10; i++) a10[i] = acc[rr * 10 + i];
      tree_reduce<10>(a10, H.R1);
      if constexpr (CS > 1) {
        // the CTAs' row sums are relative to their own row maxima: rescale to
        // the cluster maximum and add in rank order (identical in every CTA)
        double* b = H.xb + xph * XB_HALF;
        if (warp == 0) {
#pragma unroll
          for (int i = 0; i < 10; i++) b[i * 32 + lane] = a10[i];
          b[10 * 32 + lane] = rowmx[rr];
        }
        cluster_sync_all();
        if (warp == 0) {
          uint32_t base[CS];
          double mr[CS], M = -INFINITY;
#pragma unroll
          for (int r = 0; r < CS; r++) {
            base[r] = map_rank(b, r) + lane * 8u;
            mr[r] = ld_dsmem_f64(base[r] + 10 * 256u);
            M = fmax(M, mr[r]);
          }
          double f[CS];
#pragma unroll
          for (int r = 0; r < CS; r++) f[r] = mr[r] == -INFINITY ? 0.0 : exp(mr[r] - M);
#pragma unroll
          for (int i = 0; i < 10; i++) {
            double t = ld_dsmem_f64(base[0] + i * 256u) * f[0];
#pragma unroll
            for (int r = 1; r < CS; r++) t += ld_dsmem_f64(base[r] + i * 256u) * f[r];
            a10[i] = t;
          }
        }
        xph ^= 1;
      }
      const int row = 8 * (r0 + rr) + g;
      if (warp == 0 && row < KMAX) {
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          Zp[row * 40 + 8 * ct + 2 * t4] = a10[2 * ct];
          Zp[row * 40 + 8 * ct + 2 * t4 + 1] = a10[2 * ct + 1];
        }
      }
    }
  }
#if BM_LOO_ROW1
  if (row1) {
    // Row i = k - 1 of the LOO sums: lanes are candidates for the Gram entry
    // G_ij = U_i . (y0 - y_j) and the weight, then lanes are columns (y, x,
    // ones) for Zp_i = sum_j w_ij [Y|X|1]_j; a lazily raised per-warp
    // reference as in the DMMA passes, warps combined at the common maximum
    // in a fixed order.
    const int i = k - 1;
    const int nri = H.near[i];
    const double dni = H.dn[i];
    const int ncol = n + 5;
    auto colof = [&](int c) { return c < n ? c : (c < n + 4 ? 32 + c - n : ONES_COL); };
    const int cA = colof(lane), cB = colof(min(lane + 32, ncol - 1));
    const typename ZL::Ref rA = zv.ref(H, cA < 36 ? cA : 0), rB = zv.ref(H, cB < 36 ? cB : 0);
    const bool hasA = lane < ncol, hasB = lane + 32 < ncol;
    const double* Ui = Un + i * LS;
    double sA0 = 0.0, sA1 = 0.0, sB = 0.0, xr = -INFINITY;
    for (int j0 = warp * 32; j0 < m; j0 += NT) {
      const int j = j0 + lane;
      const bool v = j < m && j != nri;
      const int jc = min(j, m - 1);
      const int b = zv.base(jc);
      double ga = 0.0, gb = 0.0;
#pragma unroll 4
      for (int t = 0; t < n; t += 2) {
        ga = fma(Ui[t], y0[t] - zv.at(zv.ref(H, t), b), ga);
        if (t + 1 < n) gb = fma(Ui[t + 1], y0[t + 1] - zv.at(zv.ref(H, t + 1), b), gb);
      }
      const double x = -(dni + dS[jc] - 2.0 * (ga + gb)) * sb;
      const double wx = warp_max(v ? x : -INFINITY);
      if (wx > xr + 20.0) {  // (rare) raise the warp's reference, rescale its sums
        const double f = xr == -INFINITY ? 0.0 : exp(xr - wx);
        sA0 *= f;
        sA1 *= f;
        sB *= f;
        xr = wx;
      }
      const double w = v ? exp_wn(x - xr, exptab) : 0.0;
      const int cnt = min(32, m - j0);
#pragma unroll 2
      for (int jj = 0; jj < cnt; jj++) {
        const double wj = __shfl_sync(FULL, w, jj);
        const int bj = __shfl_sync(FULL, b, jj);
        const double za = cA == ONES_COL ? 1.0 : zv.at(rA, bj);
        if (jj & 1) sA1 = fma(wj, za, sA1);
        else sA0 = fma(wj, za, sA0);
        if (hasB) sB = fma(wj, cB == ONES_COL ? 1.0 : zv.at(rB, bj), sB);
      }
    }
    double* ws = H.R1;  // [NWARP][40] (free: the tree-reduction partials of the passes above)
    if (hasA) ws[warp * 40 + cA] = sA0 + sA1;
    if (hasB) ws[warp * 40 + cB] = sB;
    if (lane == 0) H.redmin[0][warp] = xr;
    __syncthreads();
    if (warp == 0) {
      double M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NWARP; w++) M = fmax(M, H.redmin[0][w]);
      double fw[NWARP];
#pragma unroll
      for (int w = 0; w < NWARP; w++) fw[w] = H.redmin[0][w] == -INFINITY ? 0.0 : exp(H.redmin[0][w] - M);
      double tA = 0.0, tB = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; w++) {
        if (hasA) tA = fma(ws[w * 40 + cA], fw[w], tA);
        if (hasB) tB = fma(ws[w * 40 + cB], fw[w], tB);
      }
      if (hasA) Zp[i * 40 + cA] = tA;
      if (hasB) Zp[i * 40 + cB] = tB;
    }
  }
#endif
  __syncthreads();
  BM_PHASE(11);

  // ---------------------------------- alpha (estimators.py:237-245)
  {
#if BM_TSTAGE
    // (the nearest rows on the lanes, R and u transposed: see the staging above)
    constexpr int WS = 33;
    double* u = H.R1;  // [32][WS]  u_i[t] at [t][i]
    double* R = H.R2;  // [36][WS]  (y_i - y~_i | x_i - x~_i)[q] at [q][i]  (Un is dead here)
    static_assert(36 * WS <= 1600, "R fits R2");
    for (int o = tid; o < k * 36; o += NT) {
      const int i = o / 36, q = o % 36;
      double r = 0.0;
      if (q < n || q >= 32)
        r = zv.at(zv.ref(H, q), zv.base(H.near[i])) - Zp[i * 40 + q] / Zp[i * 40 + ONES_COL];
      R[q * WS + i] = r;
    }
    __syncthreads();
    const int nh = (k + 31) >> 5;
    for (int row = warp; row < n * nh; row += NWARP) {
      const int t = row / nh, i = (row % nh) * 32 + lane;
      if (i < k) {
        double s = 0.0;
        for (int q = 0; q <= t; q++) s = fma(H.Linv[t * LS + q], R[q * WS + i], s);
        u[t * WS + i] = s;
      }
    }
    __syncthreads();
    for (int o = tid; o < 4 * k; o += NT) {
      const int q = o / k, i = o % k;
      double c = 0.0;
      for (int t = 0; t < n; t++) c = fma(H.Bm[q * 32 + t], u[t * WS + i], c);
      H.cmat[q * k + i] = c;
      H.rmat[q * k + i] = R[(32 + q) * WS + i];
    }
    __syncthreads();
#else
    double* u = H.R1;  // [KMAX][32]
    double* R = H.R2;  // [KMAX][36]: y_i - y~_i | x_i - x~_i  (Un is dead here)
    for (int o = tid; o < k * 36; o += NT) {
      const int i = o / 36, q = o % 36;
      double r = 0.0;
      if (q < n || q >= 32)
        r = zv.at(zv.ref(H, q), zv.base(H.near[i])) - Zp[i * 40 + q] / Zp[i * 40 + ONES_COL];
      R[o] = r;
    }
    __syncthreads();
    for (int o = tid; o < k * 32; o += NT) {
      const int i = o >> 5, t = o & 31;
      double s = 0.0;
      if (t < n)
        for (int q = 0; q <= t; q++) s = fma(H.Linv[t * LS + q], R[i * 36 + q], s);
      u[o] = s;
    }
    __syncthreads();
    for (int o = tid; o < 4 * k; o += NT) {
      const int q = o / k, i = o % k;
      double c = 0.0;
      for (int t = 0; t < n; t++) c = fma(H.Bm[q * 32 + t], u[i * 32 + t], c);
      H.cmat[q * k + i] = c;
      H.rmat[q * k + i] = R[i * 36 + 32 + q];
    }
    __syncthreads();
#endif
    if (warp == 0) {
      // u0 = Linv (y0 - y~0); correction = Bm u0
      double s = 0.0;
      for (int q = 0; q <= lane && q < n; q++) s = fma(H.Linv[lane * LS + q], y0[q] - H.yt[q], s);
      const double u0 = lane < n ? s : 0.0;
      double corr[4];
#pragma unroll
      for (int q = 0; q < 4; q++) corr[q] = warp_sum(H.Bm[q * 32 + lane] * u0);
#if BM_ALPHA_PAR
      // den = (c * c).sum() on lanes 0-15, num = ((x - x_pred).T * c).sum() on
      // lanes 16-31, in NumPy's pairwise order over the 4k elements (4k >= 8, a
      // multiple of 4): lane j of an 8-lane group owns the strided accumulator
      // r[j], the ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree is three xor
      // shuffles, then the tail elements in order; beyond 128 elements the
      // two halves of NumPy's split run on the two 8-lane groups.  The same
      // bits as one lane's sequential pairwise_sum_long.
      const int kk = 4 * k;
      const int sub = (lane >> 3) & 1, j8 = lane & 7;
      const double* f = (lane >> 4) ? H.rmat : H.cmat;
      const bool two = kk > 128;
      int n2 = kk / 2;
      n2 -= n2 % 8;
      const int lo = (two && sub) ? n2 : 0;
      const int nb = two ? (sub ? kk - n2 : n2) : kk;
      const int nfull = nb - (nb % 8);
      double sv = __dmul_rn(f[lo + j8], H.cmat[lo + j8]);
      for (int i = 8; i < nfull; i += 8) sv = __dadd_rn(sv, __dmul_rn(f[lo + i + j8], H.cmat[lo + i + j8]));
      sv = __dadd_rn(sv, __shfl_xor_sync(FULL, sv, 1));
      sv = __dadd_rn(sv, __shfl_xor_sync(FULL, sv, 2));
      sv = __dadd_rn(sv, __shfl_xor_sync(FULL, sv, 4));
      for (int i = nfull; i < nb; i++) sv = __dadd_rn(sv, __dmul_rn(f[lo + i], H.cmat[lo + i]));
      const double sv8 = __shfl_xor_sync(FULL, sv, 8);
      if (two) sv = __dadd_rn(sv, sv8);
      const double den = __shfl_sync(FULL, sv, 0), num = __shfl_sync(FULL, sv, 16);
#else
      // den = (c * c).sum() on lane 0, num = ((x - x_pred).T * c).sum() on
      // lane 1 (NumPy's pairwise order over the 4k elements), concurrently
      const int kk = 4 * k;
      double sv = 0.0;
      if (lane < 2) {
        const double* f = lane ? H.rmat : H.cmat;
        sv = pairwise_sum_long(kk, [&](int i) { return __dmul_rn(f[i], H.cmat[i]); });
      }
      const double den = __shfl_sync(FULL, sv, 0), num = __shfl_sync(FULL, sv, 1);
#endif
      if (lane == 0) {
        double a = 0.0;
        if (!(den < 1e-12)) {
          a = num / den;
          a = a < 0.0 ? 0.0 : (a > 4.0 ? 4.0 : a);  // np.clip keeps NaN
        }
        out.alpha = a;
        bool finite = true;
        for (int q = 0; q < 4; q++) {
          out.vals[q] = H.xt[q] + a * corr[q];
          if (!isfinite(out.vals[q])) finite = false;
        }
        out.ok = finite;  // FloatingPointError -> ladder
      }
    }
  }
  __syncthreads();
  BM_PHASE(12);
}

}  // namespace BM_NS
