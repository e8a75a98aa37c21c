// bm_api.cu — device entry points of the reference's per-patch library API
// (blockmend/__init__.py:17-45): the framework functions (extract_target,
// build_expansion_map, _collect under gather_candidates / expand_support,
// patch_scores, build_schedule) and the estimator stages (sample_covariance,
// kernel_weights, optimize_beta, optimize_alpha, idl_weights, predict_xy,
// CovarianceBlocks.solve_yy).
//
// These are not the concealment hot path (bm_conceal fuses all of it per
// cell); they serve library users and the reference's own unit tests, so
// they favour the reference's exact semantics over throughput: FP64 SIMT,
// one warp or CTA per request, NumPy's summation orders where NumPy defines
// one (pairwise sums of contiguous rows, sequential axis-0 means), a LAPACK
// style Cholesky for C_YY (estimators.py:61-68).  select_and_estimate lives
// with the fused kernel (bm_kernels.cuh, k_select) because it runs the same
// patch-step code.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/blockmend_b200.h"
#define BM_NS bmx  // this translation unit's copy of the shared helpers (own device symbols)
#include "bm_common.cuh"
#include "bm_host.h"

namespace bm_api {

using bmx::BS;
using bmx::ctx_c;
using bmx::ctx_r;
using bmx::FULL;
using bmx::ST_AV;
using bmx::ST_LO;

constexpr int NT = 256, NW = NT / 32;
constexpr int MAXM = 2048;  // candidates per estimator instance (>= 43*43)

// ------------------------------------------------------------ framework

// extract_target (framework.py:151-168): one warp per patch.
__global__ void k_extract(int H, int W, const double* __restrict__ px, const uint8_t* __restrict__ st, int count,
                          const int32_t* __restrict__ origins, uint32_t* layouts, int32_t* n_y, double* y0) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= count) return;
  const int r = origins[2 * i] - 2 + ctx_r(lane), c = origins[2 * i + 1] - 2 + ctx_c(lane);
  const bool inb = r >= 0 && r < H && c >= 0 && c < W;
  const size_t o = inb ? (size_t)r * W + c : 0;
  const bool usable = inb && st[o] != ST_LO;
  const unsigned bal = __ballot_sync(FULL, usable);
  if (usable) y0[(size_t)i * 32 + __popc(bal & ((1u << lane) - 1))] = px[o];
  if (lane == 0) {
    layouts[i] = bal;
    n_y[i] = __popc(bal);
  }
}

// _collect (framework.py:171-183): admissibility of each window origin (no
// LOST pixel at the target's used offsets: usable context, then the patch)
// and the (x, y) values of the admissible ones, compacted in list order.
// One CTA per request; request q owns origins [ooff[q], ooff[q] + ocnt[q])
// and writes its candidates at the same offsets of x [.][4] / y [.][32].
__global__ void k_collect(int H, int W, const double* __restrict__ px, const uint8_t* __restrict__ st,
                          const int32_t* __restrict__ origins, const int32_t* __restrict__ ooff,
                          const int32_t* __restrict__ ocnt, const uint32_t* __restrict__ layouts, double* xo,
                          double* yo, int32_t* mo) {
  __shared__ int wcnt[NW];
  __shared__ int16_t offr[36], offc[36];
  __shared__ int nused;
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lay = layouts[q];
  if (tid < 32) {  // used offsets (TargetContext.used_offsets): usable context then the patch cells
    const bool u = (lay >> lane) & 1u;
    const int idx = __popc(lay & ((1u << lane) - 1));
    if (u) {
      offr[idx] = (int16_t)ctx_r(lane);
      offc[idx] = (int16_t)ctx_c(lane);
    }
    const int n = __popc(lay);
    if (lane < 4) {
      offr[n + lane] = (int16_t)(2 + (lane >> 1));
      offc[n + lane] = (int16_t)(2 + (lane & 1));
    }
    if (lane == 0) nused = n;
  }
  __syncthreads();
  const int n = nused, base = ooff[q], cnt = ocnt[q];
  int m = 0;
  for (int e0 = 0; e0 < cnt; e0 += NT) {
    const int e = e0 + tid;
    bool ok = false;
    int wr = 0, wc = 0;
    if (e < cnt) {
      wr = origins[2 * (base + e)];
      wc = origins[2 * (base + e) + 1];
      ok = true;
      for (int k = 0; k < n + 4; k++) {
        const int r = wr + offr[k], c = wc + offc[k];
        if (r < 0 || r >= H || c < 0 || c >= W || st[(size_t)r * W + c] == ST_LO) {
          ok = false;
          break;
        }
      }
    }
    const unsigned bal = __ballot_sync(FULL, ok);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < NW; w++) {
      pre += w < warp ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    if (ok) {
      const size_t j = (size_t)base + m + pre + __popc(bal & ((1u << lane) - 1));
      for (int k = 0; k < n; k++) yo[j * 32 + k] = px[(size_t)(wr + offr[k]) * W + wc + offc[k]];
      for (int k = 0; k < 4; k++) xo[j * 4 + k] = px[(size_t)(wr + offr[n + k]) * W + wc + offc[n + k]];
    }
    m += tot;
    __syncthreads();
  }
  if (tid == 0) mo[q] = m;
}

// patch_scores (framework.py:230-240): (AVAILABLE, usable) context counts of
// arbitrary patch origins.  One thread per origin.
__global__ void k_patch_scores(int H, int W, const uint8_t* __restrict__ st, int count,
                               const int32_t* __restrict__ origins, int32_t* avail, int32_t* usable) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int pr = origins[2 * i], pc = origins[2 * i + 1];
  int a = 0, u = 0;
  for (int k = 0; k < 32; k++) {
    const int r = pr - 2 + ctx_r(k), c = pc - 2 + ctx_c(k);
    if (r < 0 || r >= H || c < 0 || c >= W) continue;
    const uint8_t s = st[(size_t)r * W + c];
    a += s == ST_AV;
    u += s != ST_LO;
  }
  avail[i] = a;
  usable[i] = u;
}

// build_schedule (framework.py:253-274): the simulated filling order of one
// block's lost patches, one warp per block.  Lane l owns patches l and l+32
// (raster order inside the block); the key (AVAILABLE, usable, raster) is
// maximised; a pick turns the patch's LOST pixels RECONSTRUCTED, which raises
// the usable count of exactly its 8 neighbouring patches (each neighbour's
// 6x6 window covers the whole patch) and changes nothing else.
__global__ void k_schedule(int H, int W, const uint8_t* __restrict__ st, int count,
                           const int32_t* __restrict__ blocks, int32_t* out_n, int32_t* out_origins,
                           int32_t* out_rel) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= count) return;
  const int br = blocks[2 * i] * BS, bc = blocks[2 * i + 1] * BS;
  int key[2], nlost[2];
  bool pend[2];
  for (int h = 0; h < 2; h++) {
    const int p = lane + 32 * h, pr = br + 2 * (p >> 3), pc = bc + 2 * (p & 7);
    int lost = 0;  // LOST pixels of the patch (inside the image)
    for (int q = 0; q < 4; q++) {
      const int r = pr + (q >> 1), c = pc + (q & 1);
      if (r < H && c < W) lost += st[(size_t)r * W + c] == ST_LO;
    }
    int a = 0, u = 0;
    for (int k = 0; k < 32; k++) {
      const int r = pr - 2 + ctx_r(k), c = pc - 2 + ctx_c(k);
      if (r < 0 || r >= H || c < 0 || c >= W) continue;
      const uint8_t s = st[(size_t)r * W + c];
      a += s == ST_AV;
      u += s != ST_LO;
    }
    nlost[h] = lost;
    pend[h] = lost > 0;
    key[h] = (a << 13) | (u << 7) | (63 - p);
  }
  int n = 0;
  for (;;) {
    const int mine = max(pend[0] ? key[0] : -1, pend[1] ? key[1] : -1);
    const int best = (int)__reduce_max_sync(FULL, (unsigned)(mine + 1)) - 1;
    if (best < 0) break;
    const int p = 63 - (best & 127);
    const int wb = __shfl_sync(FULL, nlost[p >> 5], p & 31);
    if (lane == 0) {
      out_origins[((size_t)i * 64 + n) * 2] = br + 2 * (p >> 3);
      out_origins[((size_t)i * 64 + n) * 2 + 1] = bc + 2 * (p & 7);
      out_rel[(size_t)i * 64 + n] = best >> 13;  // reliability = AVAILABLE context count
    }
    n++;
    for (int h = 0; h < 2; h++) {
      const int q = lane + 32 * h;
      if (q == p) pend[h] = false;
      const int dr = (q >> 3) - (p >> 3), dc = (q & 7) - (p & 7);
      if (q != p && dr >= -1 && dr <= 1 && dc >= -1 && dc <= 1) key[h] += wb << 7;
    }
  }
  if (lane == 0) out_n[i] = n;
}

// build_expansion_map (framework.py:130-148): window origins of the clipped
// support in (ring, row, col) order, from the closed-form ring enumeration
// the fused kernel uses (bm_common.cuh ring_count / ring_entry).  One CTA
// per request; out holds MAXM entries per request.
__global__ void k_emap(int H, int W, int count, const int32_t* __restrict__ origins, int32_t* out_k,
                       int32_t* out_origins, int32_t* out_rings) {
  __shared__ int off[32];
  const int q = blockIdx.x, tid = threadIdx.x;
  if (q >= count) return;
  const int pr = origins[2 * q], pc = origins[2 * q + 1];
  const int br = pr / BS * BS, bc = pc / BS * BS;
  const int r0 = max(0, br - BS), r1 = min(H, br + 2 * BS), c0 = max(0, bc - BS), c1 = min(W, bc + 2 * BS);
  bmx::RingGeom g;
  g.pr = pr;
  g.pc = pc;
  g.A0 = r0 + 2;
  g.A1 = r1 - 4;
  g.B0 = c0 + 2;
  g.B1 = c1 - 4;
  if (tid < 32) {
    const int cnt = (tid >= 1 && tid <= 30) ? bmx::ring_count(g, tid) : 0;
    int inc = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, inc, o);
      inc += tid >= o ? v : 0;
    }
    off[tid] = inc - cnt;
    if (tid == 31) out_k[q] = inc;
  }
  __syncthreads();
  const int K = off[31];
  for (int e = tid; e < K; e += blockDim.x) {
    int r = 1;
    while (r < 31 && off[r + 1] <= e) r++;
    int a, b;
    bmx::ring_entry(g, r, e - off[r], a, b);
    out_origins[((size_t)q * MAXM + e) * 2] = a - 2;  // window origin = candidate patch origin - 2
    out_origins[((size_t)q * MAXM + e) * 2 + 1] = b - 2;
    out_rings[(size_t)q * MAXM + e] = r;
  }
}

// ------------------------------------------------------- estimator stages

// NumPy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src
// pairwise_sum) of a contiguous double array: < 8 sequential, <= 128 eight
// accumulators, else split at n/2 rounded down to a multiple of 8.
__device__ __noinline__ double np_pairwise_leaf(const double* a, int n, int stride) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res += a[(size_t)i * stride];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; j++) r[j] = a[(size_t)j * stride];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] += a[(size_t)(i + j) * stride];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a[(size_t)i * stride];
  return res;
}
// the recursion unrolled at compile time (D levels cover n <= 128 * 2^D;
// no runtime recursion, so the stack size stays static)
template <int D>
__device__ __forceinline__ double np_pairwise(const double* a, int n, int stride) {
  if (n <= 128) return np_pairwise_leaf(a, n, stride);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise<D - 1>(a, n2, stride) + np_pairwise<D - 1>(a + (size_t)n2 * stride, n - n2, stride);
}
template <>
__device__ __forceinline__ double np_pairwise<0>(const double* a, int n, int stride) {
  return np_pairwise_leaf(a, n, stride);
}
__device__ __forceinline__ double np_pairwise_sum(const double* a, int n, int stride = 1) {
  return np_pairwise<5>(a, n, stride);  // n <= 4096
}

struct StageSmem {
  double y0[32];
  double L[32 * 33];   // C_YY (+ ridge) -> its lower Cholesky factor
  double cxy[4 * 32];  // C_XY (row q, col t)
  double d[MAXM];      // quadforms / distances / exponents
  double w[MAXM];      // weights
  double g[MAXM];      // Gram diagonal g_j = y_j^T C^-1 y_j (alpha)
  double red[NW][40];
  double tot[40];
  double rowv[40];
  double mean[36];
  int near[33];
  double resid[33 * 4], cdir[33 * 4];
  int fail;
};

// CTA-wide sums of N per-thread values, fixed order (warp trees, then warps in order).
template <int N>
__device__ void block_sum(double (&v)[N], StageSmem& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < N; i++) v[i] = bmx::warp_sum(v[i]);
  __syncthreads();
  if (lane == 0)
    for (int i = 0; i < N; i++) S.red[warp][i] = v[i];
  __syncthreads();
  for (int i = 0; i < N; i++) {
    double a = S.red[0][i];
    for (int w = 1; w < NW; w++) a += S.red[w][i];
    v[i] = a;
  }
  __syncthreads();
}

__device__ double block_max(double v, StageSmem& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = bmx::warp_max(v);
  __syncthreads();
  if (lane == 0) S.red[warp][0] = v;
  __syncthreads();
  double a = S.red[0][0];
  for (int w = 1; w < NW; w++) a = fmax(a, S.red[w][0]);
  __syncthreads();
  return a;
}

// Lower Cholesky of S.L (n x n, stride 33) in place on warp 0 (lanes = rows,
// left-looking column by column); S.fail = 1 when C_YY is not positive
// definite (scipy.linalg.cho_factor raises LinAlgError, estimators.py:63).
__device__ void cholesky(StageSmem& S, int n) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  bool fail = false;
  for (int j = 0; j < n && !fail; j++) {
    double t = 0.0;
    if (lane >= j && lane < n) {
      t = S.L[lane * 33 + j];
      for (int k = 0; k < j; k++) t -= S.L[lane * 33 + k] * S.L[j * 33 + k];
    }
    const double dj = __shfl_sync(FULL, t, j);
    if (!(dj > 0.0)) {
      fail = true;
      break;
    }
    const double ljj = sqrt(dj);
    __syncwarp();
    if (lane == j) S.L[j * 33 + j] = ljj;
    if (lane > j && lane < n) S.L[lane * 33 + j] = t / ljj;
    __syncwarp();
  }
  if (lane == 0) S.fail = fail;
}

// C_YY^-1 b via the factor (cho_solve): forward then back substitution.
__device__ __forceinline__ void chol_solve(const StageSmem& S, int n, double (&b)[32]) {
  for (int i = 0; i < n; i++) {
    double s = b[i];
    for (int k = 0; k < i; k++) s -= S.L[i * 33 + k] * b[k];
    b[i] = s / S.L[i * 33 + i];
  }
  for (int i = n - 1; i >= 0; i--) {
    double s = b[i];
    for (int k = i + 1; k < n; k++) s -= S.L[k * 33 + i] * b[k];
    b[i] = s / S.L[i * 33 + i];
  }
}

struct StageArgs {
  int stage, count, max_m;
  double sigma2;
  const int32_t* n_y;
  const int32_t* m;
  const double* y0;     // [count][32]
  const double* x;      // [count][max_m][4]
  const double* y;      // [count][max_m][32]
  const double* beta;   // [count]
  double* cov;          // [count][BM_COV_DOUBLES]
  double* out_w;        // [count][max_m]
  double* out_mat;      // [count][max_m][32]
  double* out_scalars;  // [count][40]
  int32_t* out_status;  // [count]
  double* scratch;      // [count][max_m][32] (alpha: C^-1 y_j)
};

// quadforms d_j = (y0 - y_j)^T C^-1 (y0 - y_j) (_context_quadforms,
// estimators.py:154-158: cho_solve, then the row dot product)
__device__ void quadforms(const StageArgs& A, StageSmem& S, const double* Y, int m, int n) {
  for (int j = threadIdx.x; j < m; j += NT) {
    double diff[32], sol[32];
    for (int t = 0; t < 32; t++) diff[t] = sol[t] = t < n ? S.y0[t] - Y[(size_t)j * 32 + t] : 0.0;
    chol_solve(S, n, sol);
    double dd = 0.0;
    for (int t = 0; t < n; t++) dd = fma(diff[t], sol[t], dd);
    S.d[j] = dd;
  }
  __syncthreads();
}

// normalised weights at beta from S.d into S.w (_weights_from_quadforms,
// estimators.py:161-164); returns (shift, total of shifted)
__device__ void beta_weights(StageSmem& S, int m, double beta, double& shift, double& total) {
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < m; j += NT) mx = fmax(mx, -S.d[j] / (2.0 * beta));
  shift = block_max(mx, S);
  for (int j = threadIdx.x; j < m; j += NT) S.w[j] = exp(-S.d[j] / (2.0 * beta) - shift);
  __syncthreads();
  if (threadIdx.x == 0) S.tot[0] = np_pairwise_sum(S.w, m);
  __syncthreads();
  total = S.tot[0];
  for (int j = threadIdx.x; j < m; j += NT) S.w[j] = S.w[j] / total;
  __syncthreads();
}

// w @ [x | y] -> S.tot[0..3] = x~, S.tot[4..4+n) = y~ (predict_xy, estimators.py:184-186)
__device__ void predict(StageSmem& S, const double* X, const double* Y, int m, int n) {
  double v[36];
  for (int i = 0; i < 36; i++) v[i] = 0.0;
  for (int j = threadIdx.x; j < m; j += NT) {
    const double wj = S.w[j];
    for (int q = 0; q < 4; q++) v[q] = fma(wj, X[(size_t)j * 4 + q], v[q]);
    for (int t = 0; t < 32; t++)
      if (t < n) v[4 + t] = fma(wj, Y[(size_t)j * 32 + t], v[4 + t]);
  }
  block_sum<36>(v, S);
  if (threadIdx.x < 36) S.tot[threadIdx.x] = v[threadIdx.x];
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) k_stages(StageArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StageSmem& S = *reinterpret_cast<StageSmem*>(smem_raw);
  const int i = blockIdx.x, tid = threadIdx.x;
  const int n = A.n_y[i], m = A.m[i];
  const double* X = A.x + (size_t)i * A.max_m * 4;
  const double* Y = A.y + (size_t)i * A.max_m * 32;
  double* cov = A.cov + (size_t)i * BM_COV_DOUBLES;  // c_xx[16] c_xy[4][32] c_yy[32][32] ridge
  double* sc = A.out_scalars + (size_t)i * 40;
  if (tid < 32) S.y0[tid] = tid < n ? A.y0[(size_t)i * 32 + tid] : 0.0;
  if (tid == 0) S.fail = 0;
  __syncthreads();
  int status = 0;

  if (A.stage == BM_STAGE_COVARIANCE) {
    // sample_covariance (estimators.py:135-151): z = [x | y], means in
    // NumPy's axis-0 order (row by row), C = centred^T centred / (m - 1),
    // ridge 1e-6 tr(C_YY) / N_y (1e-6 if the trace is 0)
    const int dz = 4 + n;
    if (tid < dz) {
      double s = 0.0;
      for (int j = 0; j < m; j++) s += tid < 4 ? X[(size_t)j * 4 + tid] : Y[(size_t)j * 32 + tid - 4];
      S.mean[tid] = s / m;
    }
    __syncthreads();
    for (int e = tid; e < dz * dz; e += NT) {
      const int a = e / dz, b = e % dz;
      if (b < a) continue;
      double s = 0.0;
      for (int j = 0; j < m; j++) {
        const double za = (a < 4 ? X[(size_t)j * 4 + a] : Y[(size_t)j * 32 + a - 4]) - S.mean[a];
        const double zb = (b < 4 ? X[(size_t)j * 4 + b] : Y[(size_t)j * 32 + b - 4]) - S.mean[b];
        s = fma(za, zb, s);
      }
      const double v = s / (double)(m - 1);
      if (a < 4 && b < 4) {
        cov[a * 4 + b] = v;
        cov[b * 4 + a] = v;
      } else if (a < 4) {
        cov[16 + a * 32 + (b - 4)] = v;
      } else {
        S.L[(a - 4) * 33 + (b - 4)] = v;
        S.L[(b - 4) * 33 + (a - 4)] = v;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const double tr = np_pairwise_sum(S.L, n, 34);  // np.trace(c_yy)
      const double ridge = tr > 0.0 ? 1e-6 * tr / n : 1e-6;
      cov[16 + 128 + 1024] = ridge;
      for (int t = 0; t < n; t++) S.L[t * 33 + t] += ridge;
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += NT) {
      const int a = e >> 5, b = e & 31;
      cov[16 + 128 + e] = (a < n && b < n) ? S.L[a * 33 + b] : 0.0;
    }
  } else if (A.stage == BM_STAGE_IDL_WEIGHTS) {
    // idl_weights (estimators.py:112-119): d2 per row in NumPy's pairwise
    // order, expo = -d2 / (2 sigma2 N_y), raw_sum = sum exp(expo), w = exp(expo - max) / sum
    const double c = 2.0 * A.sigma2 * n;
    double mx = -INFINITY;
    for (int j = tid; j < m; j += NT) {
      double sq[32];
      for (int t = 0; t < n; t++) {
        const double dd = Y[(size_t)j * 32 + t] - S.y0[t];
        sq[t] = dd * dd;
      }
      const double e = -np_pairwise_sum(sq, n) / c;
      S.d[j] = e;
      S.g[j] = exp(e);
      mx = fmax(mx, e);
    }
    mx = block_max(mx, S);
    for (int j = tid; j < m; j += NT) S.w[j] = exp(S.d[j] - mx);
    __syncthreads();
    if (tid == 0) {
      S.tot[0] = np_pairwise_sum(S.g, m);  // raw_sum (may underflow to 0)
      S.tot[1] = np_pairwise_sum(S.w, m);
    }
    __syncthreads();
    for (int j = tid; j < m; j += NT) {
      A.out_w[(size_t)i * A.max_m + j] = S.w[j] / S.tot[1];
      if (A.out_mat) A.out_mat[((size_t)i * A.max_m + j) * 32] = S.g[j];  // raw_idl_weights (estimators.py:105-109)
    }
    if (tid == 0) sc[0] = S.tot[0];
  } else if (A.stage == BM_STAGE_PREDICT) {
    // predict_xy (estimators.py:184-186): weights given in out_w
    for (int j = tid; j < m; j += NT) S.w[j] = A.out_w[(size_t)i * A.max_m + j];
    __syncthreads();
    predict(S, X, Y, m, n);
    if (tid < 4 + n) sc[tid] = S.tot[tid];
  } else {
    // stages that need C_YY's factor (given: cov)
    for (int e = tid; e < 32 * 32; e += NT) {
      const int a = e >> 5, b = e & 31;
      if (a < n && b < n) S.L[a * 33 + b] = cov[16 + 128 + e];
    }
    for (int e = tid; e < 4 * 32; e += NT) S.cxy[e] = cov[16 + e];
    __syncthreads();
    cholesky(S, n);
    __syncthreads();
    if (S.fail) {
      status = 2;  // LinAlgError
    } else if (A.stage == BM_STAGE_SOLVE) {
      // CovarianceBlocks.solve_yy (estimators.py:66-68) for the m right-hand sides y_j
      for (int j = tid; j < m; j += NT) {
        double b[32];
        for (int t = 0; t < 32; t++) b[t] = t < n ? Y[(size_t)j * 32 + t] : 0.0;
        chol_solve(S, n, b);
        for (int t = 0; t < n; t++) A.out_mat[((size_t)i * A.max_m + j) * 32 + t] = b[t];
      }
    } else if (A.stage == BM_STAGE_KERNEL_WEIGHTS) {
      // kernel_weights (estimators.py:167-181)
      quadforms(A, S, Y, m, n);
      double shift, total;
      beta_weights(S, m, A.beta[i], shift, total);
      for (int j = tid; j < m; j += NT) A.out_w[(size_t)i * A.max_m + j] = S.w[j];
      if (tid == 0) sc[0] = exp(shift) * total;  // raw_sum (estimators.py:179-180)
    } else if (A.stage == BM_STAGE_OPTIMIZE_BETA) {
      // optimize_beta / _beta_search (estimators.py:189-206): strict-< argmin
      // of eps(beta) = ||y0 - w(beta) @ y||^2 over BETA_GRID, ties -> smaller beta
      quadforms(A, S, Y, m, n);
      double best_eps = INFINITY;
      int best = 0;
      for (int gi = 0; gi < bmx::NBETA; gi++) {
        const double beta = ldexp(1.0, gi - 8);
        double shift, total;
        beta_weights(S, m, beta, shift, total);
        predict(S, X, Y, m, n);
        if (tid == 0) {
          double sq[32];
          for (int t = 0; t < n; t++) {
            const double dd = S.y0[t] - S.tot[4 + t];
            sq[t] = dd * dd;
          }
          S.rowv[0] = np_pairwise_sum(sq, n);
        }
        __syncthreads();
        const double eps = S.rowv[0];
        if (eps < best_eps) {
          best_eps = eps;
          best = gi;
        }
        __syncthreads();
      }
      if (tid == 0) {
        sc[0] = ldexp(1.0, best - 8);
        sc[1] = best_eps;
      }
    } else if (A.stage == BM_STAGE_OPTIMIZE_ALPHA) {
      // optimize_alpha (estimators.py:209-245)
      const double beta = A.beta[i];
      double alpha = 0.0;
      if (m >= 2) {
        const int k = min(n + 1, m);
        // Euclidean distances (pairwise order) and the stable k nearest: rank by (d, index)
        for (int j = tid; j < m; j += NT) {
          double sq[32];
          for (int t = 0; t < n; t++) {
            const double dd = Y[(size_t)j * 32 + t] - S.y0[t];
            sq[t] = dd * dd;
          }
          S.d[j] = np_pairwise_sum(sq, n);
        }
        __syncthreads();
        for (int j = tid; j < m; j += NT) {
          const double dj = S.d[j];
          int rank = 0;
          for (int l = 0; l < m; l++) rank += (S.d[l] < dj) || (S.d[l] == dj && l < j);
          if (rank < k) S.near[rank] = j;
        }
        // sol_j = C^-1 y_j (scratch), g_j = y_j . sol_j
        double* sol = A.scratch + (size_t)i * A.max_m * 32;
        for (int j = tid; j < m; j += NT) {
          double b[32];
          for (int t = 0; t < 32; t++) b[t] = t < n ? Y[(size_t)j * 32 + t] : 0.0;
          chol_solve(S, n, b);
          double gg = 0.0;
          for (int t = 0; t < n; t++) {
            sol[(size_t)j * 32 + t] = b[t];
            gg = fma(Y[(size_t)j * 32 + t], b[t], gg);
          }
          S.g[j] = gg;
        }
        __syncthreads();
        for (int r = 0; r < k; r++) {
          const int ni = S.near[r];
          // q_ij = g_i + g_j - 2 y_i^T C^-1 y_j; expo = -q / (2 beta), self excluded
          double mx = -INFINITY;
          for (int j = tid; j < m; j += NT) {
            double dot = 0.0;
            for (int t = 0; t < n; t++) dot = fma(Y[(size_t)ni * 32 + t], sol[(size_t)j * 32 + t], dot);
            const double e = j == ni ? -INFINITY : -(S.g[ni] + S.g[j] - 2.0 * dot) / (2.0 * beta);
            S.w[j] = e;
            mx = fmax(mx, e);
          }
          mx = block_max(mx, S);
          for (int j = tid; j < m; j += NT) S.w[j] = exp(S.w[j] - mx);
          __syncthreads();
          if (tid == 0) S.tot[39] = np_pairwise_sum(S.w, m);
          __syncthreads();
          const double tw = S.tot[39];
          for (int j = tid; j < m; j += NT) S.w[j] = S.w[j] / tw;
          __syncthreads();
          predict(S, X, Y, m, n);  // x_pred_i, y_pred_i
          if (tid < 32) {
            // corr_i = C^-1 (y_i - y_pred_i); c_i = C_XY corr_i; r_i = x_i - x_pred_i
            double b[32];
            for (int t = 0; t < 32; t++) b[t] = t < n ? Y[(size_t)ni * 32 + t] - S.tot[4 + t] : 0.0;
            chol_solve(S, n, b);
            if (tid < 4) {
              double c = 0.0;
              for (int t = 0; t < n; t++) c = fma(S.cxy[tid * 32 + t], b[t], c);
              S.cdir[tid * k + r] = c;
              S.resid[tid * k + r] = X[(size_t)ni * 4 + tid] - S.tot[tid];
            }
          }
          __syncthreads();
        }
        if (tid == 0) {
          double cc[132], rc[132];
          for (int e = 0; e < 4 * k; e++) {
            cc[e] = S.cdir[e] * S.cdir[e];
            rc[e] = S.resid[e] * S.cdir[e];
          }
          const double den = np_pairwise_sum(cc, 4 * k), num = np_pairwise_sum(rc, 4 * k);
          if (!(den < 1e-12)) {
            alpha = num / den;
            alpha = alpha < 0.0 ? 0.0 : (alpha > 4.0 ? 4.0 : alpha);  // np.clip keeps NaN
          }
        }
      }
      if (tid == 0) sc[0] = alpha;
    }
  }
  if (tid == 0) A.out_status[i] = status;
}

int status_of(cudaError_t e) { return e == cudaSuccess ? BM_OK : BM_ERR_CUDA; }

}  // namespace bm_api

using namespace bm_api;

extern "C" {

int bm_extract_targets(int height, int width, const double* pixels, const uint8_t* states, int32_t count,
                       const int32_t* origins, uint32_t* out_layouts, int32_t* out_n_y, double* out_y0,
                       void* stream) {
  if (height < 1 || width < 1 || count < 0 || !pixels || !states) return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  k_extract<<<(count * 32 + 255) / 256, 256, 0, (cudaStream_t)stream>>>(height, width, pixels, states, count,
                                                                       origins, out_layouts, out_n_y, out_y0);
  return status_of(cudaGetLastError());
}

int bm_collect(int height, int width, const double* pixels, const uint8_t* states, int32_t requests,
               const int32_t* origins, const int32_t* offsets, const int32_t* counts, const uint32_t* layouts,
               double* out_x, double* out_y, int32_t* out_m, void* stream) {
  if (height < 1 || width < 1 || requests < 0 || !pixels || !states) return BM_ERR_ARGS;
  if (requests == 0) return BM_OK;
  k_collect<<<requests, NT, 0, (cudaStream_t)stream>>>(height, width, pixels, states, origins, offsets, counts,
                                                        layouts, out_x, out_y, out_m);
  return status_of(cudaGetLastError());
}

int bm_patch_scores(int height, int width, const uint8_t* states, int32_t count, const int32_t* origins,
                    int32_t* out_avail, int32_t* out_usable, void* stream) {
  if (height < 1 || width < 1 || count < 0 || !states) return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  k_patch_scores<<<(count + 127) / 128, 128, 0, (cudaStream_t)stream>>>(height, width, states, count, origins,
                                                                       out_avail, out_usable);
  return status_of(cudaGetLastError());
}

int bm_build_schedule(int height, int width, const uint8_t* states, int32_t count, const int32_t* blocks,
                      int32_t* out_n, int32_t* out_origins, int32_t* out_reliability, void* stream) {
  if (height < 1 || width < 1 || count < 0 || !states) return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  k_schedule<<<(count * 32 + 127) / 128, 128, 0, (cudaStream_t)stream>>>(height, width, states, count, blocks, out_n,
                                                                         out_origins, out_reliability);
  return status_of(cudaGetLastError());
}

int bm_expansion_maps(int height, int width, int32_t count, const int32_t* origins, int32_t* out_k,
                      int32_t* out_origins, int32_t* out_rings, void* stream) {
  if (height < 1 || width < 1 || count < 0) return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  k_emap<<<count, NT, 0, (cudaStream_t)stream>>>(height, width, count, origins, out_k, out_origins, out_rings);
  return status_of(cudaGetLastError());
}

int bm_estimator_stages(int32_t stage, int32_t count, int32_t max_m, double sigma2, const int32_t* n_y,
                        const int32_t* m, const double* y0, const double* x, const double* y, const double* beta,
                        double* cov, double* out_w, double* out_mat, double* out_scalars, int32_t* out_status,
                        void* stream_) {
  if (stage < BM_STAGE_COVARIANCE || stage > BM_STAGE_SOLVE || count < 0 || max_m < 0 || max_m > MAXM ||
      !(sigma2 > 0.0))
    return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  cudaError_t e;
  const size_t smem = sizeof(StageSmem);
  bm_host::DevState& D = bm_host::dev_state();
  if (!D.stage_attr.load()) {
    if ((e = cudaFuncSetAttribute(k_stages, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return status_of(e);
    D.stage_attr = true;
  }
  double* scratch = nullptr;
  if (stage == BM_STAGE_OPTIMIZE_ALPHA &&
      (e = cudaMallocAsync((void**)&scratch, (size_t)count * (max_m > 0 ? max_m : 1) * 32 * 8, stream)) != cudaSuccess)
    return status_of(e);
  StageArgs A{stage, count, max_m, sigma2, n_y, m, y0, x, y, beta, cov, out_w, out_mat, out_scalars, out_status,
              scratch};
  k_stages<<<count, NT, smem, stream>>>(A);
  e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, stream);
  return status_of(e);
}

}  // extern "C"
