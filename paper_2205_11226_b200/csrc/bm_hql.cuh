// bm_hql.cuh — the FP64 high-quality layer (hql_estimate, estimators.py:248-286)
// on B200 FP64 tensor cores (mma.sync.m8n8k4.f64, "DMMA").
//
// Every candidate-sized contraction of the reference is a small GEMM with
// K = the candidate count M' (<= 1849):
//   covariance    C   = Zc^T Zc                 (40 x 40, K = M')   estimators.py:140-142
//   quadforms     V   = L^-1 (y0 - Y)^T, d = |V_j|^2 (32 x M')       estimators.py:154-158
//   beta grid     P   = W_beta [Y|X|1]          (24 x 40, K = M')   estimators.py:197-206
//   alpha Gram    G   = V_near^T V, q = d_i + d_j - 2G (40 x M')     estimators.py:225-229
//   LOO sums      Zp  = W_loo [Y|X|1]           (40 x 40, K = M')   estimators.py:231-238
// Warps own disjoint candidate slices (no barrier inside a pass), keep all
// output tiles of their slice in registers, and combine them with one
// fixed-order 3-round tree reduction -> deterministic results.
// The exponentials of the weight matrices are computed in the A-fragment
// registers (each (row, candidate) weight exactly once).
#pragma once
#include "bm_common.cuh"
#include "bm_estimators.cuh"

namespace bm {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Z view: column col of candidate j is ptr[base(j) + coff[col]] (coff >= 0) or
// the constant cconst[col].  Columns: 0..31 = y (N_y used, rest 0), 32..35 = x,
// 36 = 1 (sums), 37..39 = 0.
struct ZView {
  const double* ptr;
  const uint16_t* cand;  // tile positions (fused kernel) or nullptr (dense, stride 40)
  __device__ __forceinline__ int base(int j) const { return cand ? (int)cand[j] : j * 40; }
};

constexpr int LS = 36;  // stride of Linv / Vn: conflict-free A-fragment loads (36 = 4 mod 16)

struct HqlSmem {
  int16_t coff[40];
  double cconst[40];
  double mean[40];
  double Linv[32 * LS];
  double Bm[4 * 32];     // C_XY L^-T
  double cxy[4 * 32];
  double R1[3840];       // tree-reduction partials / cyy+L / u
  double R2[1600];       // P (24x40) / Vn (40x36) / Zp (40x40)
  double wmin[NWARP][40];
  double qmin[40];
  double dn[40];
  int near[40];
  double cmat[4 * KMAX], rmat[4 * KMAX];
  double xt[4], yt[32];
  double redmin[2][NWARP];
  int redidx[2][NWARP];
  int gbest;
  int fail;
};

// per-CTA global scratch (doubles)
constexpr size_t HQL_V = 0;                                  // V   [32][MAXCAND]
constexpr size_t HQL_Q = HQL_V + (size_t)32 * MAXCAND;       // q   [MAXCAND/8][5][32][2] fragment-native
constexpr size_t HQL_D = HQL_Q + (size_t)(MAXCAND / 8) * 5 * 64;
constexpr size_t HQL_E2 = HQL_D + MAXCAND;
constexpr size_t HQL_Z = HQL_E2 + MAXCAND;                   // dense Z [MAXCAND][40] (estimator API only)
constexpr size_t HQL_SCRATCH_FUSED = HQL_Z;
constexpr size_t HQL_SCRATCH_DENSE = HQL_Z + (size_t)MAXCAND * 40;

__device__ __forceinline__ double zval(const double* ptr, int b, int off, double cst) {
  return off >= 0 ? ptr[b + off] : cst;
}

// Fixed-order tree reduction of per-warp register tiles (8 warps -> warp 0).
template <int N>
__device__ __forceinline__ void tree_reduce(double (&acc)[N], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp >= 4) {
#pragma unroll
    for (int i = 0; i < N; i++) red[((warp - 4) * N + i) * 32 + lane] = acc[i];
  }
  __syncthreads();
  if (warp < 4) {
#pragma unroll
    for (int i = 0; i < N; i++) acc[i] += red[(warp * N + i) * 32 + lane];
  }
  __syncthreads();
  if (warp == 2 || warp == 3) {
#pragma unroll
    for (int i = 0; i < N; i++) red[((warp - 2) * N + i) * 32 + lane] = acc[i];
  }
  __syncthreads();
  if (warp < 2) {
#pragma unroll
    for (int i = 0; i < N; i++) acc[i] += red[(warp * N + i) * 32 + lane];
  }
  __syncthreads();
  if (warp == 1) {
#pragma unroll
    for (int i = 0; i < N; i++) red[i * 32 + lane] = acc[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < N; i++) acc[i] += red[i * 32 + lane];
  }
}

// Column table of the Z view for target layout n (uoff: tile offsets of the
// n usable context positions; nullptr for the dense layout).
__device__ __forceinline__ void hql_columns(HqlSmem& H, int n, const int16_t* uoff) {
  const int t = threadIdx.x;
  if (t < 40) {
    int16_t off = -1;
    double c = 0.0;
    if (t < n) off = uoff ? uoff[t] : (int16_t)t;
    else if (t >= 32 && t < 36) {
      const int q = t - 32;
      off = uoff ? (int16_t)((2 + (q >> 1)) * TS + 2 + (q & 1)) : (int16_t)t;
    } else if (t == 36) c = 1.0;
    H.coff[t] = off;
    H.cconst[t] = c;
  }
}

// The HQL pipeline for one patch.  Inputs: zv (candidates), m >= 2, n, y0
// (shared, [32]).  Outputs in H/out: ok, vals[4], beta, alpha, gap.
struct HqlOut {
  double vals[4];
  double beta, alpha;
  float gap;
  int ok;
};

__device__ void hql_mma(const ZView& zv, int m, int n, const double* y0, HqlSmem& H, double* __restrict__ gs,
                        HqlOut& out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double* gV = gs + HQL_V;
  double* gQ = gs + HQL_Q;
  double* gD = gs + HQL_D;
  double* gE2 = gs + HQL_E2;
  const int nks = (m + 3) >> 2;  // k-steps of 4 candidates
  const int nct = (m + 7) >> 3;  // column tiles of 8 candidates

  // ---------------------------------------------------------------- means
  {
    double a0 = 0.0, a1 = 0.0;
    const int off0 = H.coff[lane], off1 = lane < 8 ? H.coff[32 + lane] : -1;
    const double c0 = H.cconst[lane], c1 = lane < 8 ? H.cconst[32 + lane] : 0.0;
    for (int j = warp; j < m; j += NWARP) {
      const int b = zv.base(j);
      a0 += zval(zv.ptr, b, off0, c0);
      a1 += zval(zv.ptr, b, off1, c1);
    }
    H.wmin[warp][lane] = a0;
    if (lane < 8) H.wmin[warp][32 + lane] = a1;
    __syncthreads();
    if (tid < 40) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; w++) s += H.wmin[w][tid];
      H.mean[tid] = s / m;  // z.mean(axis=0)
    }
    __syncthreads();
  }

  // ------------------------------------------------- covariance (DMMA)
  {
    int off[5];
    double cst[5], mu[5];
#pragma unroll
    for (int tl = 0; tl < 5; tl++) {
      const int col = 8 * tl + g;
      off[tl] = H.coff[col];
      cst[tl] = H.cconst[col];
      mu[tl] = H.mean[col];
    }
    double acc[28];
#pragma unroll
    for (int i = 0; i < 28; i++) acc[i] = 0.0;
    for (int s = warp; s < nks; s += NWARP) {
      const int j = 4 * s + t4;
      const bool valid = j < m;
      const int b = valid ? zv.base(j) : 0;
      double f[5];
#pragma unroll
      for (int tl = 0; tl < 5; tl++) f[tl] = valid ? zval(zv.ptr, b, off[tl], cst[tl]) - mu[tl] : 0.0;
      int idx = 0;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int bb = a; bb < 5; bb++) {
          dmma(acc[2 * idx], acc[2 * idx + 1], f[a], f[bb]);
          idx++;
        }
    }
    tree_reduce<28>(acc, H.R1);
    double* cyy = H.R1 + 3840 - 2 * 32 * 33;  // tail of R1 (partials no longer needed)
    double* L = cyy + 32 * 33;
    if (warp == 0) {
      const double inv = 1.0 / (double)(m - 1);
      int idx = 0;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int bb = a; bb < 5; bb++) {
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int ra = 8 * a + g, cb = 8 * bb + 2 * t4 + e;
            const double v = acc[2 * idx + e] / (double)(m - 1);
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
    __syncthreads();
    // ridge (estimators.py:148-150) and Cholesky (CovarianceBlocks._factor)
    if (warp == 0) {
      double tr = 0.0;
      if (lane == 0) {
        tr = pairwise_sum_n(n, [&](int i) { return cyy[i * 33 + i]; });
        const double ridge = tr > 0.0 ? 1e-6 * tr / n : 1e-6;
        for (int i = 0; i < n; i++) cyy[i * 33 + i] += ridge;
      }
      __syncwarp();
      bool fail = false;
      for (int j = 0; j < n; j++) {
        double t = 0.0;
        if (lane >= j && lane < n) {
          t = cyy[lane * 33 + j];
          for (int k = 0; k < j; k++) t = fma(-L[lane * 33 + k], L[j * 33 + k], t);
        }
        const double sd = __shfl_sync(FULL, t, j);
        if (!(sd > 0.0)) { fail = true; break; }
        const double d = sqrt(sd);
        if (lane == j) L[j * 33 + j] = d;
        if (lane > j && lane < n) L[lane * 33 + j] = t / d;
        __syncwarp();
      }
      if (lane == 0) H.fail = fail;
      __syncwarp();
      if (!fail) {
        // L^-1, one column per lane (forward substitution on e_c), identity beyond n
        const int c = lane;
        for (int i = 0; i < 32; i++) {
          double x;
          if (i < c) x = 0.0;
          else if (i >= n) x = (i == c) ? 1.0 : 0.0;
          else if (i == c) x = 1.0 / L[i * 33 + i];
          else {
            double s = 0.0;
            for (int k = c; k < i; k++) s = fma(L[i * 33 + k], H.Linv[k * LS + c], s);
            x = -s / L[i * 33 + i];
          }
          H.Linv[i * LS + c] = x;
        }
      }
    }
    __syncthreads();
    if (H.fail) {
      if (tid == 0) out.ok = 0;
      return;
    }
    // Bm = C_XY L^-T : Bm[q][t] = sum_s C_XY[q][s] Linv[t][s]
    if (tid < 128) {
      const int q = tid >> 5, t = tid & 31;
      double s = 0.0;
      for (int k = 0; k < n; k++) s = fma(H.cxy[q * 32 + k], H.Linv[t * LS + k], s);
      H.Bm[q * 32 + t] = t < n ? s : 0.0;
    }
  }

  // ------------------------------------- V = L^-1 (y0 - Y)^T and d (DMMA)
  {
    double y0r[8];
    int offy[8];
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const int dim = 4 * kk + t4;
      y0r[kk] = dim < n ? y0[dim] : 0.0;
      offy[kk] = H.coff[dim];
    }
    for (int c = warp; c < nct; c += NWARP) {
      const int jB = 8 * c + g;
      const bool vb = jB < m;
      const int bB = vb ? zv.base(jB) : 0;
      double fb[8];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) {
        const int dim = 4 * kk + t4;
        fb[kk] = (vb && dim < n) ? y0r[kk] - zv.ptr[bB + offy[kk]] : 0.0;
      }
      double acc[8];
#pragma unroll
      for (int i = 0; i < 8; i++) acc[i] = 0.0;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int kk = 0; kk < 2 * r + 2; kk++)
          dmma(acc[2 * r], acc[2 * r + 1], H.Linv[(8 * r + g) * LS + 4 * kk + t4], fb[kk]);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int row = 8 * r + g;
        const int col = 8 * c + 2 * t4;
        if (col < m) gV[(size_t)row * MAXCAND + col] = acc[2 * r];
        if (col + 1 < m) gV[(size_t)row * MAXCAND + col + 1] = acc[2 * r + 1];
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
        if (col < m) gD[col] = s0;
        if (col + 1 < m) gD[col + 1] = s1;
      }
    }
    // Euclidean distances in NumPy's order (optimize_alpha's nearest set, estimators.py:222)
    for (int j = tid; j < m; j += NT) {
      const int b = zv.base(j);
      double v[32];
#pragma unroll
      for (int t = 0; t < 32; t++) v[t] = t < n ? zv.ptr[b + H.coff[t]] - y0[t] : 0.0;
      gE2[j] = pairwise_sq32(v, n);
    }
  }
  __syncthreads();
  double dmin;
  {
    double mn = INFINITY;
    for (int j = tid; j < m; j += NT) mn = fmin(mn, gD[j]);
    mn = warp_min(mn);
    if (lane == 0) H.redmin[0][warp] = mn;
    __syncthreads();
    dmin = H.redmin[0][0];
#pragma unroll
    for (int w = 1; w < NWARP; w++) dmin = fmin(dmin, H.redmin[0][w]);
  }

  // ------------------------------------------------ beta grid (DMMA)
  int offz[5];
  double cstz[5];
#pragma unroll
  for (int ct = 0; ct < 5; ct++) {
    offz[ct] = H.coff[8 * ct + g];
    cstz[ct] = H.cconst[8 * ct + g];
  }
  {
    double sc[3];
#pragma unroll
    for (int r = 0; r < 3; r++) sc[r] = ldexp(1.0, 7 - (8 * r + g));  // 1/(2 beta)
    double acc[30];
#pragma unroll
    for (int i = 0; i < 30; i++) acc[i] = 0.0;
    for (int s = warp; s < nks; s += NWARP) {
      const int j = 4 * s + t4;
      const bool valid = j < m;
      const int b = valid ? zv.base(j) : 0;
      const double delta = valid ? dmin - gD[j] : 0.0;
      double fa[3], fb[5];
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const int gi = 8 * r + g;
        fa[r] = (valid && gi < NBETA) ? exp(delta * sc[r]) : 0.0;  // exp(expo - expo.max())
      }
#pragma unroll
      for (int ct = 0; ct < 5; ct++) fb[ct] = valid ? zval(zv.ptr, b, offz[ct], cstz[ct]) : 0.0;
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int ct = 0; ct < 5; ct++) dmma(acc[2 * (r * 5 + ct)], acc[2 * (r * 5 + ct) + 1], fa[r], fb[ct]);
    }
    tree_reduce<30>(acc, H.R1);
    double* P = H.R2;  // [24][40]
    if (warp == 0) {
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          P[(8 * r + g) * 40 + 8 * ct + 2 * t4] = acc[2 * (r * 5 + ct)];
          P[(8 * r + g) * 40 + 8 * ct + 2 * t4 + 1] = acc[2 * (r * 5 + ct) + 1];
        }
      __syncwarp();
      // eps_g = ||y0 - y~0(beta_g)||^2 in NumPy's pairwise order; strict < argmin
      double eps = INFINITY;
      if (lane < NBETA) {
        const double S = P[lane * 40 + 36];
        eps = pairwise_sum_n(n, [&](int t) {
          const double d = y0[t] - P[lane * 40 + t] / S;
          return __dmul_rn(d, d);
        });
      }
      double best_eps = INFINITY;
      int best = 0;
      for (int gg = 0; gg < NBETA; gg++) {
        const double e = __shfl_sync(FULL, eps, gg);
        if (e < best_eps) { best_eps = e; best = gg; }
      }
      double ya = lane < n ? fabs(y0[lane]) : 0.0;
      ya = warp_max(ya);
      const double dy = 1e-11 * ya;
      const double noise = 2.0 * sqrt(best_eps * n) * dy + n * dy * dy + 1e-300;
      double gap = INFINITY;
      for (int gg = 0; gg < NBETA; gg++) {
        const double e = __shfl_sync(FULL, eps, gg);
        if (gg != best) gap = fmin(gap, fabs(e - best_eps) / noise);
      }
      const double S = P[best * 40 + 36];
      H.yt[lane] = lane < n ? P[best * 40 + lane] / S : 0.0;
      if (lane < 4) H.xt[lane] = P[best * 40 + 32 + lane] / S;
      if (lane == 0) {
        H.gbest = best;
        out.beta = ldexp(1.0, best - 8);
        out.gap = (float)gap;
      }
    }
    __syncthreads();
  }
  const double sb = ldexp(1.0, 7 - H.gbest);
  const int k = min(n + 1, m);

  // ------------------------------- nearest k by Euclidean distance (stable)
  {
    double ev[MAXCAND / NT];
#pragma unroll
    for (int i = 0; i < MAXCAND / NT; i++) {
      const int j = tid + i * NT;
      ev[i] = j < m ? gE2[j] : INFINITY;
    }
    unsigned taken = 0;
    for (int it = 0; it < k; it++) {
      double bv = INFINITY;
      int bj = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < MAXCAND / NT; i++) {
        const int j = tid + i * NT;
        if (!((taken >> i) & 1u) && (ev[i] < bv || (ev[i] == bv && j < bj))) { bv = ev[i]; bj = j; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const int oj = __shfl_xor_sync(FULL, bj, o);
        if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
      }
      const int slot = it & 1;
      if (lane == 0) { H.redmin[slot][warp] = bv; H.redidx[slot][warp] = bj; }
      __syncthreads();
      double v = H.redmin[slot][0];
      int jj = H.redidx[slot][0];
#pragma unroll
      for (int w = 1; w < NWARP; w++)
        if (H.redmin[slot][w] < v || (H.redmin[slot][w] == v && H.redidx[slot][w] < jj)) {
          v = H.redmin[slot][w];
          jj = H.redidx[slot][w];
        }
      if ((jj % NT) == tid) taken |= 1u << (jj / NT);
      if (tid == 0) H.near[it] = jj;
    }
    __syncthreads();
  }
  // stage V columns of the nearest set: Vn[i][t] (A fragments of the Gram GEMM)
  double* Vn = H.R2;  // [40][LS]
  for (int o = tid; o < 40 * 32; o += NT) {
    const int i = o >> 5, t = o & 31;
    Vn[i * LS + t] = i < k ? gV[(size_t)t * MAXCAND + H.near[i]] : 0.0;
  }
  if (tid < 40) H.dn[tid] = tid < k ? gD[H.near[tid]] : 0.0;
  __syncthreads();

  // ------------------- q_ij = (y_i - y_j)^T C^-1 (y_i - y_j) (DMMA Gram)
  {
    double mins[5];
    int nr[5];
#pragma unroll
    for (int r = 0; r < 5; r++) {
      mins[r] = INFINITY;
      const int i = 8 * r + g;
      nr[r] = i < k ? H.near[i] : -1;
    }
    for (int c = warp; c < nct; c += NWARP) {
      const int jB = 8 * c + g;
      double fb[8];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) fb[kk] = jB < m ? gV[(size_t)(4 * kk + t4) * MAXCAND + jB] : 0.0;
      const int col = 8 * c + 2 * t4;
      const double d0 = col < m ? gD[col] : 0.0, d1 = col + 1 < m ? gD[col + 1] : 0.0;
#pragma unroll
      for (int r = 0; r < 5; r++) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk++) dmma(a0, a1, Vn[(8 * r + g) * LS + 4 * kk + t4], fb[kk]);
        const int i = 8 * r + g;
        const double di = H.dn[i];
        const double q0 = di + d0 - 2.0 * a0, q1 = di + d1 - 2.0 * a1;
        double* qp = gQ + ((size_t)(c * 5 + r) * 32 + lane) * 2;
        qp[0] = q0;
        qp[1] = q1;
        if (i < k) {
          if (col < m && col != nr[r]) mins[r] = fmin(mins[r], q0);
          if (col + 1 < m && col + 1 != nr[r]) mins[r] = fmin(mins[r], q1);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 5; r++) {
      mins[r] = fmin(mins[r], __shfl_xor_sync(FULL, mins[r], 1));
      mins[r] = fmin(mins[r], __shfl_xor_sync(FULL, mins[r], 2));
      if (t4 == 0) H.wmin[warp][8 * r + g] = mins[r];
    }
    __syncthreads();
    if (tid < 40) {
      double mn = H.wmin[0][tid];
#pragma unroll
      for (int w = 1; w < NWARP; w++) mn = fmin(mn, H.wmin[w][tid]);
      H.qmin[tid] = mn;
    }
    __syncthreads();
  }

  // ------------------------ leave-one-out sums Zp = W [Y|X|1] (DMMA)
  double* Zp = H.R2;  // [40][40] (Vn is dead)
  for (int pass = 0; pass < 2; pass++) {
    const int r0 = pass ? 3 : 0, nrow = pass ? 2 : 3;
    double qm[3];
    int nr[3];
#pragma unroll
    for (int rr = 0; rr < 3; rr++) {
      const int i = 8 * (r0 + rr) + g;
      qm[rr] = (rr < nrow && i < k) ? H.qmin[i] : 0.0;
      nr[rr] = (rr < nrow && i < k) ? H.near[i] : -2;
    }
    double acc[30];
#pragma unroll
    for (int i = 0; i < 30; i++) acc[i] = 0.0;
    const int src0 = (g << 2) | (t4 >> 1), src1 = (g << 2) | (2 + (t4 >> 1));
    for (int c = warp; c < nct; c += NWARP) {
      double fb[2][5];
#pragma unroll
      for (int ks = 0; ks < 2; ks++) {
        const int j = 8 * c + 4 * ks + t4;
        const bool valid = j < m;
        const int b = valid ? zv.base(j) : 0;
#pragma unroll
        for (int ct = 0; ct < 5; ct++) fb[ks][ct] = valid ? zval(zv.ptr, b, offz[ct], cstz[ct]) : 0.0;
      }
      const int col = 8 * c + 2 * t4;
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
        if (rr >= nrow) break;
        const double* qp = gQ + ((size_t)(c * 5 + r0 + rr) * 32 + lane) * 2;
        const double q0 = qp[0], q1 = qp[1];
        double w0 = 0.0, w1 = 0.0;
        if (nr[rr] >= 0) {
          if (col < m && col != nr[rr]) w0 = exp((qm[rr] - q0) * sb);
          if (col + 1 < m && col + 1 != nr[rr]) w1 = exp((qm[rr] - q1) * sb);
        }
        // C-fragment layout (row g, cols 2t4..2t4+1) -> A fragments of the two k-steps
        const double x0 = __shfl_sync(FULL, w0, src0), x1 = __shfl_sync(FULL, w1, src0);
        const double z0 = __shfl_sync(FULL, w0, src1), z1 = __shfl_sync(FULL, w1, src1);
        const double a0 = (t4 & 1) ? x1 : x0, a1 = (t4 & 1) ? z1 : z0;
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          dmma(acc[2 * (rr * 5 + ct)], acc[2 * (rr * 5 + ct) + 1], a0, fb[0][ct]);
          dmma(acc[2 * (rr * 5 + ct)], acc[2 * (rr * 5 + ct) + 1], a1, fb[1][ct]);
        }
      }
    }
    tree_reduce<30>(acc, H.R1);
    if (warp == 0) {
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
        if (rr >= nrow) break;
#pragma unroll
        for (int ct = 0; ct < 5; ct++) {
          Zp[(8 * (r0 + rr) + g) * 40 + 8 * ct + 2 * t4] = acc[2 * (rr * 5 + ct)];
          Zp[(8 * (r0 + rr) + g) * 40 + 8 * ct + 2 * t4 + 1] = acc[2 * (rr * 5 + ct) + 1];
        }
      }
    }
  }
  __syncthreads();

  // ---------------------------------- alpha (estimators.py:237-245)
  {
    double* u = H.R1;  // [KMAX][32]
    for (int o = tid; o < k * 32; o += NT) {
      const int i = o >> 5, t = o & 31;
      const int b = zv.base(H.near[i]);
      const double S = Zp[i * 40 + 36];
      double s = 0.0;
      for (int q = 0; q <= t && q < n; q++) {
        const double r = zv.ptr[b + H.coff[q]] - Zp[i * 40 + q] / S;  // y_i - y~_i
        s = fma(H.Linv[t * LS + q], r, s);
      }
      u[i * 32 + t] = t < n ? s : 0.0;
    }
    __syncthreads();
    if (tid < 4 * k) {
      const int q = tid / k, i = tid % k;
      double c = 0.0;
      for (int t = 0; t < n; t++) c = fma(H.Bm[q * 32 + t], u[i * 32 + t], c);
      const int b = zv.base(H.near[i]);
      const double S = Zp[i * 40 + 36];
      H.cmat[q * k + i] = c;
      H.rmat[q * k + i] = zval(zv.ptr, b, H.coff[32 + q], 0.0) - Zp[i * 40 + 32 + q] / S;
    }
    __syncthreads();
    if (warp == 0) {
      // u0 = Linv (y0 - y~0); correction = Bm u0
      double s = 0.0;
      for (int q = 0; q <= lane && q < n; q++) s = fma(H.Linv[lane * LS + q], y0[q] - H.yt[q], s);
      const double u0 = lane < n ? s : 0.0;
      double corr[4];
#pragma unroll
      for (int q = 0; q < 4; q++) corr[q] = warp_sum(H.Bm[q * 32 + lane] * u0);
      if (lane == 0) {
        const int kk = 4 * k;
        const double den = pairwise_sum_n(kk, [&](int i) { return __dmul_rn(H.cmat[i], H.cmat[i]); });
        const double num = pairwise_sum_n(kk, [&](int i) { return __dmul_rn(H.rmat[i], H.cmat[i]); });
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
}

}  // namespace bm
