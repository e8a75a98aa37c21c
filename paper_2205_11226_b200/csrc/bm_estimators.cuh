// bm_estimators.cuh — CTA-cooperative BRL / IDL / HQL estimators for one
// 2x2 patch (reference: blockmend/estimators.py).
//
//  * BRL  (estimators.py:96-102): FP64 mean in NumPy's pairwise order (bit-exact).
//  * IDL  (estimators.py:105-132): Nadaraya-Watson weights in FP32
//    (distances d2 and exp), FP64 accumulation of the weighted sums; the
//    FP64 underflow predicate raw_sum == 0 is evaluated exactly from the
//    largest exponent.
//  * HQL  (estimators.py:135-286): FP64 end to end (any
//    FP32 inside HQL flips beta near-ties) — covariance, Cholesky, Mahalanobis
//    quadforms, 21-point beta grid, leave-one-out alpha fit, correction.
//
// Candidate values are read through an accessor: TileAcc gathers them from
// the shared-memory support tile (the fused concealment kernel), DenseAcc
// from dense global arrays (bm_estimate_batch, the estimator-level API).
#pragma once
#include <cfloat>
#include "bm_common.cuh"

namespace BM_NS {

struct TileAcc {
  const double* tile;     // smem [TILE*TS]
  const uint16_t* cand;   // smem window-origin tile positions
  const int16_t* uoff;    // smem used offsets: n context then 4 patch cells
  const float* tile32;    // smem FP32 shadow of the tile (BM_IDL_FP32 experiment)
  __device__ __forceinline__ double y(int j, int t) const { return tile[cand[j] + uoff[t]]; }
  __device__ __forceinline__ float yf(int j, int t) const { return tile32[cand[j] + uoff[t]]; }
  __device__ __forceinline__ double x(int j, int q) const {
    return tile[cand[j] + (2 + (q >> 1)) * TS + 2 + (q & 1)];
  }
};

struct DenseAcc {
  const double* X;  // [m][4]   (global)
  const double* Y;  // [m][32]  (global)
  __device__ __forceinline__ double y(int j, int t) const { return Y[(size_t)j * 32 + t]; }
  __device__ __forceinline__ float yf(int j, int t) const { return (float)Y[(size_t)j * 32 + t]; }
  __device__ __forceinline__ double x(int j, int q) const { return X[(size_t)j * 4 + q]; }
};

// Shared scratch of the estimators (one patch at a time per CTA).
struct EstSmem {
  double y0[32];
  float y0f[32];
  int16_t uoff[36];
  int n;
  // results
  double vals[4];
  double beta, alpha, nu_raw;
  float gap;
  int layer, fallback, ok;
  // reductions
  double red[NWARP][8];
  double redmin[NWARP];
  float redf[NWARP];
  long long t_e[2];  // diagnostics
  alignas(16) double exptab[128];  // exp_w table (init_exptab)
};

__device__ __forceinline__ void init_exptab(EstSmem& S) {
  if (threadIdx.x < 128) S.exptab[threadIdx.x] = g_exp2_64[threadIdx.x];
}

// ----------------------------------------------------------------- helpers

__device__ __forceinline__ double cta_min(double v, EstSmem& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) S.redmin[w] = v;
  __syncthreads();
  double r = S.redmin[0];
#pragma unroll
  for (int i = 1; i < NWARP; i++) r = fmin(r, S.redmin[i]);
  return r;
}

__device__ __forceinline__ float cta_minf(float v, EstSmem& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_minf(v);
  __syncthreads();
  if (lane == 0) S.redf[w] = v;
  __syncthreads();
  float r = S.redf[0];
#pragma unroll
  for (int i = 1; i < NWARP; i++) r = fminf(r, S.redf[i]);
  return r;
}

// CTA-wide sums of N per-thread values, fixed order; every thread gets the totals.
template <int N>
__device__ __forceinline__ void cta_sum_n(double (&v)[N], EstSmem& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; i++) S.red[w][i] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; i++) {
    double a = S.red[0][i];
#pragma unroll
    for (int k = 1; k < NWARP; k++) a += S.red[k][i];
    v[i] = a;
  }
}

// ----------------------------------------------------------------------- BRL
// brl_estimate (estimators.py:96-102): float(y0.mean()) = pairwise sum / n.
__device__ __forceinline__ void brl_values(EstSmem& S) {
  if (threadIdx.x == 0) {
    const int n = S.n;
    double mean = pairwise_sum_n(n, [&](int i) { return S.y0[i]; }) / n;
    for (int q = 0; q < 4; q++) S.vals[q] = mean;
  }
}

// ----------------------------------------------------------------------- IDL
// idl_weights / idl_estimate (estimators.py:112-132) in FP64, mirroring the
// reference's arithmetic: d2 in NumPy's pairwise order, expo = -d2/(2 s2 N_y),
// w = exp(expo - max) / sum, values = w @ x.  (The FP32 Nadaraya-Watson
// distance/weight work is the nu gate's screening pass in gather(); FP32 in
// the *estimate* itself is amplified ~1e4x along the patch chain and breaks
// the +-1 LSB bar.)  The exponents go through shared memory
// (exbuf, >= m doubles).  Called from one site per kernel (one inlined copy:
// instruction-cache footprint).
// Sets S.ok = 0 on WeightUnderflowError (raw_sum == 0); S.nu_raw = raw_sum.
#ifndef BM_IDL_FP32
#define BM_IDL_FP32 0
#endif
#if BM_IDL_FP32
// EXPERIMENT (tools/fp32_idl.sh; not the product build): the
// north_star's FP32 Nadaraya-Watson weighting inside the IDL estimate -
// FP32 distances (fmaf over the FP32 tile shadow), FP32 exponents and expf
// weights, FP64 accumulation of the weighted sums and normalisation, and the
// reference's FP64 underflow predicate (raw_sum == 0) evaluated from the
// largest exponent in the log domain.
template <class Acc>
__device__ __forceinline__ void idl_estimate_dev(const Acc& acc, int m, double sigma2, EstSmem& S, double* exbuf,
                                                 bool want_raw, bool final_sync = true) {
  const int n = S.n, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float invc = (float)(1.0 / (2.0 * sigma2 * n));
  float* ef = reinterpret_cast<float*>(exbuf);
  float emax = -INFINITY;
#pragma unroll 1
  for (int j = threadIdx.x; j < m; j += NT) {
    float d2a = 0.f, d2b = 0.f;
    int t = 0;
#pragma unroll 1
    for (; t + 2 <= n; t += 2) {
      const float da = acc.yf(j, t) - S.y0f[t], db = acc.yf(j, t + 1) - S.y0f[t + 1];
      d2a = fmaf(da, da, d2a);
      d2b = fmaf(db, db, d2b);
    }
    if (t < n) {
      const float da = acc.yf(j, t) - S.y0f[t];
      d2a = fmaf(da, da, d2a);
    }
    const float e = -(d2a + d2b) * invc;
    ef[j] = e;
    emax = fmaxf(emax, e);
  }
  emax = warp_minf(-emax) * -1.f;  // warp max
  if (lane == 0) S.redf[warp] = emax;
  __syncthreads();
  emax = S.redf[0];
#pragma unroll
  for (int w = 1; w < NWARP; w++) emax = fmaxf(emax, S.redf[w]);
  double v5[5] = {0, 0, 0, 0, 0};
#pragma unroll 1
  for (int j = threadIdx.x; j < m; j += NT) {
    const double sh = (double)__expf(ef[j] - emax);
    v5[0] += sh;
#pragma unroll
    for (int q = 0; q < 4; q++) v5[1 + q] = fma(sh, acc.x(j, q), v5[1 + q]);
  }
#pragma unroll
  for (int q = 0; q < 5; q++) v5[q] = warp_sum(v5[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 5; q++) S.red[warp][q] = v5[q];
  }
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    if (lane < 5) {
      t = S.red[0][lane];
#pragma unroll
      for (int w = 1; w < NWARP; w++) t += S.red[w][lane];
    }
    const double t0 = __shfl_sync(FULL, t, 0);
    if (lane >= 1 && lane < 5) S.vals[lane - 1] = t * (1.0 / t0);
    if (lane == 0) {
      if (want_raw) {
        const double e0 = exp((double)emax);  // log-domain FP64 underflow predicate
        S.nu_raw = e0 * t0;
        S.ok = e0 != 0.0;
      } else {
        S.ok = 1;
      }
    }
  }
  if (final_sync) __syncthreads();
}
#else
template <class Acc>
__device__ __forceinline__ void idl_estimate_dev(const Acc& acc, int m, double sigma2, EstSmem& S, double* exbuf,
                                                 bool want_raw, bool final_sync = true) {
  const int n = S.n, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double c = 2.0 * sigma2 * n;
  double emax = -INFINITY;
#pragma unroll 1
  for (int j = threadIdx.x; j < m; j += NT) {
    // d2 = ((y - y0) ** 2).sum(axis=1) in NumPy's pairwise order, rolled:
    // eight strided accumulators below n8, their tree, then the tail in order
    const int n8 = n - (n % 8);
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; q++) r[q] = 0.0;
#pragma unroll 1
    for (int t = 0; t < n8; t += 8) {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const double d = acc.y(j, t + q) - S.y0[t + q];
        r[q] = __dadd_rn(r[q], __dmul_rn(d, d));
      }
    }
    double d2 = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                          __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll 1
    for (int t = n8; t < n; t++) {
      const double d = acc.y(j, t) - S.y0[t];
      d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    const double e = -d2 / c;  // expo = -d2 / (2 sigma2 N_y)
    exbuf[j] = e;
    emax = fmax(emax, e);
  }
  // expo.max(): one barrier
  emax = warp_max(emax);
  if (lane == 0) S.redmin[warp] = emax;
  __syncthreads();
  if (threadIdx.x == 0) S.t_e[0] = clock64();
  emax = S.redmin[0];
#pragma unroll
  for (int w = 1; w < NWARP; w++) emax = fmax(emax, S.redmin[w]);
  // shifted weights and the unnormalised sums in one pass, one barrier
  double v5[5] = {0, 0, 0, 0, 0};
#pragma unroll 1
  for (int j = threadIdx.x; j < m; j += NT) {
    const double sh = exp_w(exbuf[j] - emax, S.exptab);
    v5[0] += sh;
#pragma unroll
    for (int q = 0; q < 4; q++) v5[1 + q] = fma(sh, acc.x(j, q), v5[1 + q]);
  }
#pragma unroll
  for (int q = 0; q < 5; q++) v5[q] = warp_sum(v5[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 5; q++) S.red[warp][q] = v5[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) S.t_e[1] = clock64();
  if (warp == 0) {
    // lane q < 5 totals sum q over the warps (fixed order)
    double t = 0.0;
    if (lane < 5) {
      t = S.red[0][lane];
#pragma unroll
      for (int w = 1; w < NWARP; w++) t += S.red[w][lane];
    }
    const double t0 = __shfl_sync(FULL, t, 0);
    if (lane >= 1 && lane < 5) S.vals[lane - 1] = t * (1.0 / t0);  // w @ x with w = shifted / sum
    if (lane == 0) {
      if (want_raw) {  // forced / fallback IDL: raw_sum and the underflow test
        const double e0 = exp(emax);  // raw_sum == 0.0 iff the largest term underflows
        S.nu_raw = e0 * t0;
        S.ok = e0 != 0.0;
      } else {
        S.ok = 1;  // gated IDL: nu >= T_nu > 0, no underflow
      }
    }
  }
  if (final_sync) __syncthreads();
}
#endif  // BM_IDL_FP32

}  // namespace BM_NS
