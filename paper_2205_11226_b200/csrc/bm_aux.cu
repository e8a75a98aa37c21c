// bm_aux.cu — the callers either side of the concealment path (SURVEY.md
// §8(f) rows 2-3), on the device:
//
//  * batched quality metrics of the benchmark harness (metrics.py:50-116):
//    PSNR over all pixels, PSNR over a selection (the originally lost set)
//    and mean SSIM (11x11 Gaussian window, sigma 1.5, windows fully inside).
//    All FP64 like the reference; sums are per-tile partials reduced in a
//    fixed order, so results are deterministic run to run.  HBM-bound
//    (1 B/px for u8 frames): one pass over both frames per metric.
//  * deterministic loss-pattern generation (loss.py:24-77): dispersed
//    (odd/odd blocks), exact-count random (SplitMix64 + Fisher-Yates, the
//    reference's draw sequence bit for bit) and macroblock-row slices (the
//    BASELINE cfg3 pattern, synth.slice_mask).  One CTA per frame; the draws
//    are counter-based (state_i = seed + i*GAMMA) and computed in parallel,
//    the swaps stay sequential on one thread in shared memory (global scratch
//    when the block count exceeds shared memory), then the CTA paints the
//    states.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/blockmend_b200.h"
#include "bm_host.h"

namespace bm_aux {

constexpr int NT = 256;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double px_at(const void* p, int dtype, size_t i) {
  return dtype == BM_PIX_F64 ? ((const double*)p)[i] : (double)((const uint8_t*)p)[i];
}

// fixed-order CTA sum (warp butterflies, then warp 0 over the warp partials)
__device__ __forceinline__ double cta_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; w++) s += red[w];
  return s;  // valid on thread 0
}

// ---------------------------------------------------------------- PSNR
// part[f * nchunk + c] = sum over chunk c of frame f of sel * (a - b)^2,
// cnt likewise (selected pixel count).  Chunks are fixed-size ranges.
__global__ void k_sqdiff(const void* a, const void* b, int dtype, const uint8_t* sel, int64_t npx, int nchunk,
                         double* part, double* cnt) {
  __shared__ double red[NT / 32], red2[NT / 32];
  const int f = blockIdx.y, c = blockIdx.x;
  const int64_t per = (npx + nchunk - 1) / nchunk;
  const int64_t lo = (int64_t)c * per, hi = lo + per < npx ? lo + per : npx;
  const size_t base = (size_t)f * npx;
  double s = 0.0, n = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += NT) {
    if (sel && !sel[base + i]) continue;
    const double d = px_at(a, dtype, base + i) - px_at(b, dtype, base + i);
    s = fma(d, d, s);
    n += 1.0;
  }
  const double ts = cta_sum(s, red);
  const double tn = cta_sum(n, red2);
  if (threadIdx.x == 0) {
    part[(size_t)f * nchunk + c] = ts;
    cnt[(size_t)f * nchunk + c] = tn;
  }
}

__global__ void k_reduce_frames(const double* part, const double* cnt, int nchunk, int B, double* out_sum,
                                double* out_cnt) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B) return;
  double s = 0.0, n = 0.0;
  for (int c = 0; c < nchunk; c++) {
    s += part[(size_t)f * nchunk + c];
    if (cnt) n += cnt[(size_t)f * nchunk + c];
  }
  out_sum[f] = s;
  if (out_cnt) out_cnt[f] = n;
}

// v[i] / d: the mean as NumPy forms it (sum / count, not sum * (1 / count))
__global__ void k_div(double* v, int n, double d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] /= d;
}

// ---------------------------------------------------------------- SSIM
constexpr int SW = 11, HALF = 5, TO = 32, TI = TO + SW - 1;  // output tile 32x32, input tile 42x42

struct SsimSmem {
  double a[TI][TI + 1], b[TI][TI + 1];
  double v[5][TO][TI + 1];  // vertical pass (metrics.py:_windowed_mean: axis 0 first): 5 moments
};

__constant__ double c_gauss[SW];

// one CTA per 32x32 tile of the valid (fully inside) SSIM map of one frame
__global__ void k_ssim_tiles(const void* A, const void* Bp, int dtype, int H, int W, int tiles_x, double* part) {
  extern __shared__ __align__(16) unsigned char smem[];
  SsimSmem& S = *reinterpret_cast<SsimSmem*>(smem);
  __shared__ double red[NT / 32];
  const int f = blockIdx.y;
  const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
  const int oy0 = ty * TO, ox0 = tx * TO;  // output coords in the valid map (image coords + HALF)
  const int vh = H - 2 * HALF, vw = W - 2 * HALF;
  const size_t base = (size_t)f * H * W;
  for (int i = threadIdx.x; i < TI * TI; i += NT) {
    const int r = i / TI, c = i % TI;
    const int y = oy0 + r, x = ox0 + c;  // image coords of the window's top-left + (r, c)
    double va = 0.0, vb = 0.0;
    if (y < H && x < W) {
      va = px_at(A, dtype, base + (size_t)y * W + x);
      vb = px_at(Bp, dtype, base + (size_t)y * W + x);
    }
    S.a[r][c] = va;
    S.b[r][c] = vb;
  }
  __syncthreads();
  // vertical 11-tap correlation (axis 0) of a, b, a*a, b*b, a*b for output rows, all 42 columns
  for (int i = threadIdx.x; i < TO * TI; i += NT) {
    const int r = i / TI, c = i % TI;
    double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
    for (int k = 0; k < SW; k++) {
      const double w = c_gauss[k], x = S.a[r + k][c], y = S.b[r + k][c];
      m0 = fma(w, x, m0);
      m1 = fma(w, y, m1);
      m2 = fma(w, x * x, m2);
      m3 = fma(w, y * y, m3);
      m4 = fma(w, x * y, m4);
    }
    S.v[0][r][c] = m0;
    S.v[1][r][c] = m1;
    S.v[2][r][c] = m2;
    S.v[3][r][c] = m3;
    S.v[4][r][c] = m4;
  }
  __syncthreads();
  const double c1 = (0.01 * 255.0) * (0.01 * 255.0), c2 = (0.03 * 255.0) * (0.03 * 255.0);
  double acc = 0.0;
  for (int i = threadIdx.x; i < TO * TO; i += NT) {
    const int r = i / TO, c = i % TO;
    if (oy0 + r >= vh || ox0 + c >= vw) continue;
    double m[5];
#pragma unroll
    for (int q = 0; q < 5; q++) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < SW; k++) s = fma(c_gauss[k], S.v[q][r][c + k], s);
      m[q] = s;
    }
    const double va = m[2] - m[0] * m[0], vb = m[3] - m[1] * m[1], cov = m[4] - m[0] * m[1];
    acc += ((2.0 * m[0] * m[1] + c1) * (2.0 * cov + c2)) / ((m[0] * m[0] + m[1] * m[1] + c1) * (va + vb + c2));
  }
  const double t = cta_sum(acc, red);
  if (threadIdx.x == 0) part[(size_t)f * gridDim.x + blockIdx.x] = t;
}

// ---------------------------------------------------------------- masks
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull, MUL1 = 0xBF58476D1CE4E5B9ull, MUL2 = 0x94D049BB133111EBull;

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {  // output i (1-based)
  uint64_t z = seed + i * GAMMA;
  z = (z ^ (z >> 30)) * MUL1;
  z = (z ^ (z >> 27)) * MUL2;
  return z ^ (z >> 31);
}

// lost-block flags [B][rows*cols] (u8), then painted into states
// kind: BM_MASK_DISPERSED, BM_MASK_RANDOM (count blocks), BM_MASK_SLICE (count MB rows)
__global__ void k_mask_blocks(int kind, int rows, int cols, int count, const uint64_t* seeds, uint32_t* scratch,
                              uint8_t* lost) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.x;
  const int total = kind == BM_MASK_SLICE ? rows : rows * cols;
  uint8_t* lf = lost + (size_t)f * rows * cols;
  for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) lf[i] = 0;
  __syncthreads();
  if (kind == BM_MASK_DISPERSED) {
    for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) {
      const int r = i / cols, c = i % cols;
      lf[i] = (r & 1) && (c & 1);
    }
    return;
  }
  // Fisher-Yates over [0, total): order[i] <-> order[draw_t % (i + 1)], t = total-1-i
  const bool in_smem = (size_t)total * 4 <= 96 * 1024;
  uint32_t* order = in_smem ? reinterpret_cast<uint32_t*>(smem) : scratch + (size_t)f * total;
  for (int i = threadIdx.x; i < total; i += blockDim.x) order[i] = (uint32_t)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t seed = seeds[f];
    uint64_t t = 1;
    for (int i = total - 1; i > 0; i--, t++) {
      const int j = (int)(splitmix_at(seed, t) % (uint64_t)(i + 1));
      const uint32_t tmp = order[i];
      order[i] = order[j];
      order[j] = tmp;
    }
  }
  __syncthreads();
  const int take = count < total ? count : total;
  if (kind == BM_MASK_RANDOM) {
    for (int i = threadIdx.x; i < take; i += blockDim.x) lf[order[i]] = 1;
  } else {  // slice: whole macroblock rows
    for (int i = threadIdx.x; i < take * cols; i += blockDim.x) lf[(size_t)order[i / cols] * cols + i % cols] = 1;
  }
}

__global__ void k_mask_paint(const uint8_t* lost, int B, int H, int W, int bs, int rows, int cols, uint8_t* states) {
  const size_t n = (size_t)B * H * W;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / ((size_t)H * W));
    const int rem = (int)(i % ((size_t)H * W));
    const int y = rem / W, x = rem % W;
    const int r = y / bs, c = x / bs;
    uint8_t s = 0;  // AVAILABLE
    if (r < rows && c < cols && lost[(size_t)f * rows * cols + r * cols + c]) s = 1;  // LOST
    states[i] = s;
  }
}

int sms() { return bm_host::sm_count(); }

int status(cudaError_t e) { return e == cudaSuccess ? BM_OK : BM_ERR_CUDA; }

}  // namespace bm_aux

using namespace bm_aux;

extern "C" {

int bm_sqdiff_batch(const void* ref, const void* test, int pixel_dtype, const uint8_t* select, int frames, int height,
                    int width, double* out_sum, double* out_count, void* stream_) {
  if (!ref || !test || !out_sum || !out_count || frames < 1 || height < 1 || width < 1) return BM_ERR_ARGS;
  if (pixel_dtype != BM_PIX_U8 && pixel_dtype != BM_PIX_F64) return BM_ERR_ARGS;
  cudaStream_t st = (cudaStream_t)stream_;
  const int64_t npx = (int64_t)height * width;
  int nchunk = (int)((npx + 65535) / 65536);
  if (nchunk > 4 * sms()) nchunk = 4 * sms();
  if (nchunk < 1) nchunk = 1;
  double* tmp = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&tmp, (size_t)frames * nchunk * 2 * sizeof(double), st)) != cudaSuccess)
    return status(e);
  k_sqdiff<<<dim3(nchunk, frames), NT, 0, st>>>(ref, test, pixel_dtype, select, npx, nchunk, tmp,
                                                 tmp + (size_t)frames * nchunk);
  k_reduce_frames<<<(frames + 127) / 128, 128, 0, st>>>(tmp, tmp + (size_t)frames * nchunk, nchunk, frames, out_sum,
                                                         out_count);
  e = cudaGetLastError();
  cudaFreeAsync(tmp, st);
  return status(e);
}

int bm_ssim_batch(const void* ref, const void* test, int pixel_dtype, int frames, int height, int width,
                  double* out_mean, void* stream_) {
  if (!ref || !test || !out_mean || frames < 1) return BM_ERR_ARGS;
  if (pixel_dtype != BM_PIX_U8 && pixel_dtype != BM_PIX_F64) return BM_ERR_ARGS;
  if (height < SW || width < SW) return BM_ERR_ARGS;  // metrics.py:96-97
  cudaStream_t st = (cudaStream_t)stream_;
  bm_host::DevState& D = bm_host::dev_state();
  if (!D.ssim_init.load()) {
    // normalised Gaussian taps (metrics.py:_gaussian_kernel_1d), computed in FP64 on the host
    double g[SW], s = 0.0;
    for (int i = 0; i < SW; i++) {
      const double x = i - HALF;
      g[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
      s += g[i];
    }
    for (int i = 0; i < SW; i++) g[i] /= s;
    if (cudaMemcpyToSymbol(c_gauss, g, sizeof(g)) != cudaSuccess) return BM_ERR_CUDA;
    if (cudaFuncSetAttribute(k_ssim_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimSmem)) !=
        cudaSuccess)
      return BM_ERR_CUDA;
    D.ssim_init = true;
  }
  const int vh = height - 2 * HALF, vw = width - 2 * HALF;
  const int tiles_y = (vh + TO - 1) / TO, tiles_x = (vw + TO - 1) / TO, ntile = tiles_x * tiles_y;
  double* part = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&part, (size_t)frames * ntile * sizeof(double), st)) != cudaSuccess)
    return status(e);
  k_ssim_tiles<<<dim3(ntile, frames), NT, sizeof(SsimSmem), st>>>(ref, test, pixel_dtype, height, width, tiles_x,
                                                                   part);
  // per-frame totals in tile order (fixed), then the mean over the valid map
  k_reduce_frames<<<(frames + 127) / 128, 128, 0, st>>>(part, nullptr, ntile, frames, out_mean, nullptr);
  k_div<<<(frames + 127) / 128, 128, 0, st>>>(out_mean, frames, (double)vh * (double)vw);
  e = cudaGetLastError();
  cudaFreeAsync(part, st);
  return status(e);
}

int bm_gen_masks(int kind, int frames, int height, int width, int block_size, int count, const uint64_t* seeds,
                 uint8_t* out_states, void* stream_) {
  if (frames < 1 || height < 1 || width < 1 || block_size < 1 || !out_states) return BM_ERR_ARGS;
  if (kind != BM_MASK_DISPERSED && kind != BM_MASK_RANDOM && kind != BM_MASK_SLICE) return BM_ERR_ARGS;
  if (kind != BM_MASK_DISPERSED && (!seeds || count < 0)) return BM_ERR_ARGS;
  cudaStream_t st = (cudaStream_t)stream_;
  const int rows = height / block_size, cols = width / block_size;
  const int total = kind == BM_MASK_SLICE ? rows : rows * cols;
  uint8_t* lost = nullptr;
  uint32_t* scratch = nullptr;
  cudaError_t e;
  const size_t nb = (size_t)frames * (rows * cols > 0 ? rows * cols : 1);
  if ((e = cudaMallocAsync((void**)&lost, nb, st)) != cudaSuccess) return status(e);
  const bool in_smem = (size_t)total * 4 <= 96 * 1024;
  if (!in_smem && (e = cudaMallocAsync((void**)&scratch, (size_t)frames * total * 4, st)) != cudaSuccess)
    return status(e);
  const int smem = in_smem ? total * 4 : 0;
  if (smem > 48 * 1024 && !bm_host::dev_state().mask_attr.load()) {
    if ((e = cudaFuncSetAttribute(k_mask_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)) !=
        cudaSuccess)
      return status(e);
    bm_host::dev_state().mask_attr = true;
  }
  if (rows > 0 && cols > 0)
    k_mask_blocks<<<frames, NT, smem, st>>>(kind, rows, cols, count, seeds, scratch, lost);
  else
    cudaMemsetAsync(lost, 0, nb, st);
  k_mask_paint<<<4 * sms(), NT, 0, st>>>(lost, frames, height, width, block_size, rows, cols, out_states);
  e = cudaGetLastError();
  cudaFreeAsync(lost, st);
  if (scratch) cudaFreeAsync(scratch, st);
  return status(e);
}

}  // extern "C"
