// Microbenchmark: FP64 DMMA (mma.sync f64) throughput vs independent chains
// per warp, m8n8k4 vs m16n8k8, and overlap with DFMA / FP64 exp on one B200.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double a2, double a3, double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}
template <int CH>
__global__ void k_chains(double* out, double a, double b) {
  double c[CH][2];
  for (int i = 0; i < CH; i++) { c[i][0] = threadIdx.x + i; c[i][1] = i * 0.5; }
  const double av = a + threadIdx.x * 1e-9;
  for (int it = 0; it < ITERS / CH; it++)
#pragma unroll
    for (int i = 0; i < CH; i++) dmma(c[i][0], c[i][1], av + i, b);
  double s = 0;
  for (int i = 0; i < CH; i++) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_chains16(double* out, double a, double b) {
  double c[CH][4];
  for (int i = 0; i < CH; i++) for (int j = 0; j < 4; j++) c[i][j] = threadIdx.x + i + j;
  const double av = a + threadIdx.x * 1e-9;
  for (int it = 0; it < ITERS / (4 * CH); it++)
#pragma unroll
    for (int i = 0; i < CH; i++) dmma16(c[i], av + i, av, b + i, b, av, b);
  double s = 0;
  for (int i = 0; i < CH; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// even warps: 8-chain DMMA; odd warps: DFMA (mode 1) or exp (mode 2) or idle (mode 0)
__global__ void k_mix(double* out, double a, double b, int mode) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (!(warp & 1)) {
    double c[8][2];
    for (int i = 0; i < 8; i++) { c[i][0] = threadIdx.x + i; c[i][1] = i; }
    const double av = a + threadIdx.x * 1e-9;
    for (int it = 0; it < ITERS / 8; it++)
#pragma unroll
      for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], av + i, b);
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  } else if (mode == 1) {
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001 + i;
    for (int it = 0; it < ITERS / 2; it++)
#pragma unroll
      for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
    for (int i = 0; i < 8; i++) s += x[i];
  } else if (mode == 2) {
    double x = threadIdx.x * -1e-3;
    for (int it = 0; it < ITERS / 32; it++) { s += exp(x); x -= a * 1e-3; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* buf; cudaMalloc(&buf, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto run = [&](const char* name, auto kern, int blocks, int thr, double flops) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      kern<<<blocks, thr>>>((double*)buf, 0.999, 0.001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("%-40s %8.3f ms  %.1f TFLOP/s\n", name, ms, flops / (ms * 1e-3) / 1e12);
  };
  for (int wps : {8, 16, 32, 64}) {  // warps per SM
    const int blocks = sms * (wps / 8), thr = 256;
    const double warps = (double)blocks * thr / 32;
    char nm[64];
    snprintf(nm, 64, "m8n8k4  1 chain   %2d warps/SM", wps); run(nm, k_chains<1>, blocks, thr, warps * ITERS * 512.0);
    snprintf(nm, 64, "m8n8k4  4 chains  %2d warps/SM", wps); run(nm, k_chains<4>, blocks, thr, warps * ITERS * 512.0);
    snprintf(nm, 64, "m8n8k4  8 chains  %2d warps/SM", wps); run(nm, k_chains<8>, blocks, thr, warps * ITERS * 512.0);
    snprintf(nm, 64, "m8n8k4 16 chains  %2d warps/SM", wps); run(nm, k_chains<16>, blocks, thr, warps * ITERS * 512.0);
    snprintf(nm, 64, "m16n8k8 2 chains  %2d warps/SM", wps); run(nm, k_chains16<2>, blocks, thr, warps * ITERS * 512.0);
    snprintf(nm, 64, "m16n8k8 4 chains  %2d warps/SM", wps); run(nm, k_chains16<4>, blocks, thr, warps * ITERS * 512.0);
  }
  const int blocks = sms * 2, thr = 512;
  const double warps = (double)blocks * thr / 32;
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      k_mix<<<blocks, thr>>>((double*)buf, 0.999, 0.001, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const char* nm[] = {"mix: DMMA warps + idle warps", "mix: DMMA warps + DFMA warps", "mix: DMMA warps + exp warps"};
    printf("%-40s %8.3f ms  DMMA part %.1f TFLOP/s\n", nm[mode], ms, warps / 2 * ITERS * 512.0 / (ms * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
