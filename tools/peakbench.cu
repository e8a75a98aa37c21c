// Microbenchmark: FP32 FFMA, FP64 DFMA, FP64 DMMA (mma.sync m8n8k4 f64) and FP64 exp throughput on one B200.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x[8]; for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dmma(double* out, double a, double b) {
  double c[4][2]; for (int i = 0; i < 4; i++) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0; for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dexp(double* out, double a) {
  double x = threadIdx.x * -1e-3, s = 0;
  for (int it = 0; it < ITERS / 16; it++) { s += exp(x); x -= a; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fexp(float* out, float a) {
  float x = threadIdx.x * -1e-3f, s = 0;
  for (int it = 0; it < ITERS / 16; it++) { s += __expf(x); x -= a; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  void* buf; cudaMalloc(&buf, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, thr = 256; float ms;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0); k_ffma<<<blocks, thr>>>((float*)buf, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA  %.1f TFLOP/s\n", 2.0 * 8 * ITERS * blocks * thr / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); k_dfma<<<blocks, thr>>>((double*)buf, 0.999, 0.001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA  %.1f TFLOP/s\n", 2.0 * 8 * ITERS * blocks * thr / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); k_dmma<<<blocks, thr>>>((double*)buf, 0.999, 0.001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA  %.1f TFLOP/s\n", 2.0 * 256 * 4 * (ITERS / 4) * (blocks * thr / 32) / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); k_dexp<<<blocks, thr>>>((double*)buf, 0.01); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("exp(f64) %.1f Gexp/s\n", 1.0 * (ITERS / 16) * blocks * thr / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0); k_fexp<<<blocks, thr>>>((float*)buf, 0.01f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("__expf %.1f Gexp/s\n", 1.0 * (ITERS / 16) * blocks * thr / (ms * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
