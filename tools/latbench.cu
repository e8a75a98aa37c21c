// Dependent-chain latencies on one warp (one CTA of 32 threads per SM):
// DMMA m8n8k4 f64, DFMA, DADD, DMUL, FFMA, LDS.64, SHFL, exp(), clock overhead.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(long long* out, double a, double b, float fa) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i * 7 + 3) % 1024;
  __syncwarp();
  long long t0, t1;
  double c0 = threadIdx.x, c1 = 1.0;
  // DMMA chain
  t0 = clock64();
  for (int i = 0; i < N; i++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  t1 = clock64();
  out[0] = (t1 - t0);
  double x = c0 + c1;
  t0 = clock64();
  for (int i = 0; i < N; i++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(a), "d"(b));
  t1 = clock64();
  out[1] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; i++) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
  t1 = clock64();
  out[2] = (t1 - t0);
  float y = fa + x;
  t0 = clock64();
  for (int i = 0; i < N; i++) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(y) : "f"(fa));
  t1 = clock64();
  out[3] = (t1 - t0);
  // LDS chain: index from loaded value
  int idx = threadIdx.x + (int)y * 0;
  t0 = clock64();
  for (int i = 0; i < N; i++) idx = (int)sm[idx];
  t1 = clock64();
  out[4] = (t1 - t0);
  double s = idx;
  t0 = clock64();
  for (int i = 0; i < N; i++) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
  t1 = clock64();
  out[5] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N / 8; i++) s = exp(-s * 1e-3);
  t1 = clock64();
  out[6] = (t1 - t0) * 8;
  // 4 independent DMMA chains
  double d[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  t0 = clock64();
  for (int i = 0; i < N / 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[2*j]), "+d"(d[2*j+1]) : "d"(a), "d"(b));
  t1 = clock64();
  out[7] = (t1 - t0);
  out[8] = (long long)(x + y + s + c0 + d[0] + d[3] + d[7]);
}
int main() {
  long long* d; cudaMalloc(&d, 16 * 8);
  long long h[16];
  for (int rep = 0; rep < 2; rep++) {
    k<<<1, 32>>>(d, 0.999, 0.001, 0.999f);
    cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  }
  const char* nm[] = {"DMMA m8n8k4 f64", "DFMA", "DADD", "FFMA", "LDS.64+cvt", "SHFL f64 + DADD", "exp() f64", "DMMA x4 indep (per MMA)"};
  for (int i = 0; i < 8; i++) printf("%-26s %6.1f cycles\n", nm[i], (double)h[i] / N);
  return 0;
}
