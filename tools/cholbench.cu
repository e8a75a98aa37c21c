// microbenchmark: 32x32 Cholesky on one warp from shared memory (variants)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chol(double* out, int variant, long long* cyc) {
  __shared__ double A[32 * 33], L[32 * 33];
  const int lane = threadIdx.x;
  for (int i = 0; i < 32; i++) A[i * 33 + lane] = (i == lane ? 100.0 : 0.0) + 1.0 / (1 + i + lane);
  __syncwarp();
  long long t0 = clock64();
  const int n = 32;
  for (int j = 0; j < n; j++) {
    double t = 0.0;
    if (lane >= j) {
      t = A[lane * 33 + j];
      for (int k = 0; k < j; k++) t = fma(-L[lane * 33 + k], L[j * 33 + k], t);
    }
    const double sd = __shfl_sync(0xffffffff, t, j);
    double d, rs;
    if (variant == 0) { rs = rsqrt(sd); d = sd * rs; }
    else if (variant == 1) { d = sqrt(sd); rs = 1.0 / d; }
    else { d = sqrt(sd); rs = __drcp_rn(d); }
    if (lane == j) L[j * 33 + j] = d;
    if (lane > j) L[lane * 33 + j] = t * rs;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[variant] = t1 - t0; }
  out[lane] = L[lane * 33 + lane];
}
__global__ void ops(long long* cyc, double x) {
  long long t0 = clock64();
  double s = x;
  for (int i = 0; i < 100; i++) s = rsqrt(s + 1.0);
  long long t1 = clock64();
  double u = x;
  for (int i = 0; i < 100; i++) u = sqrt(u + 1.0);
  long long t2 = clock64();
  double v = x;
  for (int i = 0; i < 100; i++) v = 1.0 / (v + 1.0);
  long long t3 = clock64();
  double w = x;
  for (int i = 0; i < 100; i++) w = exp(-w);
  long long t4 = clock64();
  double z = x;
  for (int i = 0; i < 100; i++) z = __shfl_sync(0xffffffff, z, (threadIdx.x + 1) & 31) + 1.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 100; cyc[3] = (t4 - t3) / 100; cyc[4] = (t5 - t4) / 100; }
  if (s + u + v + w + z == 12345.0) cyc[5] = 1;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMallocManaged(&cyc, 64);
  for (int v = 0; v < 3; v++) { chol<<<1, 32>>>(out, v, cyc); cudaDeviceSynchronize(); chol<<<1, 32>>>(out, v, cyc); cudaDeviceSynchronize(); }
  printf("chol cycles: rsqrt %lld  sqrt+div %lld  sqrt+drcp %lld\n", cyc[0], cyc[1], cyc[2]);
  ops<<<1, 32>>>(cyc, 0.5); cudaDeviceSynchronize(); ops<<<1, 32>>>(cyc, 0.5); cudaDeviceSynchronize();
  printf("latency per op: rsqrt %lld sqrt %lld div %lld exp %lld shfl+add %lld\n", cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
  return 0;
}
