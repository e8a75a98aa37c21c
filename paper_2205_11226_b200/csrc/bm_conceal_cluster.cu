// bm_conceal_cluster.cu — the concealment kernel compiled for thread-block
// clusters (namespace bmc): CS = 2 CTAs of 512 threads, one per SM, conceal
// one cell together.  Every CTA of the cluster runs the cell's control flow
// (pick, gate, IDL/BRL, the HQL serial sections) on identical data; the
// candidate loops of the HQL pipeline (means, covariance, nearest set,
// quadforms, beta grid, leave-one-out sums) are split over the cluster's
// warps and their partial results combined over distributed shared memory in
// rank order (bm_hql.cuh cluster_sum_w0), so the CTAs stay bit-identical.
// This shortens a cell's latency: the lever for dependency DAGs too narrow to
// fill the GPU (the critical path of slice chains, single images).
#define BM_NT 512
#define BM_CS 2
#define BM_NS bmc
#define BM_CONCEAL_ONLY 1
#include "bm_kernels.cuh"

namespace bm_cluster {

size_t cell_smem_bytes() { return sizeof(bmc::CellSmem); }
int cluster_size() { return bmc::CS; }

cudaError_t set_smem(size_t smem) {
  return cudaFuncSetAttribute(bmc::k_conceal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static cudaLaunchConfig_t config(int clusters, size_t smem, cudaStream_t stream, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * bmc::CS, 1, 1);
  cfg.blockDim = dim3(bmc::NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = bmc::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// clusters that can be resident at once (persistent grid)
int max_clusters(size_t smem) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = config(1, smem, nullptr, attr);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)bmc::k_conceal, &cfg) != cudaSuccess || n < 1) n = 1;
  return n;
}

// P: the bm::KParams of the launch (identical layout in every build).
cudaError_t launch(const void* P, int clusters, size_t smem, cudaStream_t stream) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = config(clusters, smem, stream, attr);
  return cudaLaunchKernelEx(&cfg, bmc::k_conceal, *reinterpret_cast<const bmc::KParams*>(P));
}

}  // namespace bm_cluster

namespace bm_cluster {
// the build's diagnostic phase counters (-DBM_DIAG=1 builds), added into out48
cudaError_t add_phase_cycles(unsigned long long* out48, int reset) {
  unsigned long long v[48];
  cudaError_t e = cudaMemcpyFromSymbol(v, bmc::g_phase_cycles, 48 * 8);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < 48; i++) out48[i] += v[i];
  if (reset) {
    unsigned long long z[48] = {0};
    e = cudaMemcpyToSymbol(bmc::g_phase_cycles, z, 48 * 8);
  }
  return e;
}
}  // namespace bm_cluster
