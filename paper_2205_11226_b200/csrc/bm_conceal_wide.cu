// bm_conceal_wide.cu — the concealment kernels compiled a second time with
// 512-thread CTAs (namespace bmw, one cell per SM) for narrow dependency DAGs
// (bm_kernels.cuh, k_conceal); bm_conceal.cu launches both builds and each
// runs only on the DAG shapes it serves.
#define BM_NT 512
#define BM_NS bmw
#define BM_CONCEAL_ONLY 1
#include "bm_kernels.cuh"

namespace bm_wide {

size_t cell_smem_bytes() { return sizeof(bmw::CellSmem); }
int threads() { return bmw::NT; }

cudaError_t set_smem(size_t smem) {
  return cudaFuncSetAttribute(bmw::k_conceal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// P: the bm::KParams of the launch (identical layout: KParams does not depend
// on the CTA width).
cudaError_t launch(const void* P, int grid, size_t smem, cudaStream_t stream) {
  bmw::k_conceal<<<grid, bmw::NT, smem, stream>>>(*reinterpret_cast<const bmw::KParams*>(P));
  return cudaGetLastError();
}

}  // namespace bm_wide

namespace bm_wide {
// the build's diagnostic phase counters (-DBM_DIAG=1 builds), added into out48
cudaError_t add_phase_cycles(unsigned long long* out48, int reset) {
  unsigned long long v[48];
  cudaError_t e = cudaMemcpyFromSymbol(v, bmw::g_phase_cycles, 48 * 8);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < 48; i++) out48[i] += v[i];
  if (reset) {
    unsigned long long z[48] = {0};
    e = cudaMemcpyToSymbol(bmw::g_phase_cycles, z, 48 * 8);
  }
  return e;
}
}  // namespace bm_wide
