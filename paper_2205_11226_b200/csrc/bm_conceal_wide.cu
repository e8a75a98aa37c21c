// bm_conceal_wide.cu — the concealment kernels compiled a second time with
// 512-thread CTAs (namespace bmw, one cell per SM) for narrow dependency DAGs
// (bm_kernels.cuh, k_conceal); bm_conceal.cu launches both builds and each
// runs only on the DAG shapes it serves.
#define BM_NT 512
#define BM_NS bmw
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
