// bm_conceal.cu — the B200 concealment path: mask preprocessing (lost-cell
// slots, dependency levels, ready FIFOs), the persistent CTA-per-lost-cell
// concealment kernel, the dense estimator kernel, and the C ABI
// (include/blockmend_b200.h).
//
// Reference path: blockmend.conceal_image (profiles.py:263-323) ->
// _conceal_block (profiles.py:191-226) -> select_and_estimate /
// _forced_estimate (profiles.py:105-171) -> framework.py gather ->
// estimators.py.
//
// Execution model:
//  * one CTA conceals one lost 16x16 cell: it stages the cell's 48x48 support
//    area (FP64 values, FP32 shadow, states, LOST bitmaps) in shared memory and
//    runs the cell's whole <=64-patch reliability-ordered chain in place;
//  * dataflow scheduling: a cell becomes ready when its last earlier-raster
//    lost 8-neighbour finishes (per-cell dependency counters), which
//    reproduces the reference's serial raster order exactly
//    while independent cells run concurrently.  Ready cells wait in NB
//    priority FIFOs keyed by the cell's height in the dependency DAG (longest
//    chain of dependants first); a CTA pops the highest non-empty FIFO and
//    never blocks on a dependency;
//  * a finished cell publishes its 16x16 FP64 values to a per-cell buffer and
//    then decrements its dependants' counters; later cells read neighbours
//    from those buffers, so the working image never exists in HBM as a full
//    FP64 copy.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bm_host.h"
#include "bm_kernels.cuh"

namespace bm_wide {  // bm_conceal_wide.cu: the 512-thread build of k_conceal
size_t cell_smem_bytes();
int threads();
cudaError_t set_smem(size_t smem);
cudaError_t launch(const void* P, int grid, size_t smem, cudaStream_t stream);
cudaError_t add_phase_cycles(unsigned long long* out48, int reset);
}  // namespace bm_wide
namespace bm_cluster {  // bm_conceal_cluster.cu: the 2-CTA cluster build of k_conceal
size_t cell_smem_bytes();
int cluster_size();
cudaError_t set_smem(size_t smem);
int max_clusters(size_t smem);
cudaError_t launch(const void* P, int clusters, size_t smem, cudaStream_t stream);
cudaError_t add_phase_cycles(unsigned long long* out48, int reset);
}  // namespace bm_cluster
static_assert(sizeof(bm::KParams) > 0, "KParams layout is shared by all builds");


// =================================================================== C ABI
using namespace bm;

namespace {

// the narrowest DAGs: the 2-CTA cluster build (1) or the 512-thread build (0) by default
constexpr int NARROW_CLUSTER_DEFAULT = 1;

struct Layout {
  size_t ncell;
  size_t off_slotmap, off_slot_cell, off_level, off_level2, off_height, off_bucket, off_queue, off_indeg, off_nslots,
      off_sched, off_flags, off_excl, off_cellbuf, off_reccnt, off_counters, off_ringtab, off_postab, off_cub, cub_bytes,
      off_scratch,
      scratch_per_cta, total;
  int grid;
};

int sm_count() { return bm_host::sm_count(); }

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

// resident concealment CTAs per SM (persistent grid = SMs x this), per device
int cells_per_sm() {
  bm_host::DevState& D = bm_host::dev_state();
  if (!D.occ) {
    const int smem = (int)sizeof(CellSmem);
    if (!D.attr.load()) {
      if (cudaFuncSetAttribute(k_conceal, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess)
        D.attr = true;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_conceal, NT, smem) != cudaSuccess || occ < 1) occ = 1;
    // dev/diagnostic override (tools/): fewer resident cells per SM
    if (const char* e = getenv("BM_CELLS_PER_SM")) {
      const int v = atoi(e);
      if (v >= 1 && v < occ) occ = v;
    }
    D.occ = occ;
  }
  return D.occ;
}

bool params_ok(const bm_params* p) {
  return p && p->frames >= 1 && p->height >= 1 && p->width >= 1 && (p->pixel_dtype == BM_PIX_U8 || p->pixel_dtype == BM_PIX_F64) &&
         p->forced_layer >= -1 && p->forced_layer <= 2 && p->sigma2 > 0.0;
}

Layout layout(const bm_params* p) {
  Layout L;
  memset(&L, 0, sizeof(L));
  const size_t GR = p->height / BS, GC = p->width / BS;
  L.ncell = (size_t)p->frames * GR * GC;
  const size_t nc = L.ncell > 0 ? L.ncell : 1;
  size_t o = 0;
  L.off_slotmap = o; o = align_up(o + nc * 4);
  L.off_slot_cell = o; o = align_up(o + nc * 4);
  L.off_level = o; o = align_up(o + nc * 4);
  L.off_level2 = o; o = align_up(o + nc * 4);
  L.off_height = o; o = align_up(o + nc * 4);
  L.off_bucket = o; o = align_up(o + nc * 4);
  L.off_queue = o; o = align_up(o + nc * 4);
  L.off_indeg = o; o = align_up(o + nc * 4);
  L.off_nslots = o; o = align_up(o + 4);
  L.off_sched = o; o = align_up(o + SCHED_WORDS * 4);
  L.off_flags = o; o = align_up(o + nc * 4);
  L.off_excl = o; o = align_up(o + nc * 4);
  L.off_cellbuf = o; o = align_up(o + nc * 256 * 8);
  L.off_reccnt = o; o = align_up(o + nc);
  L.off_counters = o; o = align_up(o + 16 * 8);
  L.off_ringtab = o; o = align_up(o + 64 * 33 * 4);
  L.off_postab = o; o = align_up(o + 64 * MAXCAND * 2);
  size_t b1 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b1, (int*)nullptr, (int*)nullptr, (int)nc);
  L.cub_bytes = b1;
  L.off_cub = o; o = align_up(o + L.cub_bytes);
  const int per_sm = cells_per_sm();
  const size_t cap = (size_t)sm_count() * per_sm;
  L.grid = (int)(nc < cap ? nc : cap);
  if (L.grid < 1) L.grid = 1;
  L.scratch_per_cta = HQL_SCRATCH_FUSED;
  L.off_scratch = o; o = align_up(o + (size_t)L.grid * L.scratch_per_cta * 8);
  L.total = o;
  return L;
}

int cuda_status(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "blockmend_b200: CUDA error: %s\n", cudaGetErrorString(e));
    return BM_ERR_CUDA;
  }
  return BM_OK;
}

constexpr int NEV = 256;
cudaEvent_t g_ev[NEV][2];
bool g_ev_init = false;
int g_nev = 0;

}  // namespace

extern "C" {

int bm_abi_version(void) { return BM_ABI_VERSION; }

int bm_debug_phase_cycles(unsigned long long* out48, int reset) {
  // the three builds' counters added (only the build that ran has non-zero ones)
  if (cudaMemcpyFromSymbol(out48, g_phase_cycles, 48 * 8) != cudaSuccess) return BM_ERR_CUDA;
  if (reset) {
    unsigned long long z[48] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, 48 * 8);
  }
  if (bm_wide::add_phase_cycles(out48, reset) != cudaSuccess) return BM_ERR_CUDA;
  if (bm_cluster::add_phase_cycles(out48, reset) != cudaSuccess) return BM_ERR_CUDA;
  return BM_OK;
}

int bm_kernel_times_ms(float* out, int cap) {
  int n = g_nev < cap ? g_nev : cap;
  for (int i = 0; i < n; i++) {
    float ms = -1.f;
    if (cudaEventSynchronize(g_ev[i][1]) != cudaSuccess) return i;
    cudaEventElapsedTime(&ms, g_ev[i][0], g_ev[i][1]);
    out[i] = ms;
  }
  return n;
}

void bm_kernel_times_reset(void) { g_nev = 0; }

int bm_device_clock_khz(void) {
  int dev = 0, khz = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev) != cudaSuccess) return 0;
  return khz;
}

const char* bm_status_string(int s) {
  switch (s) {
    case BM_OK: return "ok";
    case BM_ERR_ARGS: return "bad arguments or shape mismatch";
    case BM_ERR_LOST_LEFT: return "concealment left LOST pixels behind";
    case BM_ERR_CUDA: return "CUDA error or no CUDA device";
    case BM_ERR_WORKSPACE: return "workspace too small";
    case BM_ERR_STATES: return "mask contains a value outside the PixelState range";
    default: return "unknown status";
  }
}

size_t bm_workspace_bytes(const bm_params* p) {
  if (!params_ok(p)) return 0;
  return layout(p).total;
}

int64_t bm_max_records(const bm_params* p) {
  if (!params_ok(p)) return 0;
  return (int64_t)p->frames * (p->height / BS) * (p->width / BS) * 64;
}

int bm_conceal(const bm_params* p, const void* pixels, const uint8_t* states, double* out_f64, uint8_t* out_u8,
               bm_patch_record* out_records, bm_summary* out_summary, void* workspace, size_t workspace_bytes,
               void* stream_) {
  if (!params_ok(p) || !pixels || !states) return BM_ERR_ARGS;
  cudaStream_t stream = (cudaStream_t)stream_;
  Layout L = layout(p);
  if (!workspace || workspace_bytes < L.total) return BM_ERR_WORKSPACE;
  char* ws = (char*)workspace;
  KParams P;
  memset(&P, 0, sizeof(P));
  P.B = p->frames;
  P.H = p->height;
  P.W = p->width;
  P.GR = p->height / BS;
  P.GC = p->width / BS;
  P.pix_f64 = p->pixel_dtype == BM_PIX_F64;
  P.t_phi = p->t_phi;
  P.t_nu = p->t_nu;
  P.sigma2 = p->sigma2;
  P.forced = p->forced_layer;
  P.build = (p->flags & BM_FLAG_BUILD_CLUSTER) ? BUILD_CLUSTER
            : (p->flags & BM_FLAG_BUILD_512) ? 512 : ((p->flags & BM_FLAG_BUILD_256) ? 256 : 0);
  P.narrow_cluster = (p->flags & BM_FLAG_NARROW_512) ? 0 : NARROW_CLUSTER_DEFAULT;
  P.pixels = pixels;
  P.states = states;
  P.out_f64 = out_f64;
  P.out_u8 = out_u8;
  P.records = out_records;
  P.slotmap = (int*)(ws + L.off_slotmap);
  P.slot_cell = (int*)(ws + L.off_slot_cell);
  P.level = (unsigned*)(ws + L.off_level);
  P.queue = (unsigned*)(ws + L.off_queue);
  P.indeg = (unsigned*)(ws + L.off_indeg);
  P.bucket = (unsigned*)(ws + L.off_bucket);
  P.sched = (unsigned*)(ws + L.off_sched);
  P.nslots = (int*)(ws + L.off_nslots);
  P.cellbuf = (double*)(ws + L.off_cellbuf);
  P.rec_count = (uint8_t*)(ws + L.off_reccnt);
  P.counters = (unsigned long long*)(ws + L.off_counters);
  P.ringtab = (int*)(ws + L.off_ringtab);
  P.postab = (uint16_t*)(ws + L.off_postab);
  P.scratch = (double*)(ws + L.off_scratch);
  P.scratch_per_cta = L.scratch_per_cta;
  P.sms = sm_count();
  int* flags = (int*)(ws + L.off_flags);
  int* excl = (int*)(ws + L.off_excl);
  const int nc = (int)L.ncell;
  cudaError_t e;
  if ((e = cudaMemsetAsync(P.counters, 0, 16 * 8, stream)) != cudaSuccess) return cuda_status(e);
  if ((e = cudaMemsetAsync(P.sched, 0, SCHED_WORDS * 4, stream)) != cudaSuccess) return cuda_status(e);
  if (nc == 0) {
    if ((e = cudaMemsetAsync(P.nslots, 0, 4, stream)) != cudaSuccess) return cuda_status(e);
  }
  const int sms = sm_count();
  // dense outputs first (non-lost cells keep their input values)
  if (out_f64 || out_u8) k_init_out<<<sms * 4, 256, 0, stream>>>(P);
  // lost flags per cell, LOST pixels outside the block grid and the state
  // range check: always, also for frames smaller than one cell (ncell = 0)
  k_cell_flags<<<sms * 4, 256, 0, stream>>>(P, flags);
  if (nc > 0) {
    size_t cb = L.cub_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(ws + L.off_cub, cb, flags, excl, nc, stream)) != cudaSuccess)
      return cuda_status(e);
    k_slots<<<sms * 4, 256, 0, stream>>>(P, flags, excl);
    unsigned* height = (unsigned*)(ws + L.off_height);
    k_depth<false><<<(P.B + 7) / 8, 256, 0, stream>>>(P, P.level);
    k_depth<true><<<(P.B + 7) / 8, 256, 0, stream>>>(P, height);
    // dataflow scheduler: dependency counters, priority buckets, ready FIFOs
    if ((e = cudaMemsetAsync(P.queue, 0xFF, (size_t)nc * 4, stream)) != cudaSuccess) return cuda_status(e);
    k_sched_prep<<<sms, 256, 0, stream>>>(P, height);
    k_postab<<<64, 256, 0, stream>>>(P);
    k_sched_seed<<<sms, 256, 0, stream>>>(P);
    const size_t smem = sizeof(CellSmem), smem_w = bm_wide::cell_smem_bytes();
    bm_host::DevState& D = bm_host::dev_state();
    if (!D.attr.load()) {
      if ((e = cudaFuncSetAttribute(k_conceal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return cuda_status(e);
      D.attr = true;
    }
    if (!D.attr_w.load()) {
      if ((e = bm_wide::set_smem(smem_w)) != cudaSuccess) return cuda_status(e);
      if ((e = bm_cluster::set_smem(bm_cluster::cell_smem_bytes())) != cudaSuccess) return cuda_status(e);
      D.clusters = bm_cluster::max_clusters(bm_cluster::cell_smem_bytes());
      D.attr_w = true;
    }
    const bool timed = (p->flags & BM_FLAG_TIME_KERNEL) != 0;
    const int slot_ev = g_nev < NEV ? g_nev : NEV - 1;
    if (timed) {
      if (!g_ev_init) {
        for (int i = 0; i < NEV; i++) {
          cudaEventCreate(&g_ev[i][0]);
          cudaEventCreate(&g_ev[i][1]);
        }
        g_ev_init = true;
      }
      cudaEventRecord(g_ev[slot_ev][0], stream);
    }
    // both builds launch; each returns at once unless the DAG shape is its own
    k_conceal<<<L.grid, NT, smem, stream>>>(P);
    if ((e = bm_wide::launch(&P, sms, smem_w, stream)) != cudaSuccess) return cuda_status(e);
    if ((e = bm_cluster::launch(&P, D.clusters, bm_cluster::cell_smem_bytes(), stream)) != cudaSuccess)
      return cuda_status(e);
    if (timed) {
      cudaEventRecord(g_ev[slot_ev][1], stream);
      if (g_nev < NEV) g_nev++;
    }
  }
  if (out_summary) k_summary<<<1, 32, 0, stream>>>(P, out_summary);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e);
  return BM_OK;
}

int bm_compact_records(const bm_params* p, const bm_patch_record* slot_records, void* workspace,
                       bm_patch_record* out_records, int64_t* out_count, void* stream_) {
  if (!params_ok(p) || !slot_records || !workspace || !out_records || !out_count) return BM_ERR_ARGS;
  cudaStream_t stream = (cudaStream_t)stream_;
  Layout L = layout(p);
  char* ws = (char*)workspace;
  const int nc = (int)L.ncell;
  if (nc == 0) {
    *out_count = 0;
    return BM_OK;
  }
  int* cnt = (int*)(ws + L.off_flags);  // flags are dead after bm_conceal
  int* excl = (int*)(ws + L.off_level2);
  k_u8_to_int<<<sm_count(), 256, 0, stream>>>((const uint8_t*)(ws + L.off_reccnt), (int*)(ws + L.off_nslots), cnt, nc);
  size_t cb = L.cub_bytes;
  cudaError_t e;
  if ((e = cub::DeviceScan::ExclusiveSum(ws + L.off_cub, cb, cnt, excl, nc, stream)) != cudaSuccess)
    return cuda_status(e);
  k_compact_records<<<sm_count() * 4, 64, 0, stream>>>(slot_records, (const uint8_t*)(ws + L.off_reccnt), excl,
                                                        (int*)(ws + L.off_nslots), out_records);
  int last_excl = 0, last_cnt = 0;
  if ((e = cudaMemcpyAsync(&last_excl, excl + nc - 1, 4, cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaMemcpyAsync(&last_cnt, cnt + nc - 1, 4, cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return cuda_status(e);
  *out_count = (int64_t)last_excl + last_cnt;
  return BM_OK;
}

int bm_estimate_batch(int32_t layer, int32_t count, int32_t max_m, double sigma2, const int32_t* n_y,
                      const int32_t* m, const double* y0, const double* x, const double* y, double* out_values,
                      bm_patch_record* out_info, void* stream_) {
  if (count < 0 || max_m < 0 || max_m > MAXCAND || layer < 0 || layer > 2 || !(sigma2 > 0.0)) return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  cudaError_t e;
  double* scratch = nullptr;
  const size_t per = HQL_SCRATCH_DENSE;
  if ((e = cudaMallocAsync((void**)&scratch, (size_t)count * per * 8, stream)) != cudaSuccess) return cuda_status(e);
  EstBatchArgs A{layer, count, max_m, sigma2, n_y, m, y0, x, y, out_values, out_info, scratch};
  const size_t smem = sizeof(EstBatchSmem);
  bm_host::DevState& D = bm_host::dev_state();
  if (!D.est_attr.load()) {
    if ((e = cudaFuncSetAttribute(k_estimate_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return cuda_status(e);
    D.est_attr = true;
  }
  k_estimate_batch<<<count, NT, smem, stream>>>(A);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e);
  cudaFreeAsync(scratch, stream);
  return BM_OK;
}

int bm_select_and_estimate(const bm_params* p, const double* pixels, const uint8_t* states, int32_t count,
                           const int32_t* origins, const uint32_t* layouts, const double* y0,
                           double* out_values, bm_patch_record* out_records, void* stream_) {
  if (!params_ok(p) || p->frames != 1 || p->pixel_dtype != BM_PIX_F64 || !pixels || !states || count < 0)
    return BM_ERR_ARGS;
  if (count == 0) return BM_OK;
  if (!origins || !layouts || !y0 || !out_values || !out_records) return BM_ERR_ARGS;
  cudaStream_t stream = (cudaStream_t)stream_;
  KParams P;
  memset(&P, 0, sizeof(P));
  P.B = 1;
  P.H = p->height;
  P.W = p->width;
  P.GR = p->height / BS;
  P.GC = p->width / BS;
  P.pix_f64 = 1;
  P.t_phi = p->t_phi;
  P.t_nu = p->t_nu;
  P.sigma2 = p->sigma2;
  P.forced = p->forced_layer;
  P.pixels = pixels;
  P.states = states;  // slotmap / ringtab / records stay null: values straight from the working image
  SelectArgs A{count, origins, layouts, y0, out_values, out_records};
  const size_t smem = sizeof(CellSmem);
  cudaError_t e;
  bm_host::DevState& D = bm_host::dev_state();
  if (!D.select_attr.load()) {
    if ((e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return cuda_status(e);
    D.select_attr = true;
  }
  k_select<<<count, NT, smem, stream>>>(P, A);
  return cuda_status(cudaGetLastError());
}

// Host-buffer entry: cached device buffers per shape, pinned staging.
namespace {
std::mutex g_host_mu;
struct HostCache {
  size_t npix = 0, pixbytes = 0, ws_bytes = 0, rec_cap = 0;
  void *d_pix = nullptr, *d_ws = nullptr;
  uint8_t *d_st = nullptr, *d_u8 = nullptr;
  double* d_f64 = nullptr;
  bm_patch_record *d_rec = nullptr, *d_rec2 = nullptr;
  bm_summary* d_sum = nullptr;
  cudaStream_t stream = nullptr;
};
HostCache g_host;
}  // namespace

int bm_conceal_host(const bm_params* p, const void* pixels, const uint8_t* states, double* out_f64, uint8_t* out_u8,
                    bm_patch_record* out_records, int64_t* out_nrec, bm_summary* out_summary) {
  if (!params_ok(p) || !pixels || !states) return BM_ERR_ARGS;
  std::lock_guard<std::mutex> lk(g_host_mu);
  HostCache& C = g_host;
  cudaError_t e;
  if (!C.stream && (e = cudaStreamCreateWithFlags(&C.stream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_status(e);
  const size_t npix = (size_t)p->frames * p->height * p->width;
  const size_t pixbytes = npix * (p->pixel_dtype == BM_PIX_F64 ? 8 : 1);
  const size_t wsb = bm_workspace_bytes(p);
  const size_t rec_cap = out_records ? (size_t)bm_max_records(p) : 0;
  if (npix != C.npix || pixbytes != C.pixbytes || wsb > C.ws_bytes || rec_cap > C.rec_cap) {
    cudaStreamSynchronize(C.stream);
    cudaFree(C.d_pix); cudaFree(C.d_ws); cudaFree(C.d_st); cudaFree(C.d_u8); cudaFree(C.d_f64);
    cudaFree(C.d_rec); cudaFree(C.d_rec2); cudaFree(C.d_sum);
    cudaStreamDestroy(C.stream);
    C = HostCache{};
    if ((e = cudaStreamCreateWithFlags(&C.stream, cudaStreamNonBlocking)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaMalloc(&C.d_pix, pixbytes)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaMalloc((void**)&C.d_st, npix)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaMalloc((void**)&C.d_u8, npix)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaMalloc(&C.d_ws, wsb)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaMalloc((void**)&C.d_sum, sizeof(bm_summary))) != cudaSuccess) return cuda_status(e);
    if (rec_cap) {
      if ((e = cudaMalloc((void**)&C.d_rec, rec_cap * sizeof(bm_patch_record))) != cudaSuccess) return cuda_status(e);
      if ((e = cudaMalloc((void**)&C.d_rec2, rec_cap * sizeof(bm_patch_record))) != cudaSuccess) return cuda_status(e);
    }
    C.npix = npix;
    C.pixbytes = pixbytes;
    C.ws_bytes = wsb;
    C.rec_cap = rec_cap;
  }
  // the FP64 output buffer only when FP64 output is requested (8 B/pixel)
  if (out_f64 && !C.d_f64 && (e = cudaMalloc((void**)&C.d_f64, npix * 8)) != cudaSuccess) return cuda_status(e);
  if ((e = cudaMemcpyAsync(C.d_pix, pixels, pixbytes, cudaMemcpyHostToDevice, C.stream)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaMemcpyAsync(C.d_st, states, npix, cudaMemcpyHostToDevice, C.stream)) != cudaSuccess)
    return cuda_status(e);
  int rc = bm_conceal(p, C.d_pix, C.d_st, out_f64 ? C.d_f64 : nullptr, C.d_u8, out_records ? C.d_rec : nullptr,
                      C.d_sum, C.d_ws, C.ws_bytes, C.stream);
  if (rc) return rc;
  bm_summary sum;
  if ((e = cudaMemcpyAsync(&sum, C.d_sum, sizeof(sum), cudaMemcpyDeviceToHost, C.stream)) != cudaSuccess)
    return cuda_status(e);
  if (out_u8 && (e = cudaMemcpyAsync(out_u8, C.d_u8, npix, cudaMemcpyDeviceToHost, C.stream)) != cudaSuccess)
    return cuda_status(e);
  if (out_f64 && (e = cudaMemcpyAsync(out_f64, C.d_f64, npix * 8, cudaMemcpyDeviceToHost, C.stream)) != cudaSuccess)
    return cuda_status(e);
  if (out_records) {
    int64_t cnt = 0;
    rc = bm_compact_records(p, C.d_rec, C.d_ws, C.d_rec2, &cnt, C.stream);
    if (rc) return rc;
    if (cnt > 0 && (e = cudaMemcpyAsync(out_records, C.d_rec2, (size_t)cnt * sizeof(bm_patch_record),
                                        cudaMemcpyDeviceToHost, C.stream)) != cudaSuccess)
      return cuda_status(e);
    if (out_nrec) *out_nrec = cnt;
  }
  if ((e = cudaStreamSynchronize(C.stream)) != cudaSuccess) return cuda_status(e);
  if (out_summary) *out_summary = sum;
  if (sum.bad_states) return BM_ERR_STATES;
  if (sum.lost_left) return BM_ERR_LOST_LEFT;
  return BM_OK;
}

}  // extern "C"
