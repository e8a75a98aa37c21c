// bm_kernels.cuh — device side of the concealment path: kernel parameters,
// the per-cell shared-memory layout, mask preprocessing (lost-cell slots,
// dependency levels, ready FIFOs), the persistent CTA-per-lost-cell
// concealment kernel and the dense estimator kernel.
//
// Compiled three times (namespace BM_NS, CTA width BM_NT, cluster size
// BM_CS): bm_conceal.cu (bm, 256 threads, 2 cells per SM), bm_conceal_wide.cu
// (bmw, 512 threads, 1 cell per SM) and bm_conceal_cluster.cu (bmc, 2-CTA
// clusters of 512 threads per cell).  All three are launched; each returns at
// once unless the dependency DAG's shape selects it (k_conceal): the narrower
// the DAG, the more the per-cell latency (critical path) sets the time.
#pragma once
#include "../../include/blockmend_b200.h"
#include "bm_common.cuh"
#include "bm_estimators.cuh"
#include "bm_hql.cuh"

namespace BM_NS {

struct KParams {
  int B, H, W, GR, GC;
  int pix_f64;
  double t_phi, t_nu, sigma2;
  int forced;
  const void* pixels;
  const uint8_t* states;
  double* out_f64;
  uint8_t* out_u8;
  bm_patch_record* records;
  // workspace
  int* slotmap;        // [B*GR*GC] slot index or -1
  int* slot_cell;      // [ncell] linear cell index of slot
  unsigned* level;     // [ncell]
  unsigned* queue;     // [ncell] ready FIFOs (bucket b at boff[b]); ~0 = not yet written
  unsigned* indeg;     // [ncell] unfinished earlier-raster lost 8-neighbours
  unsigned* bucket;    // [ncell] priority bucket of the slot
  unsigned* sched;     // [SCHED_WORDS]: count[NB], head[NB], tail[NB], boff[NB], claimed
  int* nslots;         // [1]
  double* cellbuf;     // [ncell][256]
  uint8_t* rec_count;  // [ncell]
  unsigned long long* counters;  // [12]: BRL, IDL, HQL, deferred, lost_left, bad_states, -, maxlevel,
                                 //       flop64, flop32, hql_patches, gate_candidates
  double* scratch;     // per-CTA HQL scratch
  size_t scratch_per_cta;  // doubles
  int sms;             // SM count (narrow-DAG test)
  int build;           // 0: by DAG shape; 256 / 512 / BUILD_CLUSTER: force that kernel build
  int narrow_cluster;  // narrow DAGs: 1 = the cluster build, 0 = the 512-thread build
  int* ringtab;        // [64][33]: interior cells' expansion-map ring offsets per patch position + max ring
  uint16_t* postab;    // [64][MAXCAND]: interior cells' expansion map per patch position: window
                       // origin (tile row << 8 | tile col) of every entry, in (ring, row, col) order
};

constexpr int BUILD_CLUSTER = 1024;  // KParams::build code of the cluster build
#ifndef BM_GH
#define BM_GH 4  // 1024-entry chunks after the first (A/B: +0.6% on cfg5 against 512)
#endif
#ifndef BM_TABPF
#define BM_TABPF 1  // gate: a chunk's expansion-map table entries loaded before the screening loop (A/B)
#endif
constexpr int GH = BM_GH, GCH = GH * NT;  // gate: expansion-map entries per chunk, GH per thread
#ifndef BM_FIRST_GH
#define BM_FIRST_GH 1
#endif
constexpr int FIRST_GH = BM_FIRST_GH;  // entries per thread of the gated first chunk
static_assert(FIRST_GH >= 1 && FIRST_GH <= GH, "first chunk fits posbuf");

struct CellSmem {
  double tile[TILE * TS];
  float tile32[TILE * TS];
  uint64_t lostbits[TILE];
  uint64_t availbits[TILE];
  int pkey[64];  // schedule key per patch (patch_key), maintained across write-backs
  int wb_lost;   // LOST pixels of the patch just written back
  uint8_t st[TILE * TS];
  uint16_t cand[MAXCAND];
  uint16_t posbuf[GH * NT];  // screen_chunk: window positions of the chunk's entries
  union {
    float rbuf[MAXCAND];   // gate: per expansion-map entry nu weight, -1 = not admissible
    double dbuf[MAXCAND];  // HQL: d_j = |L^-1 (y0 - y_j)|^2
  };
  int pref[2];
  int wcnt[GH * NWARP];
  double ringsum[MAXRING + 2];
  int ringcnt[MAXRING + 2];
  int ring_off[32];
  // per-patch control (written by warp 0 / thread 0, read after a barrier)
  int slot, f, gr, gc;
  unsigned long long remaining, pend;
  int deferred[64];
  int ndef, progressed, nrec;
  int readers;  // some later-raster lost 8-neighbour will read cellbuf
  int pick, skip, gated_stop;
  int m, rings_used, max_ring, K, cur_ring;
  double nu, carry, phi;
  unsigned rowmask[6];
  long long t_start, t_mark, t_pick, t_gather, t_g[4];
  int idl_diag;
  unsigned long long cnt[8];  // BRL IDL HQL deferred | flop64 flop32 hql gate
  bm_patch_record rec;        // the current patch's LayerDecision (profiles.py:174-188)
  EstSmem est;
  HqlSmem hql;
  HqlOut hout;
};

__device__ __forceinline__ int patch_r(int p) { return BS + 2 * (p >> 3); }  // tile coords of patch p
__device__ __forceinline__ int patch_c(int p) { return BS + 2 * (p & 7); }

// ------------------------------------------------------------ preprocessing

// lost flag per grid cell; LOST pixels outside the grid; state range check
__global__ void k_cell_flags(KParams P, int* flags) {
  const int GR = P.GR, GC = P.GC, H = P.H, W = P.W;
  const size_t ncell = (size_t)P.B * GR * GC;
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = warp; c < ncell; c += nwarps) {
    const int f = (int)(c / ((size_t)GR * GC));
    const int rem = (int)(c % ((size_t)GR * GC));
    const int gr = rem / GC, gc = rem % GC;
    const uint8_t* s = P.states + ((size_t)f * H + gr * BS) * W + gc * BS;
    // 256 states: lane reads 8 bytes (row lane/2, half lane&1)
    const int r = lane >> 1, h = (lane & 1) * 8;
    int lost = 0, bad = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      uint8_t v = s[(size_t)r * W + h + i];
      lost |= v == ST_LO;
      bad |= v > ST_RE;
    }
    lost = __any_sync(FULL, lost);
    bad = __any_sync(FULL, bad);
    if (lane == 0) {
      flags[c] = lost;
      if (bad) atomicAdd(&P.counters[5], 1ull);
    }
  }
  // ragged margins (pixels outside the full-cell grid)
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nthr = (size_t)gridDim.x * blockDim.x;
  const int mr = H - GR * BS, mc = W - GC * BS;
  const size_t per_frame = (size_t)mr * W + (size_t)(H - mr) * mc;
  for (size_t i = tid; i < per_frame * P.B; i += nthr) {
    const int f = (int)(i / per_frame);
    size_t k = i % per_frame;
    int r, c;
    if (k < (size_t)mr * W) {
      r = GR * BS + (int)(k / W);
      c = (int)(k % W);
    } else {
      k -= (size_t)mr * W;
      r = (int)(k / mc);
      c = GC * BS + (int)(k % mc);
    }
    const uint8_t v = P.states[((size_t)f * H + r) * W + c];
    if (v == ST_LO) atomicAdd(&P.counters[4], 1ull);
    if (v > ST_RE) atomicAdd(&P.counters[5], 1ull);
  }
}

__global__ void k_slots(KParams P, const int* flags, const int* excl) {
  const size_t ncell = (size_t)P.B * P.GR * P.GC;
  for (size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += (size_t)gridDim.x * blockDim.x) {
    if (flags[c]) {
      P.slotmap[c] = excl[c];
      P.slot_cell[excl[c]] = (int)c;
    } else {
      P.slotmap[c] = -1;
    }
    if (c == ncell - 1) *P.nslots = excl[c] + flags[c];
  }
}

// Longest-path depth of every lost cell in its frame's dependency DAG, one
// warp per frame.  REV = false: level(u) = 1 + max level of its lost
// earlier-raster 8-neighbours ((r-1,c-1),(r-1,c),(r-1,c+1),(r,c-1)), rows top
// down.  REV = true: the mirrored recurrence over later-raster neighbours
// gives height(u) - 1 (longest chain of dependants).  The left-neighbour
// chain inside a row is a max-plus segmented warp scan.
template <bool REV>
__global__ void k_depth(KParams P, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (f >= P.B) return;
  const int GR = P.GR, GC = P.GC;
  const int* sm = P.slotmap + (size_t)f * GR * GC;
  auto slot_at = [&](int r, int c) { return sm[(REV ? GR - 1 - r : r) * GC + (REV ? GC - 1 - c : c)]; };
  unsigned maxlvl = 0;
  for (int r = 0; r < GR; r++) {
    int carry = -1000000;
    int left_lost = 0;
    for (int c0 = 0; c0 < GC; c0 += 32) {
      const int c = c0 + lane;
      const int slot = c < GC ? slot_at(r, c) : -1;
      int base = -1;  // -1: not lost
      if (slot >= 0) {
        int b = 0;
        if (r > 0) {
          for (int dc = -1; dc <= 1; dc++) {
            const int cc = c + dc;
            if (cc < 0 || cc >= GC) continue;
            const int s2 = slot_at(r - 1, cc);
            if (s2 >= 0) b = max(b, (int)out[s2] + 1);
          }
        }
        base = b;
      }
      // chain: depth(c) = max(base(c), depth(c-1)+1) when c-1 is lost;
      // value(c) = depth(c) - c; run-segmented prefix max of (base - c).
      const bool lost = slot >= 0;
      int val = lost ? base - c : -1000000;
      const int up_lost = __shfl_up_sync(FULL, (int)lost, 1);
      const bool prev_lost_inchunk = lane > 0 ? up_lost : left_lost;
      int seg_start = lost && !prev_lost_inchunk;
      if (lane == 0 && lost && left_lost) val = max(val, carry);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ov = __shfl_up_sync(FULL, val, o);
        const int os = __shfl_up_sync(FULL, seg_start, o);
        if (lane >= o && !seg_start) {
          val = max(val, ov);
          seg_start = os;
        }
      }
      if (lost) {
        const unsigned lv = (unsigned)(val + c);
        out[slot] = lv;
        maxlvl = max(maxlvl, lv);
      }
      carry = __shfl_sync(FULL, val, 31);
      left_lost = __shfl_sync(FULL, (int)lost, 31);
      __syncwarp();
    }
    __syncwarp();
    __threadfence_block();
  }
  maxlvl = (unsigned)__reduce_max_sync(FULL, maxlvl);
  if (!REV && lane == 0) atomicMax((unsigned long long*)&P.counters[7], (unsigned long long)maxlvl);
}

// Dataflow scheduler state.  NB ready FIFOs, bucket 0 = longest chains of
// dependants (critical-path priority); each FIFO has an exact-size region of
// the queue array since every slot is pushed exactly once.
constexpr int NB = 32;
constexpr int SCHED_COUNT = 0, SCHED_HEAD = 32, SCHED_TAIL = 64, SCHED_BOFF = 96, SCHED_CLAIMED = 128;
constexpr int SCHED_WORDS = 160;

__device__ __forceinline__ bool cell_lost(const KParams& P, int f, int r, int c, int& slot) {
  if (r < 0 || r >= P.GR || c < 0 || c >= P.GC) return false;
  slot = P.slotmap[((size_t)f * P.GR + r) * P.GC + c];
  return slot >= 0;
}

// per slot: dependency count (lost earlier-raster 8-neighbours) and priority
// bucket from the height (longest chain of dependants, k_depth<true>)
__global__ void k_sched_prep(KParams P, const unsigned* height) {
  if (blockIdx.x == 0 && threadIdx.x < 64) {
    // ring offsets of an interior cell's 64 patch positions (tile coords: the
    // support is the whole 48x48 tile, candidate origins 2..44)
    const int p = threadIdx.x;
    RingGeom g;
    g.pr = BS + 2 * (p >> 3);
    g.pc = BS + 2 * (p & 7);
    g.A0 = 2;
    g.A1 = TILE - 4;
    g.B0 = 2;
    g.B1 = TILE - 4;
    int* t = P.ringtab + p * 33;
    int off = 0, mr = 0;
    for (int r = 0; r < 32; r++) {
      t[r] = off;  // entries of rings < r
      const int c = (r >= 1 && r <= 26) ? ring_count(g, r) : 0;
      off += c;
      if (c > 0) mr = r;
    }
    t[32] = mr;
  }
  const int ns = *P.nslots;
  const unsigned maxh = (unsigned)P.counters[7];  // = max level = longest path
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    const int c = P.slot_cell[s];
    const int f = c / (P.GR * P.GC), rem = c % (P.GR * P.GC), r = rem / P.GC, cc = rem % P.GC;
    int d = 0, o;
    d += cell_lost(P, f, r - 1, cc - 1, o);
    d += cell_lost(P, f, r - 1, cc, o);
    d += cell_lost(P, f, r - 1, cc + 1, o);
    d += cell_lost(P, f, r, cc - 1, o);
    P.indeg[s] = (unsigned)d;
    const unsigned h = min(height[s], maxh);
    const unsigned b = (unsigned)(((unsigned long long)(maxh - h) * NB) / (maxh + 1));
    P.bucket[s] = b;
    atomicAdd(&P.sched[SCHED_COUNT + b], 1u);
  }
}

// The expansion map of an interior cell's 64 patch positions (window
// origins in tile coordinates; translation invariant, like ringtab), so the
// gate's screening reads an entry's window from a table instead of solving
// the ring / raster position in closed form.  One CTA per patch position.
__global__ void k_postab(KParams P) {
  __shared__ int off[32];
  const int p = blockIdx.x, tid = threadIdx.x;
  RingGeom g;
  g.pr = BS + 2 * (p >> 3);
  g.pc = BS + 2 * (p & 7);
  g.A0 = 2;
  g.A1 = TILE - 4;
  g.B0 = 2;
  g.B1 = TILE - 4;
  if (tid < 32) {
    const int cnt = (tid >= 1 && tid <= 28) ? ring_count(g, tid) : 0;
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, inc, o);
      inc += tid >= o ? v : 0;
    }
    off[tid] = inc - cnt;
  }
  __syncthreads();
  const int K = off[31];
  for (int e = tid; e < K; e += blockDim.x) {
    int r = 1;
    while (r < 31 && off[r + 1] <= e) r++;
    int a, b;
    ring_entry(g, r, e - off[r], a, b);
    P.postab[(size_t)p * MAXCAND + e] = (uint16_t)(((a - 2) << 8) | (b - 2));
  }
}

// bucket offsets (every block computes them; block 0 publishes) and the
// initially ready cells (no lost earlier-raster neighbour)
__global__ void k_sched_seed(KParams P) {
  __shared__ unsigned boff[NB];
  if (threadIdx.x == 0) {
    unsigned o = 0;
    for (int b = 0; b < NB; b++) {
      boff[b] = o;
      o += P.sched[SCHED_COUNT + b];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < NB) P.sched[SCHED_BOFF + threadIdx.x] = boff[threadIdx.x];
  const int ns = *P.nslots;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    if (P.indeg[s] == 0) {
      const unsigned b = P.bucket[s];
      const unsigned t = atomicAdd(&P.sched[SCHED_TAIL + b], 1u);
      P.queue[boff[b] + t] = (unsigned)s;
    }
  }
}

__device__ __forceinline__ unsigned atom_dec_acq_rel(unsigned* p) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(0xFFFFFFFFu) : "memory");
  return old;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Pop the next ready cell (warp 0): the highest-priority non-empty FIFO.
// Returns the slot, or -1 when every cell has been claimed.
__device__ int sched_pop(const KParams& P, int nslots) {
  const int lane = threadIdx.x & 31;
  unsigned* sc = P.sched;
  for (;;) {
    const unsigned h = ld_relaxed_u32(&sc[SCHED_HEAD + lane]);
    const unsigned t = ld_relaxed_u32(&sc[SCHED_TAIL + lane]);
    const unsigned ne = __ballot_sync(FULL, h < t);
    if (ne) {
      const int b = __ffs(ne) - 1;
      int slot = -2;
      if (lane == b) {
        if (atomicCAS(&sc[SCHED_HEAD + b], h, h + 1) == h) {
          const unsigned* q = P.queue + sc[SCHED_BOFF + b] + h;
          unsigned v;
          while ((v = ld_acquire_u32(q)) == 0xFFFFFFFFu) __nanosleep(32);  // reserved, being written
          slot = (int)v;
          atomicAdd(&sc[SCHED_CLAIMED], 1u);
        }
      }
      slot = __shfl_sync(FULL, slot, b);
      if (slot >= 0) return slot;
      continue;  // lost the race: rescan
    }
    if ((int)ld_relaxed_u32(&sc[SCHED_CLAIMED]) >= nslots) return -1;
    __nanosleep(256);
  }
}

// --------------------------------------------------------- the cell kernel

// Stage the cell's 48x48 support tile: FP64 values, FP32 shadow, states and
// the per-row LOST / AVAILABLE bitmaps.  Interior tiles of u8 frames take the
// vector path: one thread per (tile row, 16-column chunk) - each chunk lies
// inside one neighbouring cell - moves 16 pixels and 16 states with two
// 16-byte loads (or, for a finished earlier-raster neighbour, its 16 final
// FP64 values from the cell buffer with eight 16-byte loads) and builds the
// chunk's 16-bit LOST / AVAILABLE masks on the way.
__device__ void load_tile(const KParams& P, CellSmem& S) {
  const int f = S.f, gr = S.gr, gc = S.gc;
  const int R0 = gr * BS - BS, C0 = gc * BS - BS;
  const int H = P.H, W = P.W;
  const bool vec = !P.pix_f64 && (W & 15) == 0 && R0 >= 0 && R0 + TILE <= H && C0 >= 0 && C0 + TILE <= W &&
                   ((reinterpret_cast<uintptr_t>(P.pixels) | reinterpret_cast<uintptr_t>(P.states)) & 15) == 0;
  if (vec) {
    __shared__ uint16_t lmask[TILE * 3], amask[TILE * 3];
    for (int t = threadIdx.x; t < TILE * 3; t += NT) {
      const int tr = t / 3, ch = t % 3;  // tile row, 16-column chunk (= neighbour column ch)
      const size_t o = ((size_t)f * H + R0 + tr) * W + C0 + 16 * ch;
      const uint4 sv = __ldg(reinterpret_cast<const uint4*>(P.states + o));
      const int ntr = tr / BS;
      int pslot = -1;
      if (P.slotmap && (ntr == 0 || (ntr == 1 && ch == 0)))
        pslot = P.slotmap[((size_t)f * P.GR + gr - 1 + ntr) * P.GC + gc - 1 + ch];
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(&sv);
      double* trow = S.tile + tr * TS + 16 * ch;
      float* frow = S.tile32 + tr * TS + 16 * ch;
      uint8_t* srow = S.st + tr * TS + 16 * ch;
      unsigned lm = 0, am = 0;
      if (pslot >= 0) {  // finished earlier-raster neighbour: its final values, LOST -> RECONSTRUCTED
        const double2* cb = reinterpret_cast<const double2*>(P.cellbuf + (size_t)pslot * 256 + (tr % BS) * BS);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const double2 v = __ldcg(cb + q);
          trow[2 * q] = v.x;
          trow[2 * q + 1] = v.y;
          frow[2 * q] = (float)v.x;
          frow[2 * q + 1] = (float)v.y;
        }
#pragma unroll
        for (int q = 0; q < 16; q++) {
          const uint8_t st = sb[q] == ST_LO ? ST_RE : sb[q];
          srow[q] = st;
          am |= (unsigned)(st == ST_AV) << q;
        }
      } else {
        const uint4 pv = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(P.pixels) + o));
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(&pv);
#pragma unroll
        for (int q = 0; q < 16; q++) {
          trow[q] = (double)pb[q];
          frow[q] = (float)pb[q];
          srow[q] = sb[q];
          lm |= (unsigned)(sb[q] == ST_LO) << q;
          am |= (unsigned)(sb[q] == ST_AV) << q;
        }
      }
      lmask[t] = (uint16_t)lm;
      amask[t] = (uint16_t)am;
    }
    __syncthreads();
    if (threadIdx.x < TILE) {
      const int r = threadIdx.x;
      S.lostbits[r] = (uint64_t)lmask[3 * r] | ((uint64_t)lmask[3 * r + 1] << 16) | ((uint64_t)lmask[3 * r + 2] << 32);
      S.availbits[r] = (uint64_t)amask[3 * r] | ((uint64_t)amask[3 * r + 1] << 16) | ((uint64_t)amask[3 * r + 2] << 32);
    }
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < TILE * TILE; i += NT) {
    const int tr = i / TILE, tc = i % TILE;
    const int r = R0 + tr, c = C0 + tc;
    double v = 0.0;
    uint8_t s = ST_LO;  // out of image: never usable (framework.py:160)
    if (r >= 0 && r < H && c >= 0 && c < W) {
      const size_t o = ((size_t)f * H + r) * W + c;
      s = P.states[o];
      const int ntr = tr / BS, ntc = tc / BS;
      const int nr = gr - 1 + ntr, nc = gc - 1 + ntc;
      int pslot = -1;
      if (P.slotmap && (ntr == 0 || (ntr == 1 && ntc == 0)) && nr >= 0 && nc >= 0 && nc < P.GC)
        pslot = P.slotmap[((size_t)f * P.GR + nr) * P.GC + nc];
      if (pslot >= 0) {  // finished earlier-raster neighbour: its final values
        v = __ldcg(&P.cellbuf[(size_t)pslot * 256 + (tr % BS) * BS + (tc % BS)]);
        if (s == ST_LO) s = ST_RE;
      } else {
        v = P.pix_f64 ? ((const double*)P.pixels)[o] : (double)((const uint8_t*)P.pixels)[o];
      }
    }
    S.tile[tr * TS + tc] = v;
    S.tile32[tr * TS + tc] = (float)v;
    S.st[tr * TS + tc] = s;
  }
  __syncthreads();
  if (threadIdx.x < TILE) {
    uint64_t b = 0, a = 0;
    for (int c = 0; c < TILE; c++) {
      const uint8_t st = S.st[threadIdx.x * TS + c];
      b |= (uint64_t)(st == ST_LO) << c;
      a |= (uint64_t)(st == ST_AV) << c;
    }
    S.lostbits[threadIdx.x] = b;
    S.availbits[threadIdx.x] = a;
  }
  __syncthreads();
}

// Gather of the admissible candidates in (ring, row, col) order with the ring
// by ring nu gate (profiles.py:113-124, framework.py:171-207), or the one-shot
// full gather of _forced_estimate (profiles.py:148-149).  Sets S.m, rings_used,
// nu; S.cand holds the candidates.
// Screen entries [e0, e0 + GCH) of the expansion map: admissibility
// (framework.py:176), FP32 nu weight in gated mode (raw_idl_weights,
// estimators.py:105-109), ordered ballot compaction into S.cand after the
// m_total candidates already gathered.  r is stored per entry in S.rbuf
// (-1 = not admissible).  Returns the chunk's admissible count (all threads).
// nu screening weight of the admissible window at tile position pos: FP32
// Nadaraya-Watson distance and weight (raw_idl_weights, estimators.py:105-109).
__device__ __forceinline__ float nu_weight(const CellSmem& S, int pos, int n, float invf) {
  const EstSmem& E = S.est;
  const float* tp = S.tile32 + pos;
  float d2a = 0.f, d2b = 0.f;
  int k = 0;
  for (; k + 2 <= n; k += 2) {
    const float da = tp[E.uoff[k]] - E.y0f[k];
    const float db = tp[E.uoff[k + 1]] - E.y0f[k + 1];
    d2a = fmaf(da, da, d2a);
    d2b = fmaf(db, db, d2b);
  }
  if (k < n) {
    const float da = tp[E.uoff[k]] - E.y0f[k];
    d2a = fmaf(da, da, d2a);
  }
  return expf(-(d2a + d2b) * invf);
}

__device__ __forceinline__ int screen_chunk(CellSmem& S, const RingGeom& g, int e0, int gh, int K, int max_ring,
                                            int R0, int C0, bool gated, float invf, int m0, bool sync_end,
                                            const uint16_t* __restrict__ tab) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  EstSmem& E = S.est;
  const int n = E.n;
  // rolled over the gh <= GH entries per thread (one code copy); the window
  // positions wait in posbuf for the compaction (0xFFFF = not admissible)
#if BM_TABPF
  static_assert(GH <= 4, "prefetched table entries fit one 64-bit register");
  unsigned long long tabv = 0;
  if (tab) {
#pragma unroll
    for (int h = 0; h < GH; h++) {
      const int e = e0 + h * NT + tid;
      if (h < gh && e < K) tabv |= (unsigned long long)__ldg(tab + e) << (16 * h);
    }
  }
#endif
#pragma unroll 1
  for (int h = 0; h < gh; h++) {
    const int e = e0 + h * NT + tid;
    bool adm = false;
    int pos = 0xFFFF;
    if (e < K) {
      // ring of entry e: the last ring starting at or before e (empty rings
      // share their successor's offset), branch-free binary search over the
      // 32 ring offsets (rings past max_ring start at K > e)
      int wr, wc;  // window origin, tile coords
      if (tab) {     // interior cell: the precomputed expansion map (k_postab)
#if BM_TABPF
        const unsigned v = (unsigned)(tabv >> (16 * h)) & 0xFFFFu;
#else
        const unsigned v = __ldg(tab + e);
#endif
        wr = (int)(v >> 8);
        wc = (int)(v & 255u);
      } else {
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) lo += S.ring_off[lo + step] <= e ? step : 0;
        int a, b;
        ring_entry(g, lo, e - S.ring_off[lo], a, b);
        wr = a - 2 - R0;
        wc = b - 2 - C0;
      }
      bool ok = true;
#pragma unroll
      for (int q = 0; q < 6; q++)
        if ((S.lostbits[wr + q] >> wc) & S.rowmask[q]) ok = false;
      adm = ok;
      float rw = -1.f;
      if (ok) {
        pos = wr * TS + wc;
        rw = gated ? nu_weight(S, pos, n, invf) : 0.f;
      }
      S.rbuf[e] = rw;
    }
    S.posbuf[h * NT + tid] = (uint16_t)pos;
    const unsigned bal = __ballot_sync(FULL, adm);
    if (lane == 0) S.wcnt[h * NWARP + warp] = __popc(bal);
  }
  __syncthreads();
  // ordered compaction (entries are in (h, warp, lane) = expansion-map order)
  int tot = 0;
#pragma unroll 1
  for (int h = 0; h < gh; h++) {
    int base = tot;
#pragma unroll
    for (int w = 0; w < NWARP; w++) {
      const int c = S.wcnt[h * NWARP + w];
      if (w < warp) base += c;
      tot += c;
    }
    const int pos = S.posbuf[h * NT + tid];
    const bool adm = pos != 0xFFFF;
    const unsigned bal = __ballot_sync(FULL, adm);
    const int wpre = __popc(bal & ((1u << lane) - 1));
    if (adm) S.cand[m0 + base + wpre] = (uint16_t)pos;
  }
  // (wcnt / posbuf are reused by the next chunk; when the nu accounting
  // follows, its barrier comes first)
  if (sync_end) __syncthreads();
  return tot;
}

// Gather of the admissible candidates in (ring, row, col) order with the ring
// by ring nu gate (profiles.py:113-124, framework.py:171-207), or the one-shot
// full gather of _forced_estimate (profiles.py:148-149).  Sets S.m, rings_used,
// nu; S.cand holds the candidates.  The gate walks the first chunk (rings
// 1..~5, where IDL decisions fall) ring by ring; if nu has not reached T_nu
// the rest of the map is screened in one barrier-light sweep and the per-ring
// sums are formed afterwards, giving the same stopping ring.
__device__ void gather(const KParams& P, CellSmem& S, int pr_t, int pc_t, bool gated) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  EstSmem& E = S.est;
  const int n = E.n;
  // geometry (absolute coordinates)
  const int br = S.gr * BS, bc = S.gc * BS;
  const int R0 = br - BS, C0 = bc - BS;
  RingGeom g;
  g.pr = R0 + pr_t;
  g.pc = C0 + pc_t;
  const int r0 = max(0, br - BS), r1 = min(P.H, br + 2 * BS);
  const int c0 = max(0, bc - BS), c1 = min(P.W, bc + 2 * BS);
  g.A0 = r0 + 2;
  g.A1 = r1 - 4;
  g.B0 = c0 + 2;
  g.B1 = c1 - 4;
  if (warp == 0) {
    int mr, K;
    if (P.ringtab && ((pr_t | pc_t) & 1) == 0 && r0 == br - BS && c0 == bc - BS && r1 == br + 2 * BS &&
        c1 == bc + 2 * BS) {
      // interior cell: the patch position's ring offsets from the table
      // (k_sched_prep; the geometry is translation invariant)
      const int* t = P.ringtab + (size_t)((pr_t - BS) / 2 * 8 + (pc_t - BS) / 2) * 33;
      S.ring_off[lane] = t[lane];
      mr = t[32];
      K = t[31];
    } else {
      const int cnt = (lane >= 1 && lane <= 28) ? ring_count(g, lane) : 0;
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, inc, o);
        inc += lane >= o ? v : 0;
      }
      S.ring_off[lane] = inc - cnt;  // ring_off[r] = entries of rings < r (K past the last ring)
      const unsigned nz = __ballot_sync(FULL, cnt > 0);
      mr = nz ? 31 - __clz(nz) : 0;
      K = __shfl_sync(FULL, inc, mr);
    }
    __syncwarp();
    if (lane == 0) {
      S.max_ring = mr;
      S.K = mr ? K : 0;
      S.ring_off[mr + 1] = S.K;
      S.m = 0;
      S.nu = 0.0;
      S.carry = 0.0;
      S.pref[0] = 0;
      S.cur_ring = 0;
      S.gated_stop = 0;
      S.rings_used = 0;
    }
  }
  __syncthreads();
  if (tid == 0) S.t_g[0] = clock64();
  const int K = S.K, max_ring = S.max_ring;
  if (max_ring == 0) {  // empty expansion map: exhausted before the first ring
    if (tid == 0) { S.m = 0; S.rings_used = 0; }
    __syncthreads();
    return;
  }
  const float invf = (float)(1.0 / (2.0 * P.sigma2 * n));
  // interior cells at schedule positions: the expansion map from the table
  const bool interior = r0 == br - BS && c0 == bc - BS && r1 == br + 2 * BS && c1 == bc + 2 * BS;
  const uint16_t* tab = (P.postab && P.ringtab && ((pr_t | pc_t) & 1) == 0 && interior)
                            ? P.postab + (size_t)((pr_t - BS) / 2 * 8 + (pc_t - BS) / 2) * MAXCAND
                            : nullptr;
  // one screening loop (a single inlined copy of screen_chunk): ungated = the
  // whole map; gated = the first chunk, its ring-by-ring nu stop, then the
  // rest of the map in one sweep.  The nu accounting (per-ring sums, one warp
  // per ring, then the reference's sequential nu loop on thread 0) is one
  // code copy run over entry window [0, e1) after the first chunk and, if nu
  // has not reached T_nu, over [e1, K) after the last.
  const int gh1 = gated ? FIRST_GH : GH;  // gated: a smaller first chunk (IDL stops fall in rings 1..~3)
  const int e1 = min(gh1 * NT, K);
  int mtot = 0;  // admissible candidates gathered so far (the same in every thread)
  for (int e0 = 0; e0 < K; e0 += (e0 == 0 ? gh1 : GH) * NT) {
    const int gh = e0 == 0 ? gh1 : GH;
    const bool acct = gated && (e0 == 0 || e0 + gh * NT >= K);  // nu accounting after this chunk
    mtot += screen_chunk(S, g, e0, gh, K, max_ring, R0, C0, gated, invf, mtot, !acct, tab);
    if (!acct) continue;
    const int elo = e0 == 0 ? 0 : e1, ehi = e0 == 0 ? e1 : K;
    const int rs = e0 == 0 ? 1 : S.cur_ring;  // first ring not yet accounted (may carry a partial sum)
    if (tid == 0) S.t_g[1] = clock64();
    for (int r = rs + warp; r <= max_ring && S.ring_off[r] < ehi; r += NWARP) {
      const int lo = max(S.ring_off[r], elo), hi = min(S.ring_off[r + 1], ehi);
      double part = 0.0;
      int c = 0;
      for (int i = lo + lane; i < hi; i += 32) {
        const float v = S.rbuf[i];
        const bool ok = v >= 0.f;  // admissible
        part += ok ? (double)v : 0.0;
        c += ok;
      }
      part = warp_sum(part);
      c = warp_sumi(c);
      if (lane == 0) {
        S.ringsum[r] = part;
        S.ringcnt[r] = c;
      }
    }
    __syncthreads();
    if (tid == 0) S.t_g[2] = clock64();
    if (tid == 0) {
      double nu = S.nu, carry = S.carry;
      int m = S.pref[0], stop = 0, r = rs;
      for (; r <= max_ring; r++) {
        if (S.ring_off[r] >= ehi) break;  // ring starts past the window
        m += S.ringcnt[r];
        const double ring = (r == rs ? carry : 0.0) + S.ringsum[r];
        if (S.ring_off[r + 1] > ehi) {  // ring continues past the window
          carry = ring;
          break;
        }
        nu += ring;  // nu += sum of the ring's raw weights (profiles.py:122)
        if (!(nu < P.t_nu) || r >= max_ring) {
          stop = 1;
          break;
        }
      }
      S.gated_stop = stop;
      S.nu = nu;
      S.carry = carry;
      S.cur_ring = r;  // stop ring, or the first ring not fully accounted
      S.pref[0] = m;   // admissible entries of the accounted part
      if (stop) {
        S.rings_used = r;
        S.m = m;
      }
    }
    __syncthreads();
    if (tid == 0) S.t_g[3] = clock64();
#if BM_DIAG
    // gate sub-phases of the patches that go past the first window (diagnostic)
    if (tid == 0) {
      if (e0 == 0 && !S.gated_stop) {
        BM_DIAG_ADD(43, (S.t_g[3] - S.t_g[0]));  // first window: screening + accounting
        S.t_pick = S.t_g[3];                     // (free until estimate_only's bookkeeping)
      } else if (e0 != 0) {
        BM_DIAG_ADD(44, (S.t_g[1] - S.t_pick));  // rest of the map screened
        BM_DIAG_ADD(45, (S.t_g[2] - S.t_g[1]));  // its ring sums
        BM_DIAG_ADD(46, (S.t_g[3] - S.t_g[2]));  // its nu scan
        BM_DIAG_ADD(47, 1);
      }
    }
#endif
    if (S.gated_stop) return;
  }
  if (tid == 0) {  // ungated: the whole map (_forced_estimate, profiles.py:148-149)
    S.m = mtot;
    S.rings_used = max_ring;
  }
  __syncthreads();
}

// Algorithmic FLOPs of one patch; exps are SFU work, not counted.
__device__ __forceinline__ unsigned long long idl_flops(long long M, long long n) { return (unsigned long long)(M * (3 * n + 15)); }
__device__ __forceinline__ unsigned long long hql_flops(long long M, long long n) {
  const long long G = NBETA, k = min(n + 1, M);
  long long f = 2 * M * (4 * n + n * (n + 1) / 2) + 2 * M * (n + 4);  // covariance (+ centring)
  f += n * n * n / 3;                                                 // Cholesky
  f += M * (n * n + 3 * n);                                           // quadforms
  f += G * (M * (2 * n + 4) + 3 * n);                                 // beta grid
  f += 2 * M * (n + 4);                                               // x~0, y~0
  f += M * (n * n + 2 * n) + 2 * k * M * n + 2 * k * M * (n + 4) + 2 * k * n * n + 8 * n * k;  // alpha
  f += 2 * n * n + 8 * n;                                             // correction
  return (unsigned long long)f;
}

__device__ void write_record(const KParams& P, CellSmem& S, const bm_patch_record& rec) {
  if (P.records && cluster_rank() == 0) P.records[(size_t)S.slot * 64 + S.nrec] = rec;
}

// One patch at tile position (pr_t, pc_t): gate + estimate
// (select_and_estimate / _forced_estimate, profiles.py:105-171) into E.vals
// and S.rec; no write-back.
__device__ void estimate_only(const KParams& P, CellSmem& S, int pr_t, int pc_t, double* gS) {
  const int tid = threadIdx.x;
  EstSmem& E = S.est;
  const int forced = P.forced;
  const bool brl = forced >= 0 ? forced == BM_LAYER_BRL : S.phi <= P.t_phi;
  bm_patch_record& rec = S.rec;
  if (tid == 0) {
    memset(&rec, 0, sizeof(rec));
    rec.frame = S.f;
    rec.row = S.gr * BS - BS + pr_t;
    rec.col = S.gc * BS - BS + pc_t;
    rec.phi = S.phi;
    rec.nu = rec.beta = rec.alpha = __longlong_as_double(0x7ff8000000000000ll);
    rec.flags = BM_REC_HAS_PHI | BM_REC_HAS_M;
    rec.n_y = (uint8_t)E.n;
    rec.beta_gap = __int_as_float(0x7fc00000);
  }
  if (brl) {
    brl_values(E);
    if (tid == 0) {
      rec.layer = BM_LAYER_BRL;
      rec.m_candidates = 0;
      rec.rings_used = 0;
    }
    __syncthreads();
  } else {
    const bool gated = forced < 0;
    if (tid == 0) S.t_mark = clock64();
    gather(P, S, pr_t, pc_t, gated);
    const int m = S.m;
    if (tid == 0) {  // diagnostics: pick/extract and gather time of gated IDL-bound patches
      const long long now = clock64();
      S.t_pick = S.t_mark - S.t_start;
      S.t_gather = now - S.t_mark;
      S.t_mark = now;
    }
    if (tid == 0 && gated) {
      // nu loop: M_g (3n + 2) FP32 flops; exps counted separately
      S.cnt[5] += (unsigned long long)m * (3 * E.n + 2);
      S.cnt[7] += (unsigned long long)m;
    }
    TileAcc acc{S.tile, S.cand, E.uoff, S.tile32};
    if (tid == 0) {
      rec.rings_used = (uint8_t)S.rings_used;
      rec.m_candidates = m;
    }
    // layer ladder with one IDL call site: 0 = gated IDL (nu >= T_nu,
    // profiles.py:123-124), 1 = forced IDL (profiles.py:144-153), 2 = HQL
    // with its ladder HQL -> IDL -> BRL (estimators.py:248-286)
    const int mode = (gated && !(S.nu < P.t_nu)) ? 0 : (forced == BM_LAYER_IDL ? 1 : 2);
    bool done = false;
    if (mode == 2 && m >= 2) {
      if (tid == 0) BM_DIAG_ADD(0, (clock64() - S.t_start));
      hql_columns(S.hql, E.n, E.uoff);
      __syncthreads();
      TileLoader zv{S.tile, S.cand};
      hql_mma(zv, m, E.n, E.y0, S.hql, gS, S.hout, E.exptab, S.dbuf);
      __syncthreads();
      if (S.hout.ok) {
        done = true;
        if (tid == 0) {
          for (int q = 0; q < 4; q++) E.vals[q] = S.hout.vals[q];
          S.cnt[4] += hql_flops(m, E.n);
          S.cnt[6]++;
          rec.layer = BM_LAYER_HQL;
          rec.beta = S.hout.beta;
          rec.alpha = S.hout.alpha;
          rec.beta_gap = S.hout.gap;
          rec.flags |= BM_REC_HAS_BW;
        }
      }
    }
    const bool run_idl = !done && m >= 1;  // (mode 0 has m >= 1: nu > 0)
    if (run_idl) {
      // gated IDL (mode 0): only thread 0 reads the outcome, and the branch
      // ends with a CTA barrier -> no barrier after the estimate's last step
      idl_estimate_dev(acc, m, P.sigma2, E, S.hql.R1, mode != 0, mode != 0);
      if (tid == 0) S.cnt[4] += idl_flops(m, E.n);
    }
    if (mode == 0) {
      if (tid == 0 && m < 64) {  // small-m IDL patches: gather / estimate sub-phases
        BM_DIAG_ADD(24, (S.t_g[0] - (S.t_mark - S.t_gather)));
        BM_DIAG_ADD(25, (S.t_g[1] - S.t_g[0]));
        BM_DIAG_ADD(26, (S.t_g[2] - S.t_g[1]));
        BM_DIAG_ADD(27, (S.t_g[3] - S.t_g[2]));
        BM_DIAG_ADD(28, (E.t_e[0] - S.t_g[3]));
        BM_DIAG_ADD(29, (E.t_e[1] - E.t_e[0]));
        BM_DIAG_ADD(30, (clock64() - E.t_e[1]));
        BM_DIAG_ADD(31, 1);
      }
      if (tid == 0) {
        BM_DIAG_ADD(16, S.t_pick);
        BM_DIAG_ADD(17, S.t_gather);
        BM_DIAG_ADD(18, (clock64() - S.t_mark));
        S.t_mark = clock64();
        S.idl_diag = 1;
        rec.layer = BM_LAYER_IDL;
        rec.nu = S.nu;
        rec.flags |= BM_REC_HAS_NU;
      }
    } else if (mode == 1) {
      if (run_idl && E.ok) {
        if (tid == 0) {
          rec.layer = BM_LAYER_IDL;
          rec.nu = E.nu_raw;
          rec.flags |= BM_REC_HAS_NU;
        }
      } else {
        brl_values(E);
        if (tid == 0) {
          rec.layer = BM_LAYER_BRL;
          rec.m_candidates = 0;
          rec.flags |= BM_REC_FALLBACK;
        }
      }
    } else {
      if (run_idl && E.ok) {
        done = true;
        if (tid == 0) {
          rec.layer = BM_LAYER_IDL;
          rec.flags |= BM_REC_FALLBACK;
          if (!gated) {
            rec.nu = E.nu_raw;
            rec.flags |= BM_REC_HAS_NU;
          }
        }
      }
      if (!done) {
        brl_values(E);
        if (tid == 0) {
          rec.layer = BM_LAYER_BRL;
          rec.flags |= BM_REC_FALLBACK;
        }
      }
      if (gated && tid == 0) {
        rec.nu = S.nu;
        rec.flags |= BM_REC_HAS_NU;
      }
    }
    __syncthreads();
  }
}

// _write_patch (profiles.py:229-235) of patch p of the cell + its record, on
// warp 0 (write-back, the 8 neighbours' schedule keys, the LOST bitmap rows,
// the record), then one CTA barrier.
__device__ void commit_patch(const KParams& P, CellSmem& S, int p) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    EstSmem& E = S.est;
    const int pr_t = patch_r(p), pc_t = patch_c(p);
    bm_patch_record& rec = S.rec;
    bool lost = false;
    if (tid < 4) {
      const int o = (pr_t + (tid >> 1)) * TS + pc_t + (tid & 1);
      lost = S.st[o] == ST_LO;
      if (lost) {
        S.tile[o] = E.vals[tid];
        S.tile32[o] = (float)E.vals[tid];
        S.st[o] = ST_RE;
      }
    }
    const int wb_lost = __popc(__ballot_sync(FULL, lost));
    __syncwarp();
    if (tid >= 8 && tid < 16) {  // the 8 neighbouring patches gain usable context
      const int k = tid - 8, d = k < 4 ? k : k + 1;  // 3x3 neighbourhood minus the centre
      const int qr = (p >> 3) + d / 3 - 1, qc = (p & 7) + d % 3 - 1;
      if (qr >= 0 && qr < 8 && qc >= 0 && qc < 8) S.pkey[qr * 8 + qc] += wb_lost << 7;
    }
    if (tid < 2) {
      const int r = pr_t + tid;
      uint64_t b = S.lostbits[r];
      b &= ~(3ull << pc_t);
      b |= (uint64_t)(S.st[r * TS + pc_t] == ST_LO) << pc_t;
      b |= (uint64_t)(S.st[r * TS + pc_t + 1] == ST_LO) << (pc_t + 1);
      S.lostbits[r] = b;
    }
    if (tid == 0) {
      if (S.idl_diag) {
        BM_DIAG_ADD(19, (clock64() - S.t_mark));
        S.idl_diag = 0;
      }
      rec.cycles = (uint32_t)(clock64() - S.t_start);
      if (rec.layer >= BM_LAYER_IDL) BM_DIAG_ADD(13 + rec.layer, rec.cycles);
      else BM_DIAG_ADD(21, rec.cycles);
      write_record(P, S, rec);
      S.nrec++;
      S.cnt[rec.layer]++;
      S.progressed = 1;
    }
  }
  __syncthreads();
}

// pick_next_patch (framework.py:243-250) + extract_target (framework.py:151-168)
// by warp 0.  Returns via S.pick / S.skip.
// Schedule key of patch p (patch_scores, framework.py:230-240): AVAILABLE
// count, then usable (not LOST) count over the 32 context offsets, then raster
// order; from the row bitmaps (6 window rows of 6 bits, patch cells masked out;
// out-of-image positions are LOST).  Computed for the 64 patches at cell start;
// a write-back only raises the usable counts of the 8 neighbouring patches
// (every neighbour's window covers the whole written patch; AVAILABLE pixels
// never change), so the keys are maintained incrementally (commit of a patch).
__device__ __forceinline__ int patch_key(const CellSmem& S, int p) {
  const int pr = patch_r(p), pc = patch_c(p);
  int av = 0, us = 0;
#pragma unroll
  for (int q = 0; q < 6; q++) {
    const unsigned m6 = (q == 2 || q == 3) ? 0x33u : 0x3Fu;
    const unsigned lb = (unsigned)(S.lostbits[pr - 2 + q] >> (pc - 2)) & m6;
    const unsigned ab = (unsigned)(S.availbits[pr - 2 + q] >> (pc - 2)) & m6;
    us += __popc(m6 & ~lb);
    av += __popc(ab);
  }
  return (av << 13) | (us << 7) | (63 - p);
}

__device__ void pick_and_extract(CellSmem& S) {
  const int lane = threadIdx.x & 31;
  EstSmem& E = S.est;
  const unsigned long long pend = S.pend;
  // pick_next_patch (framework.py:243-250): the pending patch with the largest
  // schedule key (patch_key, maintained as patches are written back)
  int best_key = -1;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int p = lane + 32 * h;
    if ((pend >> p) & 1ull) best_key = max(best_key, S.pkey[p]);
  }
  best_key = __reduce_max_sync(FULL, (unsigned)(best_key + 1)) - 1;
  const int p = 63 - (best_key & 127);
  // extract target
  const int pr = patch_r(p), pc = patch_c(p);
  const int o = (pr - 2 + ctx_r(lane)) * TS + pc - 2 + ctx_c(lane);
  const bool usable = S.st[o] != ST_LO;
  const unsigned bal = __ballot_sync(FULL, usable);
  const int n = __popc(bal);
  if (usable) {
    const int idx = __popc(bal & ((1u << lane) - 1));
    E.y0[idx] = S.tile[o];
    E.y0f[idx] = S.tile32[o];
    E.uoff[idx] = (int16_t)(ctx_r(lane) * TS + ctx_c(lane));
  }
  // row masks of used window positions (usable context + patch cells) from
  // the usable ballot: context offsets 0-5 / 6-11 are window rows 0 / 1
  // (cols 0-5), 12-15 / 16-19 rows 2 / 3 (cols 0, 1, 4, 5; the patch cells 2,
  // 3 are always used), 20-25 / 26-31 rows 4 / 5 (CONTEXT_OFFSETS, framework.py:33-36)
  if (lane < 6) {
    const int sh = lane < 2 ? 6 * lane : (lane < 4 ? 12 + 4 * (lane - 2) : 20 + 6 * (lane - 4));
    const unsigned b = bal >> sh;
    S.rowmask[lane] = (lane == 2 || lane == 3) ? ((b & 3u) | ((b & 0xCu) << 2) | 0xCu) : (b & 0x3Fu);
  }
  if (lane < 4) E.uoff[n + lane] = (int16_t)((2 + (lane >> 1)) * TS + 2 + (lane & 1));
  // flatness (profiles.py:98-102): exact max / min of y0 by redux on
  // order-preserving 64-bit keys (hi word, then lo word)
  const double yv = usable ? S.tile[o] : 0.0;
  const unsigned long long ub = (unsigned long long)__double_as_longlong(yv);
  const unsigned long long key = (ub >> 63) ? ~ub : (ub | 0x8000000000000000ull);
  const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
  const unsigned mxh = __reduce_max_sync(FULL, usable ? khi : 0u);
  const unsigned mxl = __reduce_max_sync(FULL, usable && khi == mxh ? klo : 0u);
  const unsigned mnh = __reduce_min_sync(FULL, usable ? khi : 0xFFFFFFFFu);
  const unsigned mnl = __reduce_min_sync(FULL, usable && khi == mnh ? klo : 0xFFFFFFFFu);
  auto unkey = [](unsigned h, unsigned l) {
    const unsigned long long k = ((unsigned long long)h << 32) | l;
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
  };
  const double ymax = unkey(mxh, mxl), ymin = unkey(mnh, mnl);
  __syncwarp();
  if (lane == 0) {
    S.pick = p;
    S.pend = pend & ~(1ull << p);
    E.n = n;
    S.skip = n == 0;
    S.phi = ymax - ymin;
  }
}

#ifndef BM_CONCEAL_ONLY  // the library-API kernels: the 256-thread translation unit only
// A TargetContext supplied by the caller (the per-patch library API,
// framework.py:60-77): usable bits over CONTEXT_OFFSETS and y0 in layout
// order, instead of pick_and_extract's extraction.  Warp 0.
__device__ void set_target(CellSmem& S, unsigned layout, const double* __restrict__ y0g) {
  const int lane = threadIdx.x & 31;
  EstSmem& E = S.est;
  const bool usable = (layout >> lane) & 1u;
  const int n = __popc(layout);
  double yv = 0.0;
  if (usable) {
    const int idx = __popc(layout & ((1u << lane) - 1));
    yv = y0g[idx];
    E.y0[idx] = yv;
    E.y0f[idx] = (float)yv;
    E.uoff[idx] = (int16_t)(ctx_r(lane) * TS + ctx_c(lane));
  }
  if (lane < 6) {  // window row masks (see pick_and_extract)
    const int sh = lane < 2 ? 6 * lane : (lane < 4 ? 12 + 4 * (lane - 2) : 20 + 6 * (lane - 4));
    const unsigned b = layout >> sh;
    S.rowmask[lane] = (lane == 2 || lane == 3) ? ((b & 3u) | ((b & 0xCu) << 2) | 0xCu) : (b & 0x3Fu);
  }
  if (lane < 4) E.uoff[n + lane] = (int16_t)((2 + (lane >> 1)) * TS + 2 + (lane & 1));
  const double ymax = warp_max(usable ? yv : -INFINITY), ymin = warp_min(usable ? yv : INFINITY);
  __syncwarp();
  if (lane == 0) {
    E.n = n;
    S.skip = n == 0;
    S.phi = ymax - ymin;  // flatness (profiles.py:98-102)
  }
}

// select_and_estimate (profiles.py:105-133), or _forced_estimate
// (profiles.py:141-171) with P.forced >= 0, for independent patches of one
// working image (P.pixels f64 [H,W], P.states): one CTA per patch, the same
// device code as the fused kernel's patch step, no write-back.  The caller's
// TargetContext (layout bits, y0) defines the context.
struct SelectArgs {
  int count;
  const int32_t* origins;   // [count][2] patch origins (absolute)
  const uint32_t* layouts;  // [count]
  const double* y0;         // [count][32]
  double* out_values;       // [count][4]
  bm_patch_record* out_rec; // [count]
};

__global__ void __launch_bounds__(NT, 1) k_select(KParams P, SelectArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CellSmem& S = *reinterpret_cast<CellSmem*>(smem_raw);
  const int tid = threadIdx.x, i = blockIdx.x;
  if (i >= A.count) return;
  if (tid < 8) S.cnt[tid] = 0;
  init_exptab(S.est);
  const int pr = A.origins[2 * i], pc = A.origins[2 * i + 1];
  if (tid == 0) {
    S.f = 0;
    S.gr = pr / BS;  // block_origin_of (framework.py:114-116)
    S.gc = pc / BS;
    S.slot = 0;
    S.nrec = 0;
    S.idl_diag = 0;
    S.t_start = clock64();
  }
  __syncthreads();
  load_tile(P, S);
  const int pr_t = pr - (S.gr * BS - BS), pc_t = pc - (S.gc * BS - BS);
  if (tid < 32) set_target(S, A.layouts[i], A.y0 + (size_t)i * 32);
  __syncthreads();
  estimate_only(P, S, pr_t, pc_t, nullptr);
  if (tid == 0) {
    S.rec.cycles = (uint32_t)(clock64() - S.t_start);
    A.out_rec[i] = S.rec;
    for (int q = 0; q < 4; q++) A.out_values[(size_t)i * 4 + q] = S.est.vals[q];
  }
}

#endif  // BM_CONCEAL_ONLY

__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) k_conceal(KParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CellSmem& S = *reinterpret_cast<CellSmem*>(smem_raw);
  const int tid = threadIdx.x;
  double* gS = P.scratch + (size_t)blockIdx.x * P.scratch_per_cta;
  if (tid < 8) S.cnt[tid] = 0;
  init_exptab(S.est);
  if (tid == 0) S.idl_diag = 0;
  const int nslots = *((volatile int*)P.nslots);
  // Build choice (identical in every CTA of the three launched builds): by
  // the dependency DAG's average width W = lost cells / levels against each
  // build's concurrent cells (256-thread: 2 per SM, 512-thread: 1 per SM,
  // cluster: 1 per 2 SMs) and the workload's weight.  Narrow DAGs are
  // latency-bound on their critical path, where fewer, faster cell workers
  // win; all-HQL work is heavy enough to stay throughput-bound at smaller W.
  // Thresholds measured on cfg1-cfg5 and cfg5 shards of 16..256 frames
  // (profiles/scale_sim_r02.txt).
  {
    const double levels = (double)(P.counters[7] + 1);
    const double w = (double)nslots / levels * (148.0 / (double)P.sms);
    const bool all_hql = P.forced == BM_LAYER_HQL || (P.forced < 0 && P.t_phi < 0.0 && isinf(P.t_nu));
    const bool gated = P.forced < 0 && !all_hql;
    const double w_cluster = gated ? 450.0 : 96.0, w_512 = gated ? 1000.0 : 192.0;
    int want = w <= w_cluster ? (P.narrow_cluster ? BUILD_CLUSTER : 512) : (w <= w_512 ? 512 : 256);
    if (P.build) want = P.build;
    const int mine = NT <= 256 ? 256 : (CS > 1 ? BUILD_CLUSTER : 512);
    if (mine != want) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) P.counters[6] = (unsigned long long)mine;  // the build that ran
  }
  const unsigned crank = cluster_rank();
  const long long t_cta0 = clock64();
  for (;;) {
    const long long t_w0 = clock64();
    if (crank == 0 && tid < 32) {
      const int slot = sched_pop(P, nslots);
      if (tid == 0) S.slot = slot;
    }
    if constexpr (CS > 1) {
      // rank 0 pops; the cluster's other CTAs take the same cell (the acquire
      // chain: rank 0's queue acquire, then the cluster barrier's)
      cluster_sync_all();
      if (crank != 0 && tid == 0) S.slot = ld_dsmem_s32(map_rank(&S.slot, 0));
      cluster_sync_all();  // rank 0 pops again only after every peer has read
    } else {
      __syncthreads();
    }
    if (S.slot < 0) break;
    if (tid == 0) {
      const int slot = S.slot;
      const int c = P.slot_cell[slot];
      S.f = c / (P.GR * P.GC);
      const int rem = c % (P.GR * P.GC);
      S.gr = rem / P.GC;
      S.gc = rem % P.GC;
    }
    __syncthreads();
    if (tid == 0) BM_DIAG_ADD(20, (clock64() - t_w0));  // scheduling wait
    const long long t_lt = clock64();
    load_tile(P, S);
    if (tid == 0) {  // the staging (gather) stage: cycles, cells, finished-neighbour buffers read (diagnostic)
      BM_DIAG_ADD(40, (clock64() - t_lt));
      BM_DIAG_ADD(41, 1);
#if BM_DIAG
      int nb = 0, ps;
      for (int q = 0; q < 4; q++) nb += cell_lost(P, S.f, S.gr - 1 + (q < 3 ? 0 : 1), S.gc - 1 + (q < 3 ? q : 0), ps);
      BM_DIAG_ADD(42, nb);
#endif
    }
    // lost_patch_origins (framework.py:219-227)
    if (tid < 32) {
      unsigned long long bits = 0;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int p = tid + 32 * h;
        const int o = patch_r(p) * TS + patch_c(p);
        const bool l = S.st[o] == ST_LO || S.st[o + 1] == ST_LO || S.st[o + TS] == ST_LO || S.st[o + TS + 1] == ST_LO;
        const unsigned b = __ballot_sync(FULL, l);
        bits |= (unsigned long long)b << (32 * h);
        S.pkey[p] = patch_key(S, p);
      }
      // later-raster lost 8-neighbours read this cell's values from cellbuf;
      // with none, the FP64 publish is skipped (DRAM writes)
      int ps;
      const int dr = tid == 0 ? 0 : 1, dc = tid == 0 ? 1 : tid - 2;
      const unsigned rd = __ballot_sync(FULL, tid < 4 && cell_lost(P, S.f, S.gr + dr, S.gc + dc, ps));
      if (tid == 0) {
        S.remaining = bits;
        S.nrec = 0;
        S.readers = rd != 0u;
      }
    }
    __syncthreads();
    // _conceal_block (profiles.py:191-226)
    while (S.remaining) {
      if (tid == 0) {
        S.ndef = 0;
        S.progressed = 0;
        S.pend = S.remaining;
      }
      __syncthreads();
      while (S.pend) {
        if (tid == 0) S.t_start = clock64();
        if (tid < 32) pick_and_extract(S);
        __syncthreads();
        if (S.skip) {  // EmptyContextError -> deferred
          if (tid == 0) S.deferred[S.ndef++] = S.pick;
          __syncthreads();
          continue;
        }
        estimate_only(P, S, patch_r(S.pick), patch_c(S.pick), gS);
        commit_patch(P, S, S.pick);  // ends with a CTA barrier
      }
      if (S.ndef == 0) break;
      if (S.progressed) {
        __syncthreads();
        if (tid == 0) {
          unsigned long long b = 0;
          for (int i = 0; i < S.ndef; i++) b |= 1ull << S.deferred[i];
          S.remaining = b;
        }
        __syncthreads();
      } else {
        // 128 fill in deferral order (profiles.py:219-225)
        if (tid == 0) {
          for (int i = 0; i < S.ndef; i++) {
            const int p = S.deferred[i];
            const int pr_t = patch_r(p), pc_t = patch_c(p);
            for (int q = 0; q < 4; q++) {
              const int o = (pr_t + (q >> 1)) * TS + pc_t + (q & 1);
              if (S.st[o] == ST_LO) {
                S.tile[o] = 128.0;
                S.tile32[o] = 128.f;
                S.st[o] = ST_RE;
              }
            }
            bm_patch_record rec;
            memset(&rec, 0, sizeof(rec));
            rec.frame = S.f;
            rec.row = S.gr * BS - BS + pr_t;
            rec.col = S.gc * BS - BS + pc_t;
            rec.layer = BM_LAYER_NONE;
            rec.flags = BM_REC_DEFERRED;
            rec.m_candidates = -1;
            rec.phi = rec.nu = rec.beta = rec.alpha = __longlong_as_double(0x7ff8000000000000ll);
            rec.beta_gap = __int_as_float(0x7fc00000);
            write_record(P, S, rec);
            S.nrec++;
            S.cnt[3]++;
          }
          S.remaining = 0;
        }
        __syncthreads();
        break;
      }
    }
    __syncthreads();
    // publish the cell (values, outputs), then release the flag (cluster
    // build: rank 0; the other CTAs hold the same values)
    if (crank == 0) {
      const size_t slot = S.slot;
      const int f = S.f;
      const int r0 = S.gr * BS, c0 = S.gc * BS;
      for (int i = tid; i < 256; i += NT) {
        const int rr = i / BS, cc = i % BS;
        const double v = S.tile[(BS + rr) * TS + BS + cc];
        if (S.readers) P.cellbuf[slot * 256 + i] = v;
        const size_t o = ((size_t)f * P.H + r0 + rr) * P.W + c0 + cc;
        if (P.out_f64) P.out_f64[o] = v;
        if (P.out_u8) P.out_u8[o] = (uint8_t)floor(fmin(fmax(v, 0.0), 255.0) + 0.5);  // image.py:53-56
      }
      if (tid == 0 && P.records) P.rec_count[slot] = (uint8_t)S.nrec;
      __threadfence();
      __syncthreads();
      // release the later-raster lost 8-neighbours; the last predecessor of a
      // cell pushes it to its ready FIFO (acq_rel chain: its data is visible
      // to whoever pops it)
      if (tid < 4) {
        const int dr[4] = {0, 1, 1, 1}, dc[4] = {1, -1, 0, 1};
        int ps;
        if (cell_lost(P, f, S.gr + dr[tid], S.gc + dc[tid], ps) && atom_dec_acq_rel(&P.indeg[ps]) == 1u) {
          const unsigned b = P.bucket[ps];
          const unsigned t = atomicAdd(&P.sched[SCHED_TAIL + b], 1u);
          st_release_u32(&P.queue[P.sched[SCHED_BOFF + b] + t], (unsigned)ps);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    BM_DIAG_ADD(22, (clock64() - t_cta0));  // CTA lifetime
    BM_DIAG_ADD(23, 1);
  }
  if (crank == 0) {  // (cluster build: every CTA counted the same cells)
    if (tid < 4 && S.cnt[tid]) atomicAdd(&P.counters[tid], S.cnt[tid]);
    if (tid >= 4 && tid < 8 && S.cnt[tid]) atomicAdd(&P.counters[tid + 4], S.cnt[tid]);
  }
}

// Dense output initialisation: out_f64 = pixels, out_u8 = quantized(pixels).
__global__ void k_init_out(KParams P) {
  const size_t n = (size_t)P.B * P.H * P.W;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double v = P.pix_f64 ? ((const double*)P.pixels)[i] : (double)((const uint8_t*)P.pixels)[i];
    if (P.out_f64) P.out_f64[i] = v;
    if (P.out_u8) P.out_u8[i] = (uint8_t)floor(fmin(fmax(v, 0.0), 255.0) + 0.5);
  }
}

__global__ void k_summary(KParams P, bm_summary* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    bm_summary s;
    memset(&s, 0, sizeof(s));
    s.lost_cells = *P.nslots;
    for (int i = 0; i < 3; i++) s.layer_counts[i] = (int64_t)P.counters[i];
    s.deferred_fills = (int64_t)P.counters[3];
    s.patches = s.layer_counts[0] + s.layer_counts[1] + s.layer_counts[2] + s.deferred_fills;
    s.lost_left = (int64_t)P.counters[4];
    s.max_level = (int32_t)P.counters[7];
    s.bad_states = (int32_t)P.counters[5];
    s.flop64 = (int64_t)P.counters[8];
    s.flop32 = (int64_t)P.counters[9];
    s.hql_patches = (int64_t)P.counters[10];
    s.gate_candidates = (int64_t)P.counters[11];
    s.kernel_build = (int32_t)P.counters[6];
    *out = s;
  }
}

// ------------------------------------------------------- dense estimator API
#ifndef BM_CONCEAL_ONLY

struct EstBatchArgs {
  int layer, count, max_m;
  double sigma2;
  const int32_t* n_y;
  const int32_t* m;
  const double* y0;
  const double* x;
  const double* y;
  double* out_values;
  bm_patch_record* out_info;
  double* scratch;
};

struct EstBatchSmem {
  double dbuf[MAXCAND];
  EstSmem est;
  HqlSmem hql;
  HqlOut hout;
};

__global__ void __launch_bounds__(NT, 1) k_estimate_batch(EstBatchArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EstBatchSmem& S = *reinterpret_cast<EstBatchSmem*>(smem_raw);
  EstSmem& E = S.est;
  const int i = blockIdx.x, tid = threadIdx.x;
  const int n = A.n_y[i], m = A.m[i];
  const double* X = A.x + (size_t)i * A.max_m * 4;
  const double* Y = A.y + (size_t)i * A.max_m * 32;
  double* gs = A.scratch + (size_t)blockIdx.x * HQL_SCRATCH_DENSE;
  init_exptab(E);
  if (tid < 32) {
    E.y0[tid] = tid < n ? A.y0[(size_t)i * 32 + tid] : 0.0;
    E.y0f[tid] = (float)E.y0[tid];
  }
  if (tid == 0) E.n = n;
  // dense Z [m][40]: y | x | 1 (the HQL column convention)
  double* Z = gs + HQL_Z;
  for (int o = tid; o < m * 40; o += NT) {
    const int j = o / 40, c = o % 40;
    Z[o] = c < n ? Y[(size_t)j * 32 + c] : (c >= 32 && c < 36 ? X[(size_t)j * 4 + c - 32] : (c == 36 ? 1.0 : 0.0));
  }
  hql_columns(S.hql, n, nullptr);
  __syncthreads();
  DenseAcc acc{X, Y};
  bm_patch_record rec;
  memset(&rec, 0, sizeof(rec));
  rec.nu = rec.beta = rec.alpha = __longlong_as_double(0x7ff8000000000000ll);
  rec.m_candidates = m;
  rec.n_y = (uint8_t)n;
  rec.flags = BM_REC_HAS_M;
  int layer = BM_LAYER_BRL, fallback = 0;
  bool done = false;
  if (A.layer == BM_LAYER_HQL && m >= 2) {
    DenseLoader zv{Z};
    hql_mma(zv, m, n, E.y0, S.hql, gs, S.hout, E.exptab, S.dbuf);
    __syncthreads();
    if (S.hout.ok) {
      done = true;
      layer = BM_LAYER_HQL;
      rec.beta = S.hout.beta;
      rec.alpha = S.hout.alpha;
      rec.beta_gap = S.hout.gap;
      rec.flags |= BM_REC_HAS_BW;
      if (tid == 0)
        for (int q = 0; q < 4; q++) E.vals[q] = S.hout.vals[q];
    }
  }
  if (!done && A.layer != BM_LAYER_BRL && m >= 1) {
    idl_estimate_dev(acc, m, A.sigma2, E, S.hql.R1, true);
    rec.nu = E.nu_raw;
    rec.flags |= BM_REC_HAS_NU;
    if (E.ok) {
      done = true;
      layer = BM_LAYER_IDL;
      fallback = A.layer == BM_LAYER_HQL;
    }
  }
  if (!done) {
    brl_values(E);
    fallback = A.layer != BM_LAYER_BRL;
    if (A.layer != BM_LAYER_HQL) rec.m_candidates = 0;
  }
  __syncthreads();
  if (tid == 0) {
    rec.layer = (int8_t)layer;
    if (fallback) rec.flags |= BM_REC_FALLBACK;
    A.out_info[i] = rec;
    for (int q = 0; q < 4; q++) A.out_values[(size_t)i * 4 + q] = E.vals[q];
  }
}

#endif  // BM_CONCEAL_ONLY

__global__ void k_compact_records(const bm_patch_record* slot_rec, const uint8_t* cnt, const int* excl,
                                  const int* nslots, bm_patch_record* out) {
  const int ns = *nslots;
  for (int s = blockIdx.x; s < ns; s += gridDim.x) {
    const int c = cnt[s], base = excl[s];
    for (int i = threadIdx.x; i < c; i += blockDim.x) out[base + i] = slot_rec[(size_t)s * 64 + i];
  }
}
__global__ void k_u8_to_int(const uint8_t* c, const int* nslots, int* o, int n) {
  const int ns = *nslots;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = i < ns ? c[i] : 0;
}

}  // namespace BM_NS
