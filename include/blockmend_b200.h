/*
 * blockmend_b200.h — C ABI of the B200-native concealment hot path.
 *
 * This is the drop-in boundary for the reference package `blockmend`
 * (/root/reference/pkg/src/blockmend).  The reference is pure Python, so the
 * "FFI a maintainer would bind" is ctypes; INTEGRATION.md shows the stub.
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - All pointers passed to bm_conceal / bm_estimate_batch are DEVICE pointers
 *    (caller-owned, e.g. torch tensors' data_ptr()); the stream is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - bm_conceal_host takes HOST pointers and does the host<->device copies
 *    itself (pinned staging), i.e. the call a non-torch user makes.
 *  - Status codes map onto the reference's exceptions (errors.py:4-25,
 *    image.py:122-124, profiles.py:305); see bm_status_string().
 *  - No CPU fallback: every compute entry point launches sm_100a kernels and
 *    fails with BM_ERR_CUDA when no device is present.
 */
#ifndef BLOCKMEND_B200_H
#define BLOCKMEND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 1

/* status codes */
#define BM_OK 0
#define BM_ERR_ARGS 1       /* bad shape / argument  -> ValueError / DimensionMismatchError (image.py:122-124) */
#define BM_ERR_LOST_LEFT 2  /* LOST pixels outside the 16x16 block grid remain -> AssertionError (profiles.py:305) */
#define BM_ERR_CUDA 3       /* CUDA runtime error / no device */
#define BM_ERR_WORKSPACE 4  /* workspace too small */
#define BM_ERR_STATES 5     /* a state value > 2 -> ValueError (image.py:69-70) */

/* layers (estimators.py:39-42); -1 = deferred mid-gray fill (profiles.py:215-225) */
#define BM_LAYER_NONE (-1)
#define BM_LAYER_BRL 0
#define BM_LAYER_IDL 1
#define BM_LAYER_HQL 2

/* pixel dtypes of the input frames */
#define BM_PIX_U8 0
#define BM_PIX_F64 1

/* bm_patch_record.flags */
#define BM_REC_FALLBACK 1u  /* LayerDecision.fallback      (profiles.py:90) */
#define BM_REC_DEFERRED 2u  /* LayerDecision.deferred_fill (profiles.py:91) */
#define BM_REC_HAS_NU 4u    /* LayerDecision.nu is not None */
#define BM_REC_HAS_PHI 8u   /* LayerDecision.phi is not None */
#define BM_REC_HAS_BW 16u   /* LayerDecision.beta/alpha are not None (HQL) */
#define BM_REC_HAS_M 32u    /* LayerDecision.m_candidates is not None */

/* Run parameters: Profile (profiles.py:49-78) + conceal_image keywords
 * (profiles.py:263-271). */
typedef struct bm_params {
  int32_t frames;       /* B: frames in the batch (conceal_image is B = 1) */
  int32_t height;       /* H */
  int32_t width;        /* W */
  int32_t pixel_dtype;  /* BM_PIX_U8 or BM_PIX_F64 */
  double t_phi;         /* Profile.t_phi */
  double t_nu;          /* Profile.t_nu (may be +inf: sentinel) */
  double sigma2;        /* DEFAULT_SIGMA2 = 10 (estimators.py:31) */
  int32_t forced_layer; /* -1 = gated (select_and_estimate), else BM_LAYER_* (_forced_estimate) */
  int32_t flags;        /* BM_FLAG_* (0 = defaults) */
} bm_params;

/* One LayerDecision (profiles.py:81-95) in the reference's order
 * (lost cell raster order, then schedule/deferral order). 64 bytes. */
typedef struct bm_patch_record {
  int32_t frame;
  int32_t row, col;     /* patch_origin */
  int8_t layer;         /* BM_LAYER_* ; -1 for a deferred fill */
  uint8_t flags;        /* BM_REC_* */
  uint8_t n_y;          /* usable context count N_y (0 for deferred fills) */
  uint8_t rings_used;   /* LayerDecision.rings_used */
  int32_t m_candidates; /* valid if BM_REC_HAS_M */
  uint32_t cycles;      /* SM clock cycles spent on the patch (-> elapsed_s) */
  float beta_gap;       /* HQL: min over the other grid betas of |eps_g - eps_best|, in units of
                           the eps change a 1e-11 relative perturbation of y0 can cause
                           (2 sqrt(eps_best N_y) dy + N_y dy^2, dy = 1e-11 max|y0|); < 1 means
                           the choice was decided at rounding level (tests/parity.py) */
  uint32_t pad;
  double phi, nu, beta, alpha;
} bm_patch_record;

/* Per-batch summary (ConcealmentReport counts, metrics.py:21-43). */
typedef struct bm_summary {
  int64_t lost_cells;     /* lost 16x16 cells concealed (the throughput unit) */
  int64_t patches;        /* records produced (incl. deferred fills) */
  int64_t layer_counts[3];/* BRL, IDL, HQL (fallbacks counted under the layer used, profiles.py:309-314) */
  int64_t deferred_fills;
  int64_t lost_left;      /* LOST pixels outside the block grid (must be 0) */
  int32_t max_level;      /* depth of the cross-cell dependency DAG */
  int32_t bad_states;     /* cells/pixels with a state value > 2 */
  /* algorithmic work (SURVEY.md §8(d) formulas, counted per patch) */
  int64_t flop64;         /* FP64: HQL pipeline + IDL estimate */
  int64_t flop32;         /* FP32: nu-gate distance/weight screening */
  int64_t hql_patches;    /* patches that ran the full HQL pipeline */
  int64_t gate_candidates;/* candidates screened by the FP32 nu gate */
  int32_t kernel_build;   /* the concealment build that ran: 256, 512 or 1024 (2-CTA clusters); 0 = none */
  int32_t reserved;
} bm_summary;

/* bm_params.flags */
#define BM_FLAG_TIME_KERNEL 1 /* time the concealment kernel with CUDA events (bm_last_kernel_ms) */
/* Kernel build (default: by the shape of the cross-cell dependency DAG): the
 * 256-thread CTAs (2 cells per SM) or the 512-thread CTAs (1 cell per SM).
 * Both meet the parity bar; their FP64 reduction orders differ, so results
 * can differ in the last bits between builds (tests, A/B). */
#define BM_FLAG_BUILD_256 2
#define BM_FLAG_BUILD_512 4
/* the cluster build: 2-CTA thread-block clusters of 512 threads per cell, the
 * HQL candidate loops split across the two SMs over distributed shared memory */
#define BM_FLAG_BUILD_CLUSTER 8
/* narrow DAGs (default choice): the 512-thread build instead of the cluster build */
#define BM_FLAG_NARROW_512 16

/* ---- queries ---- */
int bm_abi_version(void);
const char* bm_status_string(int status);
/* bytes of device workspace bm_conceal needs for these params */
size_t bm_workspace_bytes(const bm_params* p);
/* upper bound on records (64 per 16x16 cell of the grid) */
int64_t bm_max_records(const bm_params* p);
/* Durations (ms) of the concealment kernels launched with BM_FLAG_TIME_KERNEL
 * since the last reset (CUDA events recorded on the launch stream around each
 * launch; up to 256 kept).  Synchronises on the events.  Returns the count. */
int bm_kernel_times_ms(float* out, int cap);
void bm_kernel_times_reset(void);
/* Diagnostics: 48 cumulative SM-cycle counters (HQL phases, IDL patch
 * phases, scheduling; filled only by -DBM_DIAG=1 builds); names in
 * _native.PHASES. */
int bm_debug_phase_cycles(unsigned long long* out48, int reset);
/* ---- callers either side of the path ---------- */

/* Batched squared-error sums for PSNR (metrics.py:50-75): per frame,
 * out_sum[f] = sum over selected pixels of (ref - test)^2 (FP64) and
 * out_count[f] = number of selected pixels; select = NULL selects all (psnr),
 * else a u8 [B,H,W] 0/1 selection (psnr_masked, e.g. the originally lost set).
 * Device pointers; PSNR = 10 log10(255^2 / (sum / count)) on the host. */
int bm_sqdiff_batch(const void* ref, const void* test, int pixel_dtype, const uint8_t* select, int frames,
                    int height, int width, double* out_sum, double* out_count, void* stream);
/* Batched mean SSIM (metrics.py:86-116): 11x11 Gaussian window (sigma 1.5),
 * K1 0.01, K2 0.03, L 255, windows fully inside the frame, FP64.
 * out_mean[f] (device).  BM_ERR_ARGS when a side is < 11 (ValueError). */
int bm_ssim_batch(const void* ref, const void* test, int pixel_dtype, int frames, int height, int width,
                  double* out_mean, void* stream);
/* Loss-pattern generation on the device (loss.py:24-77), bit-identical to the
 * reference generators: writes PixelState values (0 AVAILABLE, 1 LOST) into
 * out_states [B,H,W].  BM_MASK_DISPERSED: blocks with odd row and odd column
 * (gen_dispersed_mask); BM_MASK_RANDOM: exactly `count` blocks, the first
 * `count` of a SplitMix64(seeds[f]) Fisher-Yates shuffle of the block indices
 * (gen_random_mask with count = round_half_up(rate * blocks)); BM_MASK_SLICE:
 * `count` whole block rows, the first of a Fisher-Yates shuffle of the rows
 * (the BASELINE slice-loss pattern).  seeds: device u64 [B]. */
#define BM_MASK_DISPERSED 0
#define BM_MASK_RANDOM 1
#define BM_MASK_SLICE 2
int bm_gen_masks(int kind, int frames, int height, int width, int block_size, int count, const uint64_t* seeds,
                 uint8_t* out_states, void* stream);

/* SM clock of the current device in kHz (converts bm_patch_record.cycles to
 * seconds for ConcealmentReport.patch_times); 0 when no device. */
int bm_device_clock_khz(void);

/*
 * bm_conceal — replaces blockmend.conceal_image (profiles.py:263-323) for a
 * batch of B frames: _lost_block_ids + the raster-order _conceal_block loop
 * (profiles.py:238-302), select_and_estimate / _forced_estimate per patch
 * (profiles.py:105-171), and ImageBuffer.quantized (image.py:53-56).
 *
 *   pixels      [B,H,W] u8 or f64 (device)            ImageBuffer.pixels
 *   states      [B,H,W] u8 {0,1,2} (device)           LossMask.states
 *   out_f64     [B,H,W] f64 or NULL                   returned ImageBuffer.pixels
 *   out_u8      [B,H,W] u8  or NULL                   ImageBuffer.quantized()
 *   out_records [bm_max_records] or NULL              report.decisions (slot layout,
 *                                                     compact with bm_compact_records)
 *   out_summary device bm_summary* or NULL
 *   workspace   device, >= bm_workspace_bytes(p)
 * Inputs are never modified.  Asynchronous on `stream`; returns BM_OK once
 * enqueued (argument errors are reported synchronously).
 */
int bm_conceal(const bm_params* p, const void* pixels, const uint8_t* states,
               double* out_f64, uint8_t* out_u8, bm_patch_record* out_records,
               bm_summary* out_summary, void* workspace, size_t workspace_bytes,
               void* stream);

/*
 * bm_compact_records — gathers the slot-layout records written by bm_conceal
 * into the reference's decision order (device -> device).  Returns the count
 * in *out_count (host).  Synchronises `stream`.
 */
int bm_compact_records(const bm_params* p, const bm_patch_record* slot_records,
                       void* workspace, bm_patch_record* out_records,
                       int64_t* out_count, void* stream);

/*
 * bm_conceal_host — the same call with HOST buffers: copies pixels/states to
 * the device, runs bm_conceal, copies the u8 (and optionally f64) result and
 * the summary back.  Device buffers are cached across calls per (B,H,W).
 * out_records (host) may be NULL; when given it receives *out_nrec compacted
 * records (capacity bm_max_records).
 */
int bm_conceal_host(const bm_params* p, const void* pixels, const uint8_t* states,
                    double* out_f64, uint8_t* out_u8, bm_patch_record* out_records,
                    int64_t* out_nrec, bm_summary* out_summary);

/*
 * bm_estimate_batch — per-instance estimator entry (device pointers):
 * brl_estimate / idl_estimate / hql_estimate (estimators.py:96-132, 248-286)
 * on `count` independent (target, candidate set) instances in dense layout.
 *   layer       BM_LAYER_BRL / IDL / HQL (HQL includes its IDL->BRL ladder)
 *   n_y[i]      context length of instance i (1..32)
 *   m[i]        candidate count of instance i (0..max_m)
 *   y0          [count][32]        target context (first n_y used)
 *   x           [count][max_m][4]  candidate patch values
 *   y           [count][max_m][32] candidate contexts (first n_y used)
 *   out_values  [count][4]
 *   out_info    [count] records: layer, flags (fallback), m, nu (IDL raw_sum), beta, alpha
 */
int bm_estimate_batch(int32_t layer, int32_t count, int32_t max_m, double sigma2,
                      const int32_t* n_y, const int32_t* m, const double* y0,
                      const double* x, const double* y, double* out_values,
                      bm_patch_record* out_info, void* stream);

/* ---- the per-patch library API (blockmend/__init__.py:17-58) ------------
 * Device entry points behind the reference's framework / estimator / profile
 * functions that a library user (or the reference's own unit tests) calls
 * one patch at a time.  Device pointers, one working image [H,W] (FP64
 * pixels, u8 PixelState states), asynchronous on `stream`. */

/* select_and_estimate (profiles.py:105-133) — or _forced_estimate
 * (profiles.py:141-171) when p->forced_layer >= 0 — for `count` independent
 * patches of the working image (p->frames = 1, p->pixel_dtype = BM_PIX_F64):
 * the fused kernel's patch step (gate, ring gather with the nu loop, IDL /
 * HQL with the ladder), no write-back.  The caller's TargetContext per patch:
 * origins [count][2], layouts [count] (bit k = CONTEXT_OFFSETS[k] usable,
 * framework.py:33-36), y0 [count][32] (layout order).  Outputs: values
 * [count][4] and one bm_patch_record per patch (layer, phi, nu, rings,
 * m_candidates, beta, alpha, fallback). */
int bm_select_and_estimate(const bm_params* p, const double* pixels, const uint8_t* states, int32_t count,
                           const int32_t* origins, const uint32_t* layouts, const double* y0,
                           double* out_values, bm_patch_record* out_records, void* stream);

/* extract_target (framework.py:151-168) for `count` patch origins:
 * out_layouts [count], out_n_y [count], out_y0 [count][32]. */
int bm_extract_targets(int height, int width, const double* pixels, const uint8_t* states, int32_t count,
                       const int32_t* origins, uint32_t* out_layouts, int32_t* out_n_y, double* out_y0,
                       void* stream);

/* _collect (framework.py:171-183), the masked gather under gather_candidates
 * / expand_support (framework.py:186-207): request q screens the window
 * origins [offsets[q], offsets[q] + counts[q]) of `origins` ([.][2]) with
 * layout layouts[q] and writes its admissible candidates, in list order, at
 * the same offsets of out_x [.][4] and out_y [.][32]; out_m[q] = their count. */
int bm_collect(int height, int width, const double* pixels, const uint8_t* states, int32_t requests,
               const int32_t* origins, const int32_t* offsets, const int32_t* counts, const uint32_t* layouts,
               double* out_x, double* out_y, int32_t* out_m, void* stream);

/* patch_scores (framework.py:230-240): AVAILABLE / usable context counts. */
int bm_patch_scores(int height, int width, const uint8_t* states, int32_t count, const int32_t* origins,
                    int32_t* out_avail, int32_t* out_usable, void* stream);

/* build_schedule (framework.py:253-274) for `count` blocks (block ids
 * [count][2]): out_n [count] jobs, out_origins [count][64][2],
 * out_reliability [count][64], in filling order. */
int bm_build_schedule(int height, int width, const uint8_t* states, int32_t count, const int32_t* blocks,
                      int32_t* out_n, int32_t* out_origins, int32_t* out_reliability, void* stream);

/* build_expansion_map (framework.py:130-148) for `count` patch origins:
 * out_k [count] entries, out_origins [count][2048][2] window origins and
 * out_rings [count][2048], sorted by (ring, row, col). */
int bm_expansion_maps(int height, int width, int32_t count, const int32_t* origins, int32_t* out_k,
                      int32_t* out_origins, int32_t* out_rings, void* stream);

/* Estimator stages (estimators.py:105-245) on `count` dense instances (the
 * bm_estimate_batch layout: n_y, m, y0 [count][32], x [count][max_m][4],
 * y [count][max_m][32]).  cov [count][BM_COV_DOUBLES] = c_xx [4][4],
 * c_xy [4][32], c_yy [32][32] (ridge included), ridge: written by
 * BM_STAGE_COVARIANCE, read by the stages that take a CovarianceBlocks.
 * out_status[i]: 0 ok, 2 C_YY not positive definite (LinAlgError). */
#define BM_STAGE_COVARIANCE 0     /* sample_covariance -> cov */
#define BM_STAGE_KERNEL_WEIGHTS 1 /* kernel_weights(beta[i], cov) -> out_w [count][max_m], scalars[0] raw_sum */
#define BM_STAGE_OPTIMIZE_BETA 2  /* optimize_beta(cov) -> scalars[0] beta, [1] its eps */
#define BM_STAGE_OPTIMIZE_ALPHA 3 /* optimize_alpha(beta[i], cov) -> scalars[0] alpha */
#define BM_STAGE_IDL_WEIGHTS 4    /* idl_weights(sigma2) -> out_w, scalars[0] raw_sum; out_mat[i][j][0] (if
                                     not NULL) = raw_idl_weights r_j */
#define BM_STAGE_PREDICT 5        /* predict_xy(w = out_w as input) -> scalars[0..3] x~, [4..4+n) y~ */
#define BM_STAGE_SOLVE 6          /* CovarianceBlocks.solve_yy: out_mat [count][max_m][32] = C_YY^-1 y_j */
#define BM_COV_DOUBLES (16 + 128 + 1024 + 1)
int bm_estimator_stages(int32_t stage, int32_t count, int32_t max_m, double sigma2, const int32_t* n_y,
                        const int32_t* m, const double* y0, const double* x, const double* y, const double* beta,
                        double* cov, double* out_w, double* out_mat, double* out_scalars, int32_t* out_status,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKMEND_B200_H */
