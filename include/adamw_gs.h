/*
 * adamw_gs.h — C ABI of the B200-native AdamW-GS optimizer step.
 *
 * Drop-in boundary for the reference optimizer's step family
 * (/root/reference/pkg/src/splatlab/optimizer.py).  Every entry point is
 * stream-ordered, never allocates, never synchronises the host, and takes
 * plain device pointers + sizes.  Buffers belong to the caller.
 *
 * Status: every function returns GS_OK (0) or a negative GS_ERR_* code;
 * gs_last_error() describes the last failure of the calling thread.
 * Data errors (non-finite gradients, tau/kappa outside the activation
 * domain) are not status codes: they are counted in the step statistics
 * (fused check) or raised in a device flag (strict check), so the host can
 * raise GradientError / DomainError without a per-step sync.
 *
 * Reference interface each entry point replaces (file:line under
 * /root/reference/pkg/src/splatlab/):
 *   gs_compact_u8 / gs_compact_i32  np.flatnonzero(vis)            optimizer.py:235,249
 *   gs_step                         adam_step_sync / sparse_adam_step /
 *                                   dar_step (_decoupled_reg_step) /
 *                                   adamw_const_step (+ coupled_reg_grad
 *                                   folded in for the coupled modes)
 *                                   optimizer.py:222-324, loss.py:177-198
 *   gs_check_grads                  ParamGrads.finite_check / _check_grads
 *                                   gradients.py:50-58, optimizer.py:181-184
 *   gs_rsr_apply                    rsr_apply                       optimizer.py:327-340
 *   gs_reset_rows                   reset_rows                      optimizer.py:159-165
 *   gs_stats_all                    classify_active + moment_stats  primitives.py:228-238,
 *                                                                   optimizer.py:489-506
 */
#ifndef ADAMW_GS_H
#define ADAMW_GS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 4
#define GS_MAX_GROUPS 8

/* gs_build_flags() bits */
#define GS_BUILD_FLAG_VARIANTS 1 /* measured K2 alternatives compiled in (-DGS_BUILD_VARIANTS=1) */
#define GS_BUILD_FLAG_TMA4 2     /* the 2-D TMA (tile::gather4 / scatter4) record kernel */

/* status codes */
#define GS_OK 0
#define GS_ERR_ARG (-1)
#define GS_ERR_LAUNCH (-2)
#define GS_ERR_WORKSPACE (-3)
#define GS_ERR_ALIGN (-4)

/* attribute-group roles (optimizer.py:217,259-263) */
#define GS_ROLE_PLAIN 0
#define GS_ROLE_POSITION 1 /* takes mu_lr_scale (already folded into lr) */
#define GS_ROLE_OPACITY 2  /* tau: sigma'(tau) penalty */
#define GS_ROLE_SCALE 3    /* kappa: exp(kappa) penalty, kappa <= 80 */

/* step modes (optimizer.py:55 MODES) */
#define GS_MODE_COUPLED_ADAM 0     /* dense sync Adam, global clock (+ coupled reg) */
#define GS_MODE_SPARSE_ADAM 1      /* masked Adam (+ coupled reg / N_v) */
#define GS_MODE_ADAMW_CONST 2      /* decoupled + lambda*R'(theta) */
#define GS_MODE_ADAMW_CONST_CLIP 3 /* decoupled + min(lambda*R'(theta), clip) */
#define GS_MODE_ADAMW_GS 4         /* decoupled + DAR min(lambda*(R'/N_I')/(sqrt(v^)+eps), C_t) */

/* error-check policies */
#define GS_CHECK_FUSED 0  /* rows with bad gradients / domain are skipped and counted */
#define GS_CHECK_STRICT 1 /* step is a no-op when *abort_flag != 0 (from gs_check_grads) */

/* indices of the per-step statistics written by gs_step (doubles) */
#define GS_STAT_N_VISIBLE 0      /* rows in the index list */
#define GS_STAT_N_STEPPED 1      /* rows updated */
#define GS_STAT_N_BAD_GRAD 2     /* rows skipped: non-finite gradient */
#define GS_STAT_N_BAD_DOMAIN 3   /* rows skipped: tau non-finite / kappa > 80 */
#define GS_STAT_N_ACTIVE_PRE 4   /* stepped rows with sigma(tau) > 1/255 before */
#define GS_STAT_N_ACTIVE_POST 5  /* ... after */
#define GS_STAT_N_CLIP_OPACITY 6 /* opacity penalty terms that hit C_t / clip */
#define GS_STAT_N_CLIP_SCALE 7   /* scale penalty terms that hit C_t / clip */
#define GS_STAT_SUM_EXTRA_OPACITY 8
#define GS_STAT_SUM_EXTRA_SCALE 9
#define GS_STAT_N_RUNS 10        /* layout hint: row runs that start a new run within a chunk of
                                  * the record kernels (0 from the other kernels); n_visible /
                                  * n_runs near 1 = scattered rows, >> 1 = index-coherent masks */
#define GS_STEP_STATS 11

/* One attribute group: row-major [n_rows, width] fp32, contiguous rows. */
typedef struct gs_group {
  float* param;
  const float* grad;
  float* exp_avg;    /* first moment m  */
  float* exp_avg_sq; /* second moment v */
  int64_t width;
  int32_t role; /* GS_ROLE_* */
  float lr;     /* effective learning rate of this step */
  /* Row strides (elements) of param and grad; 0 = width (dense rows).  A
   * stride > width lets the attributes be views of one row-interleaved
   * parameter record (and its gradient record): every visible row is then
   * one contiguous run in HBM instead of one narrow piece per attribute.
   * exp_avg / exp_avg_sq (per-group state layout) are always dense. */
  int64_t param_stride;
  int64_t grad_stride;
} gs_group;

typedef struct gs_step_cfg {
  int32_t mode;  /* GS_MODE_* */
  int32_t check; /* GS_CHECK_* */
  float one_minus_beta1;
  float one_minus_beta2;
  float eps;
  float active_logit; /* tau > active_logit  <=>  sigmoid(tau) > 1/255 (f64) */
  double lambda_opacity; /* DAR / const / coupled lambda for the opacity group */
  double lambda_scale;
  double clip_opacity; /* C_t (adamw-gs) or clip (adamw-const-clip) */
  double clip_scale;
  double n_pixels_rounded; /* N_I' (optimizer.py:168-178), adamw-gs only */
  const float* bias_lut;   /* device float2 per clock t: 1/(1-b1^t), 1/(1-b2^t) */
  int32_t lut_len;
  int32_t global_t;     /* coupled-adam: the incremented global clock */
  double beta1, beta2;  /* bias correction beyond the LUT */
  const int32_t* n_visible_norm; /* device N_v for the coupled modes (may be NULL) */
  double n_visible_host;         /* used when n_visible_norm == NULL */
  const int32_t* abort_flag;    /* strict mode: device flag written by gs_check_grads */
  /* fused densification statistics (DensifyStats.observe, pipeline.py:67-91):
   * for every stepped row, accum[row] += ||grad[group densify_group][row]||_2
   * * densify_scale and count[row] += 1.  densify_group < 0 disables. */
  float* densify_accum;
  int32_t* densify_count;
  float densify_scale;
  int32_t densify_group;
} gs_step_cfg;

int32_t gs_abi_version(void);
const char* gs_last_error(void);
int32_t gs_device_sm_count(void);

/* Device address of page-locked (pinned, mapped) host memory.  Gradient
 * pointers in gs_group may be such addresses: the step then gathers only the
 * visible rows' gradients over PCIe instead of a dense host->device copy
 * (zero-copy; the reference's gradients come from the host renderer,
 * pipeline.py:299-304). */
int gs_host_device_pointer(const void* host_ptr, void** dev_ptr);

/* K1 — visibility compaction: ascending int32 indices of nonzero mask bytes
 * (or radii > 0), count written to *count_out (device).  Bit-exact with
 * np.flatnonzero.  ws: gs_compact_workspace_bytes(n) bytes (one int per
 * 8192-row tile, an arrival counter, one selection bit per row): zero it
 * once before the first call; every call leaves the counter at zero
 * (graph-capturable).  Two launches: per-tile counts plus the selection
 * bitmap (the last CTA scans the counts into offsets), then ordered writes
 * from the bitmap. */
size_t gs_compact_workspace_bytes(int64_t n);
int gs_compact_u8(const uint8_t* mask, int64_t n, int32_t* idx_out, int32_t* count_out,
                  void* ws, size_t ws_bytes, void* stream);
int gs_compact_i32(const int32_t* radii, int64_t n, int32_t* idx_out, int32_t* count_out,
                   void* ws, size_t ws_bytes, void* stream);
/* Generalised selection: rows with mask != 0 (invert = 0) or mask == 0
 * (invert != 0), restricted to alive[row] != 0 when alive is not NULL — e.g.
 * the invisible alive rows of aiu_apply, np.flatnonzero(alive & ~vis)
 * (optimizer.py:437). */
int gs_compact_select_u8(const uint8_t* mask, const uint8_t* alive, int32_t invert, int64_t n,
                         int32_t* idx_out, int32_t* count_out, void* ws, size_t ws_bytes,
                         void* stream);

/* K2 — the fused step over the rows listed in rows[0 .. *n_rows_dev) (or all
 * max_rows rows in coupled-adam mode, rows == NULL).  clock: int32 per row.
 * stats_out: GS_STEP_STATS doubles (overwritten).  ws: gs_step_workspace_bytes(),
 * zero-filled once at allocation. */
size_t gs_step_workspace_bytes(void);
int gs_step(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
            const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
            int32_t* clock, double* stats_out, void* ws, size_t ws_bytes, void* stream);

/* Strict pre-check: non-finite gradients over ALL n_rows rows (bit 0), and
 * over the listed visible rows rows[0 .. *n_list_dev) tau non-finite when
 * lambda_opacity != 0 or kappa non-finite / > 80 when lambda_scale != 0
 * (bit 1).  *abort_flag is reset then OR-ed; bad_rows_out (nullable, 4-byte
 * aligned, n_rows bytes) gets the per-row bits.  rows may be NULL (no domain
 * check). */
int gs_check_grads(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                   const int32_t* rows, const int32_t* n_list_dev, double lambda_opacity,
                   double lambda_scale, uint8_t* bad_rows_out, int32_t* abort_flag,
                   void* stream);

/* K3 — re-state regularisation m *= alpha1, v *= alpha2 on the k rows
 * (clock untouched), and relocation resets m = v = 0, clock = 0. */
int gs_rsr_apply(const gs_group* groups, int32_t n_groups, const int32_t* rows, int64_t k,
                 int64_t n_rows, double alpha1, double alpha2, void* stream);
int gs_reset_rows(const gs_group* groups, int32_t n_groups, int32_t* clock,
                  const int32_t* rows, int64_t k, int64_t n_rows, void* stream);
/* (K3 entry points skip row ids outside [0, n_rows); the host validates and
 * de-duplicates index lists before they reach the device.) */

/* K4 — all-row statistics.  out (device doubles, 2 + 5*n_groups):
 *   [0] n_alive, [1] n_active (opacity group tau > active_logit, alive rows),
 *   then per group g at 2+5g: sum sqrt(v), max sqrt(v), n(v>0),
 *   sum |m|/sqrt(v) over v>0, max |m|/sqrt(v).
 * alive may be NULL (all rows alive).  ws: gs_stats_workspace_bytes(). */
size_t gs_stats_workspace_bytes(int32_t n_groups);
int gs_stats_all(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                 const uint8_t* alive, float active_logit, double* out, void* ws,
                 size_t ws_bytes, void* stream);

/* ---- row-record optimizer state (the default AdamWGS layout) -------------
 * record[row] = { (m_0, v_0), ..., (m_{P-1}, v_{P-1}), (clock:int32, pad) },
 * P = sum of the group widths in group order, record_stride >= 2*(P+1)
 * floats (even).  The exp_avg / exp_avg_sq fields of gs_group are ignored by
 * these entry points; param / grad / width / role / lr are used.  One
 * contiguous record per visible row replaces 2*n_groups narrow scattered
 * spans plus the clock (see paper_2601_16736_b200/csrc/gs_step_rows.cu). */
/* AIU — artificial implicit updates (optimizer.py:425-450): picked row i is
 * inv_idx[jlist[i]] for i < *k_dev (<= max_k); each picked row with clock > 0
 * steps theta -= (lr_eta * m^) / (sqrt(v^) + eps) with its frozen record
 * state; m, v, clock untouched.  groups[g].lr carries fl32(lr_g * eta).
 * picked_out (nullable) receives the picked rows in order. */
int gs_aiu_apply_rows(const gs_group* groups, int32_t n_groups, float* record,
                      int64_t record_stride, const int32_t* inv_idx, const int32_t* jlist,
                      const int32_t* k_dev, int64_t max_k, const float* bias_lut,
                      int32_t lut_len, float eps, int32_t* picked_out, void* stream);

/* MCMC relocation (pipeline.py:197-233): for i < k, row dead[i] takes every
 * attribute of row targets[i]; the opacity group (width 1) of both rows is set
 * to tau_new[i] (the blend-preserving logit, float64 on the host); the state
 * record row of dead[i] is zeroed (moments and clock, reset_rows,
 * optimizer.py:159-165).  Dead rows must be distinct and disjoint from the
 * targets (the reference's dead / live split guarantees it). */
int gs_relocate_rows(const gs_group* groups, int32_t n_groups, int32_t opacity_group,
                     const int32_t* dead, const int32_t* targets, const float* tau_new,
                     int64_t k, float* record, int64_t record_stride, void* stream);

/* Opacity-gated position noise (optimizer.py:453-486): for every alive row,
 * delta = -eta_ratio * lr_position * sigmoid(-lambda_mu (sigmoid(tau) -
 * lambda_t)) * Sigma gamma, Sigma = R diag(exp(2 log_scale)) R^T, gamma from a
 * Philox4x32-10 stream keyed by seed, counted by (row, iteration).  dims 2:
 * position [n,2], log_scale [n,2], rotation = angle [n]; dims 3 (3DGS):
 * position [n,3], log_scale [n,3], rotation = quaternion (w,x,y,z) [n,4].
 * delta_out (nullable, [n,dims]) receives delta; add_in_place adds it to
 * position.  Statistical parity with the reference (host RNG not reproduced). */
int gs_noise_perturb(float* position, const float* log_scale, const float* rotation,
                     const float* opacity_logit, const uint8_t* alive, int64_t n, int32_t dims,
                     float lr_position, float eta_ratio, float lambda_mu, float lambda_t,
                     uint64_t seed, uint32_t iteration, float* delta_out, int32_t add_in_place,
                     const int64_t* row_strides, void* stream);
/* row_strides: nullable; else 4 row strides (elements) of position,
 * log_scale, rotation, opacity_logit (0 = dense), for record views. */

size_t gs_step_rows_workspace_bytes(void);
/* Workspace of gs_step_rows_masked that enables the two-phase kernel for a
 * mask of n_rows rows (the base workspace + per-CTA counts + an n_rows
 * int32 id list).  No reference counterpart (device workspace). */
size_t gs_step_rows_masked_workspace_bytes(int64_t n_rows);
/* Select the (rows-in-flight, residency) variant of the SH-3 step kernel
 * (0 = default; tuning only, results are identical).  Returns the previous
 * variant.  The GS_ROWS_VARIANT environment variable sets the initial one. */
int32_t gs_set_rows_variant(int32_t variant);
/* Select the variant of the compile-time-layout (3DGS SH-3) step kernel that
 * gs_step_rows dispatches to for that layout: 0 = default, > 0 tuning
 * variants (identical results), -1 = disable the fixed-layout path (the
 * generic row kernel runs).  Returns the previous value.  GS_FIXED_VARIANT
 * sets the initial one. */
int32_t gs_set_fixed_variant(int32_t variant);
int gs_step_rows(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                 const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                 float* record, int64_t record_stride, double* stats_out, void* ws,
                 size_t ws_bytes, void* stream);
int gs_rsr_apply_rows(float* record, int64_t record_stride, int32_t n_elems,
                      const int32_t* rows, int64_t k, int64_t n_rows, double alpha1,
                      double alpha2, void* stream);
int gs_reset_rows_rows(float* record, int64_t record_stride, int32_t n_elems,
                       const int32_t* rows, int64_t k, int64_t n_rows, void* stream);

/* Densification statistics of the listed rows (DensifyStats.observe,
 * pipeline.py:77-82): for i < *n_list_dev (<= max_rows), row r = rows[i]:
 * accum[r] += ||grad[r, 0:width]||_2 * scale, count[r] += 1 (fp32, the
 * fused kernels' order).  Used with the dense coupled-adam step, which
 * updates every row but observes only the visible ones.  abort_flag
 * (nullable): a strict pre-check's flag; non-zero makes the call a no-op. */
int gs_densify_rows(const float* grad, int64_t grad_stride, int32_t width, const int32_t* rows,
                    const int32_t* n_list_dev, int64_t max_rows, float* accum, int32_t* count,
                    float scale, const int32_t* abort_flag, void* stream);

/* Fused K1 + K2 (the fused check): the step of the visible rows of a mask
 * (uint8 mask != 0, or int32 radii > 0; exactly one of the two) without a
 * separate compaction pass or index list.  *launched = 1 if this layout ran
 * (the SH-3 row records with device-resident gradients on the 2-D TMA
 * kernel; not the dense coupled-adam mode); *launched = 0 (status GS_OK)
 * asks the caller to compact and call gs_step_rows.  Two kernels serve it:
 * large clouds stream the mask through the step kernel's loader; with a
 * workspace of gs_step_rows_masked_workspace_bytes(n_rows) bytes (16-byte
 * aligned), smaller clouds with index-coherent masks (GS_MASKED_COHERENT)
 * or a coupled sparse-adam step without cfg->n_visible_norm run the
 * two-phase kernel (the mask compacted into the workspace, a grid barrier,
 * even shares of the visible rows per CTA; it counts N_v itself).
 * Otherwise a coupled sparse-adam step needs cfg->n_visible_norm (e.g. from
 * gs_count_visible; the sharded global count always comes this way).  The
 * statistics' n_visible is the mask's visible count; results equal
 * gs_compact + gs_step_rows bit for bit (rows are independent).  flags:
 * GS_MASKED_LOW_VISIBILITY picks the kernel shape for sparse masks (a few %
 * visible), GS_MASKED_COHERENT the two-phase kernel for small clouds,
 * GS_MASKED_BALANCE_TAIL the dynamic tail of the tile dealing (same results
 * in every case). */
#define GS_MASKED_LOW_VISIBILITY 1
/* flags: the mask's visible rows come in long index runs (e.g. the last
 * step's GS_STAT_N_RUNS hint); small clouds then balance them (two-phase). */
#define GS_MASKED_COHERENT 2
/* flags: the mask is not very sparse (>= ~2 % visible, e.g. the last step's
 * statistics): the streaming kernel claims its last mask tiles dynamically
 * so that the CTAs finish together (same results). */
#define GS_MASKED_BALANCE_TAIL 4
int gs_step_rows_masked(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                        const uint8_t* mask, const int32_t* radii, int64_t n_rows, float* record,
                        int64_t record_stride, double* stats_out, void* ws, size_t ws_bytes,
                        int32_t flags, int32_t* launched, void* stream);

/* The reference's host Bernoulli draw (aiu_apply, optimizer.py:437-440:
 * rng.random(n) < prob with rng a numpy Generator over Philox4x64-10,
 * rng.py:17-30) on the device, bit for bit: out[i] = (u(first + i) < prob)
 * with u(j) = (philox4x64_10(counter + 1 + j/4, key)[j % 4] >> 11) * 2^-53,
 * i.e. draw j of a generator with an empty buffer at that counter.
 * counter: 4 uint64 (host pointer), key: 2 uint64 (host pointer). */
int gs_philox_bernoulli(const uint64_t* counter, const uint64_t* key, int64_t first, int64_t n,
                        double prob, uint8_t* out, void* stream);

/* The visible count alone (the count pass of gs_compact_u8 / _i32, no
 * index list): N_v = popcount(vis) (loss.py:190) for the coupled
 * normaliser ahead of gs_step_rows_masked.  Exactly one of mask / radii;
 * workspace as gs_compact. */
int gs_count_visible(const uint8_t* mask, const int32_t* radii, int64_t n, int32_t* count_out,
                     void* ws, size_t ws_bytes, void* stream);

/* Copy up to two small device buffers (4-byte multiples, <= 4 KB each; a
 * size of 0 skips one) into page-locked host memory through mapped
 * pointers, with one small kernel in the stream: the step statistics and
 * the strict abort flag for an asynchronous error check (the reference
 * raises in step(), optimizer.py:181-184; the optimizer reads the copies
 * once the stream has passed them).  No reference counterpart. */
int gs_mirror_to_host(const void* src0, void* dst0_host, size_t bytes0, const void* src1,
                      void* dst1_host, size_t bytes1, void* stream);

/* GS_BUILD_FLAG_* bits of this build. */
int32_t gs_build_flags(void);
int gs_stats_all_rows(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                      const float* record, int64_t record_stride, const uint8_t* alive,
                      float active_logit, double* out, void* ws, size_t ws_bytes,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADAMW_GS_H */
