// K2 (row-record state) — the fused AdamW-GS step with the optimizer state
// stored as one contiguous record per primitive.
//
// State layout (owned by the optimizer, exposed to the host as strided
// per-group m / v views and an int32 clock view):
//
//     record[row] = { (m_0, v_0), (m_1, v_1), ..., (m_{P-1}, v_{P-1}), (clock, pad) }
//
// P = the summed widths of the attribute groups (59 for 3DGS SH-3), so a
// record is 8*(P+1) bytes (480 B for SH-3: 15 DRAM sectors, no partial
// sector).  A visible row therefore touches its optimizer state as one
// contiguous, fully-coalesced span instead of 2*G scattered narrow spans plus
// a 4-byte clock — for i.i.d. 30% visibility this cuts DRAM sector traffic
// from 1.37x to 1.16x of the algorithmic bytes (parameters and gradients stay
// in the caller's per-group struct-of-arrays layout).
//
// Work decomposition: a sub-warp of L lanes owns one row; lane q of the
// sub-warp owns record slots q, q+L, ..., q+(J-1)L (element s of the row is
// slot s; slot P is the clock).  The lane->(group, column) map is fixed for
// the whole launch, so per row a lane issues J float2 state loads, J
// parameter and J gradient loads, then votes: a row with any non-finite
// gradient (or tau / kappa outside the activation domain where a penalty is
// active) is skipped as a whole, with no second pass.  R rows per sub-warp
// are kept in flight for memory-level parallelism.
//
// Arithmetic per element is identical to gs_step.cu (and to
// oracle/adamw_gs_oracle.py::step_fp32).
#include <stdlib.h>

#include "gs_common.cuh"

int gs_step_fixed_try(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                      const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                      float* record, int64_t record_stride, double* stats_out, double* partials,
                      unsigned int* counter, void* stream);
int gs_step_fixed_masked_try(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                             const uint8_t* mask, const int32_t* radii, int64_t n_rows,
                             float* record, int64_t record_stride, double* stats_out,
                             double* partials, unsigned int* counter, unsigned int* tp_bar,
                             int32_t* tp_counts, int32_t* tp_ids, unsigned int* tile_ctr,
                             int32_t flags, void* stream);

namespace gs {

struct RowGroup {
  float* param;
  const float* grad;
  int width;
  int role;
  float lr;
  int offset;  // first element of the group in the record
  int ps;      // param / grad row strides (elements)
  int gs;
};

struct RowParams {
  RowGroup g[GS_MAX_GROUPS];
  int n_groups;
  int P;  // elements per row
  float active_logit;
  StepConsts K;
  const float* lut;
  int lut_len;
  int global_t;
  double beta1, beta2;
  const int32_t* nv_dev;
  double nv_host;
  const int32_t* abort_flag;
  DensifyArgs D;
  const int32_t* rows;
  const int32_t* n_rows_dev;
  int64_t max_rows;
  float* record;
  int64_t stride;  // floats per record
  double* stats_out;
  double* partials;
  unsigned int* counter;
};

constexpr int kRowThreads = 256;
constexpr int kRowBlocksPerSM = 4;   // default residency target
constexpr int kRowMaxBlocksPerSM = 8;  // workspace sizing over all variants

// per-lane, launch-constant description of one record slot
struct Slot {
  float* param;
  const float* grad;
  int ps;  // row strides of param / grad
  int gs;
  int col;
  int role;  // -1 inactive, -2 clock, else GS_ROLE_*
  float lr;
};

template <int MODE>
struct RowModeTraits {
  static constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  static constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
};

template <int MODE, bool STRICT, int L, int J, int R, int MINB>
__global__ void __launch_bounds__(kRowThreads, MINB)
    step_rows_kernel(const RowParams P) {
  using T = RowModeTraits<MODE>;
  __shared__ double s_red[GS_STEP_STATS * (kRowThreads / 32)];
  constexpr int kSub = 32 / L;  // rows handled side by side by one warp
  const int lane = threadIdx.x & 31;
  const int q = lane % L;       // lane within the sub-warp
  const int sub = lane / L;     // sub-warp index within the warp
  const unsigned sub_mask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (sub * L));

  int64_t n_rows = T::kDense ? P.max_rows : (int64_t)(*P.n_rows_dev);
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  // decoupled modes read the constants straight from the parameter bank;
  // the coupled modes patch in 1/N_v (loss.py:190-192: no term when N_v = 0)
  StepConsts Kc = P.K;
  if (T::kCoupled) {
    const float nv = P.nv_dev ? (float)(*P.nv_dev) : (float)P.nv_host;
    Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
    if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
  }
  const StepConsts& K = T::kCoupled ? Kc : P.K;

  // ---- launch-constant slot map ------------------------------------------
  Slot sl[J];
  const int clock_lane = P.P % L;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int s = q + L * j;
    Slot x{nullptr, nullptr, 1, 1, 0, -1, 0.f};
    if (s == P.P) {
      x.role = -2;
    } else if (s < P.P) {
      for (int gi = 0; gi < P.n_groups; ++gi) {
        const RowGroup& G = P.g[gi];
        if (s >= G.offset && s < G.offset + G.width) {
          x.param = G.param;
          x.grad = G.grad;
          x.ps = G.ps;
          x.gs = G.gs;
          x.col = s - G.offset;
          x.role = G.role;
          x.lr = G.lr;
        }
      }
    }
    sl[j] = x;
  }

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  const int64_t warps_total = (int64_t)gridDim.x * (kRowThreads / 32);
  const int64_t warp_id = (int64_t)blockIdx.x * (kRowThreads / 32) + (threadIdx.x >> 5);
  constexpr int kRowsPerIter = kSub * R;  // rows per warp per iteration

  for (int64_t base = warp_id * kRowsPerIter; base < n_rows; base += warps_total * kRowsPerIter) {
    int32_t row[R];
    bool valid[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = base + r * kSub + sub;
      valid[r] = i < n_rows;
      row[r] = valid[r] ? (T::kDense ? (int32_t)i : __ldg(P.rows + i)) : 0;
    }
    // ---- loads for R rows -------------------------------------------------
    float2 mv[R][J];
    float th[R][J], gr[R][J];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float* rec = P.record + (int64_t)row[r] * P.stride;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int s = q + L * j;
        mv[r][j] = make_float2(0.f, 0.f);
        th[r][j] = 0.f;
        gr[r][j] = 0.f;
        if (valid[r] && sl[j].role != -1) {
          mv[r][j] = *reinterpret_cast<const float2*>(rec + 2 * s);
          if (sl[j].role >= 0) {
            th[r][j] = sl[j].param[(int64_t)row[r] * sl[j].ps + sl[j].col];
            gr[r][j] = __ldg(sl[j].grad + (int64_t)row[r] * sl[j].gs + sl[j].col);
          }
        }
      }
    }
    // ---- per row: validity vote, clock, bias factors, update ----------------
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float* rec = P.record + (int64_t)row[r] * P.stride;
      int bad = 0;
      if (!STRICT) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          if (sl[j].role >= 0) {
            float g = gr[r][j];
            if (!isfinite(g)) bad |= 1;
            const float lam = sl[j].role == GS_ROLE_OPACITY ? K.lam_op
                              : sl[j].role == GS_ROLE_SCALE ? K.lam_sc : 0.0f;
            if (lam != 0.0f && domain_bad(sl[j].role, th[r][j])) bad |= 2;
          }
        }
      }
      const unsigned b1 = __ballot_sync(0xffffffffu, bad & 1) & sub_mask;
      const unsigned b2 = __ballot_sync(0xffffffffu, bad & 2) & sub_mask;
      const bool row_bad = (b1 | b2) != 0;
      // clock lane: t -> t+1, bias factors
      float2 bc = make_float2(1.f, 1.f);
      int tn = 0;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (sl[j].role == -2) {
          tn = __float_as_int(mv[r][j].x) + 1;
          bc = bias_factors(P.lut, P.lut_len, T::kDense ? P.global_t : tn, P.beta1, P.beta2);
        }
      }
      const int src = sub * L + clock_lane;
      bc.x = __shfl_sync(0xffffffffu, bc.x, src);
      bc.y = __shfl_sync(0xffffffffu, bc.y, src);
      if (!valid[r]) continue;  // uniform within the sub-warp
      if (q == clock_lane) {
        ++c_vis;
        if (!row_bad && P.D.group >= 0) {
          const RowGroup& DG = P.g[P.D.group];
          densify_row(P.D, (uint32_t)row[r], DG.grad + (int64_t)row[r] * DG.gs, DG.width, 1);
        }
        if (!row_bad) ++c_step;
        else if (b1) ++c_badg;
        else ++c_badd;
      }
      if (row_bad) continue;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int s = q + L * j;
        const int role = sl[j].role;
        if (role == -2) {
          // clock slot: keep the pad word, bump the count
          reinterpret_cast<int*>(rec)[2 * s] = tn;
          continue;
        }
        if (role < 0) continue;
        const float thv = th[r][j];
        float tn_th, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, sl[j].lr, thv, gr[r][j], mv[r][j].x, mv[r][j].y, bc, K, tn_th,
                             mn, vn, ex, clipped);
        if (!T::kCoupled) {
          if (role == GS_ROLE_OPACITY) {
            c_clo += clipped;
            s_exo += (double)ex;
          } else if (role == GS_ROLE_SCALE) {
            c_cls += clipped;
            s_exs += (double)ex;
          }
        }
        if (role == GS_ROLE_OPACITY) {
          c_apre += thv > P.active_logit;
          c_apost += tn_th > P.active_logit;
        }
        sl[j].param[(int64_t)row[r] * sl[j].ps + sl[j].col] = tn_th;
        *reinterpret_cast<float2*>(rec + 2 * s) = make_float2(mn, vn);
      }
    }
  }

  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce<GS_STEP_STATS>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f)
      P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter))
    final_reduce<GS_STEP_STATS>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out, is_max, s_red);
}

struct RowStepWorkspace {
  unsigned int counter;  // last-block-done counter of the statistics
  unsigned int bar[2];   // grid barrier of the two-phase fused kernel
  unsigned int tile_ctr; // claim counter of the streaming fused kernel's dynamic tail
  unsigned int pad[12];
};

int max_row_blocks() { return gs_sm_count() * kRowMaxBlocksPerSM; }

// Tuning variants of the SH-3 shape (L=32, J=2): rows in flight per warp R
// and the residency target MINB (registers = 64K / (256 * MINB)).
static int g_rows_variant = -1;

int rows_variant() {
  if (g_rows_variant < 0) {
    const char* e = getenv("GS_ROWS_VARIANT");
    g_rows_variant = e ? atoi(e) : 0;
  }
  return g_rows_variant;
}

template <int MODE, bool STRICT, int L, int J, int R, int MINB>
void launch_rows_v(const RowParams& P, int grid, cudaStream_t s) {
  const int g = std::min(grid, gs_sm_count() * MINB);
  step_rows_kernel<MODE, STRICT, L, J, R, MINB><<<g, kRowThreads, 0, s>>>(P);
}

template <int MODE, bool STRICT, int L, int J>
void launch_rows(const RowParams& P, int grid, cudaStream_t s) {
  if constexpr (L == 32 && J == 2 && MODE == GS_MODE_ADAMW_GS && !STRICT) {
    switch (rows_variant()) {
      case 1: launch_rows_v<MODE, STRICT, L, J, 1, 4>(P, grid, s); return;
      case 2: launch_rows_v<MODE, STRICT, L, J, 2, 3>(P, grid, s); return;
      case 3: launch_rows_v<MODE, STRICT, L, J, 4, 2>(P, grid, s); return;
      case 4: launch_rows_v<MODE, STRICT, L, J, 1, 6>(P, grid, s); return;
      case 5: launch_rows_v<MODE, STRICT, L, J, 2, 6>(P, grid, s); return;
      case 6: launch_rows_v<MODE, STRICT, L, J, 4, 4>(P, grid, s); return;
      default: break;
    }
  }
  constexpr int R = (L == 32) ? 2 : 1;
  launch_rows_v<MODE, STRICT, L, J, R, kRowBlocksPerSM>(P, grid, s);
}

template <bool STRICT, int L, int J>
void dispatch_mode(int mode, const RowParams& P, int grid, cudaStream_t s) {
  switch (mode) {
    case GS_MODE_COUPLED_ADAM: launch_rows<GS_MODE_COUPLED_ADAM, STRICT, L, J>(P, grid, s); break;
    case GS_MODE_SPARSE_ADAM: launch_rows<GS_MODE_SPARSE_ADAM, STRICT, L, J>(P, grid, s); break;
    case GS_MODE_ADAMW_CONST: launch_rows<GS_MODE_ADAMW_CONST, STRICT, L, J>(P, grid, s); break;
    case GS_MODE_ADAMW_CONST_CLIP:
      launch_rows<GS_MODE_ADAMW_CONST_CLIP, STRICT, L, J>(P, grid, s);
      break;
    default: launch_rows<GS_MODE_ADAMW_GS, STRICT, L, J>(P, grid, s); break;
  }
}

template <bool STRICT>
int dispatch_shape(int slots, int mode, const RowParams& P, int grid, cudaStream_t s) {
  // slots = P + 1 (elements + clock); L lanes per row, J slots per lane
  if (slots <= 16) dispatch_mode<STRICT, 8, 2>(mode, P, grid, s);
  else if (slots <= 32) dispatch_mode<STRICT, 16, 2>(mode, P, grid, s);
  else if (slots <= 64) dispatch_mode<STRICT, 32, 2>(mode, P, grid, s);
  else if (slots <= 128) dispatch_mode<STRICT, 32, 4>(mode, P, grid, s);
  else return GS_ERR_ARG;
  return GS_OK;
}

}  // namespace gs

extern "C" int32_t gs_set_rows_variant(int32_t variant) {
  const int32_t prev = gs::rows_variant();
  gs::g_rows_variant = variant < 0 ? 0 : variant;
  return prev;
}

extern "C" size_t gs_step_rows_workspace_bytes(void) {
  return sizeof(gs::RowStepWorkspace) +
         (size_t)gs::max_row_blocks() * GS_STEP_STATS * sizeof(double);
}

// gs_step_rows_masked with the two-phase compaction: the base workspace, then
// the per-CTA counts and an n_rows id list (16-byte aligned pieces).
extern "C" size_t gs_step_rows_masked_workspace_bytes(int64_t n_rows) {
  const size_t counts = ((size_t)gs::max_row_blocks() * sizeof(int32_t) + 15) & ~(size_t)15;
  return ((gs_step_rows_workspace_bytes() + 15) & ~(size_t)15) + counts +
         (((size_t)(n_rows > 0 ? n_rows : 0) * sizeof(int32_t) + 15) & ~(size_t)15);
}

extern "C" int gs_step_rows(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                            const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                            float* record, int64_t record_stride, double* stats_out, void* ws,
                            size_t ws_bytes, void* stream) {
  using namespace gs;
  if (!groups || !cfg || n_groups < 1 || n_groups > GS_MAX_GROUPS || !record || !stats_out ||
      max_rows < 0 || max_rows >= (int64_t)INT32_MAX) {
    gs_set_error("gs_step_rows: invalid arguments");
    return GS_ERR_ARG;
  }
  if (cfg->mode < GS_MODE_COUPLED_ADAM || cfg->mode > GS_MODE_ADAMW_GS) {
    gs_set_error("gs_step_rows: unknown mode %d", cfg->mode);
    return GS_ERR_ARG;
  }
  const bool dense = cfg->mode == GS_MODE_COUPLED_ADAM;
  if (!dense && (!rows || !n_rows_dev)) {
    gs_set_error("gs_step_rows: sparse modes need the index list and its device count");
    return GS_ERR_ARG;
  }
  if (cfg->check == GS_CHECK_STRICT && !cfg->abort_flag) {
    gs_set_error("gs_step_rows: strict check needs abort_flag");
    return GS_ERR_ARG;
  }
  if (!cfg->bias_lut || cfg->lut_len < 2) {
    gs_set_error("gs_step_rows: bias-correction LUT missing");
    return GS_ERR_ARG;
  }
  if (cfg->mode == GS_MODE_ADAMW_GS && !(cfg->n_pixels_rounded > 0.0)) {
    gs_set_error("gs_step_rows: adamw-gs needs N_I' > 0");
    return GS_ERR_ARG;
  }
  if (!ws || ws_bytes < gs_step_rows_workspace_bytes()) {
    gs_set_error("gs_step_rows: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  if (reinterpret_cast<uintptr_t>(record) & 7u) {
    gs_set_error("gs_step_rows: record must be 8-byte aligned");
    return GS_ERR_ALIGN;
  }
  RowParams P{};
  int off = 0;
  for (int i = 0; i < n_groups; ++i) {
    const gs_group& g = groups[i];
    if (!g.param || !g.grad || g.width < 1 || g.width > 127 ||
        (g.param_stride != 0 && (g.param_stride < g.width || g.param_stride > INT32_MAX)) ||
        (g.grad_stride != 0 && (g.grad_stride < g.width || g.grad_stride > INT32_MAX))) {
      gs_set_error("gs_step_rows: group %d invalid", i);
      return GS_ERR_ARG;
    }
    P.g[i] = RowGroup{g.param, g.grad, (int)g.width, g.role, g.lr, off,
                      (int)(g.param_stride ? g.param_stride : g.width),
                      (int)(g.grad_stride ? g.grad_stride : g.width)};
    off += (int)g.width;
  }
  if (record_stride < 2 * (off + 1) || (record_stride & 1)) {
    gs_set_error("gs_step_rows: record stride %lld < 2*(P+1) = %d", (long long)record_stride,
                 2 * (off + 1));
    return GS_ERR_ARG;
  }
  P.n_groups = n_groups;
  P.P = off;
  P.active_logit = cfg->active_logit;
  P.K = make_consts(cfg);
  P.lut = cfg->bias_lut;
  P.lut_len = cfg->lut_len;
  P.global_t = cfg->global_t;
  P.beta1 = cfg->beta1;
  P.beta2 = cfg->beta2;
  P.nv_dev = cfg->n_visible_norm;
  P.nv_host = cfg->n_visible_host;
  P.abort_flag = cfg->abort_flag;
  P.D = DensifyArgs{cfg->densify_accum, cfg->densify_count, cfg->densify_scale,
                    cfg->densify_group};
  if (P.D.group >= n_groups || (P.D.group >= 0 && (!P.D.accum || !P.D.count))) {
    gs_set_error("gs_step_rows: bad densification-statistics arguments");
    return GS_ERR_ARG;
  }
  P.rows = rows;
  P.n_rows_dev = n_rows_dev;
  P.max_rows = max_rows;
  P.record = record;
  P.stride = record_stride;
  P.stats_out = stats_out;
  auto* hdr = reinterpret_cast<RowStepWorkspace*>(ws);
  P.counter = &hdr->counter;
  P.partials = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + sizeof(RowStepWorkspace));

  if (gs_step_fixed_try(groups, n_groups, cfg, rows, n_rows_dev, max_rows, record, record_stride,
                        stats_out, P.partials, P.counter, stream))
    return gs_check_launch("gs_step_rows[fixed layout]");
  const int slots = off + 1;
  const int rows_per_block = (kRowThreads / 32) * (slots <= 16 ? 4 : slots <= 32 ? 2 : 1) *
                             (slots > 32 && slots <= 64 ? 2 : 1);
  const int64_t need = (max_rows + rows_per_block - 1) / rows_per_block;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, max_row_blocks()));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = cfg->check == GS_CHECK_STRICT
               ? dispatch_shape<true>(slots, cfg->mode, P, grid, s)
               : dispatch_shape<false>(slots, cfg->mode, P, grid, s);
  if (rc) {
    gs_set_error("gs_step_rows: %d elements per row exceed the compiled record shapes", off);
    return rc;
  }
  return gs_check_launch("gs_step_rows");
}

extern "C" int gs_step_rows_masked(const gs_group* groups, int32_t n_groups,
                                   const gs_step_cfg* cfg, const uint8_t* mask,
                                   const int32_t* radii, int64_t n_rows, float* record,
                                   int64_t record_stride, double* stats_out, void* ws,
                                   size_t ws_bytes, int32_t flags, int32_t* launched,
                                   void* stream) {
  using namespace gs;
  if (!launched) {
    gs_set_error("gs_step_rows_masked: launched must not be null");
    return GS_ERR_ARG;
  }
  *launched = 0;
  if (!groups || !cfg || n_groups < 1 || n_groups > GS_MAX_GROUPS || !record || !stats_out ||
      n_rows < 0 || n_rows >= (int64_t)INT32_MAX || (!mask && !radii) || (mask && radii)) {
    gs_set_error("gs_step_rows_masked: invalid arguments");
    return GS_ERR_ARG;
  }
  if (cfg->mode < GS_MODE_COUPLED_ADAM || cfg->mode > GS_MODE_ADAMW_GS || !cfg->bias_lut ||
      cfg->lut_len < 2 || (cfg->mode == GS_MODE_ADAMW_GS && !(cfg->n_pixels_rounded > 0.0))) {
    gs_set_error("gs_step_rows_masked: invalid step configuration");
    return GS_ERR_ARG;
  }
  if (!ws || ws_bytes < gs_step_rows_workspace_bytes()) {
    gs_set_error("gs_step_rows_masked: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  for (int i = 0; i < n_groups; ++i) {
    const gs_group& g = groups[i];
    if (!g.param || !g.grad || g.width < 1) {
      gs_set_error("gs_step_rows_masked: group %d invalid", i);
      return GS_ERR_ARG;
    }
  }
  if (cfg->densify_group >= n_groups ||
      (cfg->densify_group >= 0 && (!cfg->densify_accum || !cfg->densify_count))) {
    gs_set_error("gs_step_rows_masked: bad densification-statistics arguments");
    return GS_ERR_ARG;
  }
  auto* hdr = reinterpret_cast<RowStepWorkspace*>(ws);
  double* partials =
      reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + sizeof(RowStepWorkspace));
  // the two-phase compaction needs its counts and id list in the workspace
  int32_t* tp_counts = nullptr;
  int32_t* tp_ids = nullptr;
  if (ws_bytes >= gs_step_rows_masked_workspace_bytes(n_rows) &&
      (reinterpret_cast<uintptr_t>(ws) & 15u) == 0) {
    char* base = reinterpret_cast<char*>(ws) + gs_step_rows_workspace_bytes();
    base += (16 - (reinterpret_cast<uintptr_t>(base) & 15u)) & 15u;
    tp_counts = reinterpret_cast<int32_t*>(base);
    tp_ids = reinterpret_cast<int32_t*>(
        base + (((size_t)max_row_blocks() * sizeof(int32_t) + 15) & ~(size_t)15));
  }
  if (!gs_step_fixed_masked_try(groups, n_groups, cfg, mask, radii, n_rows, record, record_stride,
                                stats_out, partials, &hdr->counter, hdr->bar, tp_counts, tp_ids,
                                &hdr->tile_ctr, flags, stream))
    return GS_OK;  // not this layout: the caller compacts and calls gs_step_rows
  *launched = 1;
  return gs_check_launch("gs_step_rows_masked");
}
