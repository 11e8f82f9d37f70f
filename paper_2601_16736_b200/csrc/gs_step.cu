// K2 — the fused AdamW-GS step (replaces optimizer.py:207-324 and the coupled
// regularisation of loss.py:177-198 for the coupled modes).
//
// Work decomposition: the visible-row index list (K1 output) is cut into
// chunks of kThreads rows; a persistent grid of CTAs walks the chunks.  For a
// chunk, the CTA
//   0. loads the row ids and their clocks (one per row — SURVEY §0 fact 6),
//   1. (fused check) streams the chunk's gradients group by group and marks
//      rows carrying a non-finite gradient, or tau/kappa outside the
//      activation domain where a penalty is active; those rows are skipped,
//   2. bumps the clocks of the surviving rows and fetches the fp32 bias
//      correction factors (float64-derived LUT),
//   3. streams every group as a flattened (row, column) element sequence so a
//      warp touches contiguous bytes of consecutive columns of a row, updates
//      m, v and theta in place, and folds the DAR / const / coupled term and
//      the per-step statistics into the same pass.
// Statistics are reduced deterministically (per-CTA partials, last CTA sums
// them in CTA order).
//
// Per-element arithmetic is the contract mirrored by
// oracle/adamw_gs_oracle.py::step_fp32 (explicit _rn intrinsics, no FMA).
#include "gs_common.cuh"

namespace gs {

struct GroupDev {
  float* param;
  const float* grad;
  float* m;
  float* v;
  int width;
  int role;
  float lr;
  int pad;
  int64_t ps;  // param / grad row strides (elements)
  int64_t gs;
};

struct StepParams {
  GroupDev g[GS_MAX_GROUPS];
  int n_groups;
  int check;
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
  int32_t* clock;
  double* stats_out;
  double* partials;
  unsigned int* counter;
};

constexpr int kStepBlocksPerSM = 4;

template <int MODE>
struct ModeTraits {
  static constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  static constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  static constexpr bool kDecoupled = !kCoupled;
};

template <int MODE, bool STRICT>
__global__ void __launch_bounds__(kThreads, kStepBlocksPerSM) step_kernel(const StepParams P) {
  using T = ModeTraits<MODE>;
  __shared__ int32_t s_row[kThreads];
  __shared__ float2 s_bc[kThreads];
  __shared__ int s_bad[kThreads];
  __shared__ double s_red[GS_STEP_STATS * (kThreads / 32)];

  const int tid = threadIdx.x;
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

  unsigned int c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0,
               c_clo = 0, c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  const int64_t n_chunks = (n_rows + kThreads - 1) / kThreads;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const int64_t base = chunk * kThreads;
    const int nvalid = (int)(n_rows - base < kThreads ? n_rows - base : kThreads);
    const bool valid = tid < nvalid;
    int32_t row = -1;
    int t = 0;
    if (valid) {
      row = T::kDense ? (int32_t)(base + tid) : __ldg(P.rows + base + tid);
      t = P.clock[row];
    }
    s_row[tid] = row;
    s_bad[tid] = valid ? 0 : 4;
    __syncthreads();

    // ---- pass A: row validity (fused check) -----------------------------
    if (!STRICT) {
      for (int gi = 0; gi < P.n_groups; ++gi) {
        const GroupDev G = P.g[gi];
        const int W = G.width;
        const int E = nvalid * W;
        const float lam = G.role == GS_ROLE_OPACITY ? K.lam_op
                          : G.role == GS_ROLE_SCALE ? K.lam_sc : 0.0f;
        const bool dom = lam != 0.0f;
        const int dq = kThreads / W, dr = kThreads % W;
        int lr = tid / W, lc = tid % W;
        for (int e = tid; e < E; e += kThreads) {
          const int32_t r = s_row[lr];
          const float gv = __ldg(G.grad + (int64_t)r * G.gs + lc);
          int bad = finitef(gv) ? 0 : 1;
          if (dom && domain_bad(G.role, G.param[(int64_t)r * G.ps + lc])) bad |= 2;
          if (bad) atomicOr(&s_bad[lr], bad);
          lc += dr;
          lr += dq;
          if (lc >= W) { lc -= W; ++lr; }
        }
      }
      __syncthreads();
    }

    // ---- clocks + bias correction ----------------------------------------
    if (valid) {
      ++c_vis;
      const int bad = s_bad[tid];
      if (bad == 0) {
        const int tn = t + 1;
        P.clock[row] = tn;
        if (P.D.group >= 0) {
          const GroupDev& DG = P.g[P.D.group];
          densify_row(P.D, (uint32_t)row, DG.grad + (int64_t)row * DG.gs, DG.width, 1);
        }
        const int tb = T::kDense ? P.global_t : tn;
        s_bc[tid] = bias_factors(P.lut, P.lut_len, tb, P.beta1, P.beta2);
        ++c_step;
      } else if (bad & 1) {
        ++c_badg;
      } else {
        ++c_badd;
      }
    }
    __syncthreads();

    // ---- pass B: the update ------------------------------------------------
    for (int gi = 0; gi < P.n_groups; ++gi) {
      const GroupDev G = P.g[gi];
      const int W = G.width;
      const int E = nvalid * W;
      const int role = G.role;
      const float lrf = G.lr;
      const int dq = kThreads / W, dr = kThreads % W;
      int lr = tid / W, lc = tid % W;
      for (int e = tid; e < E; e += kThreads) {
        const int this_lr = lr;
        const int this_lc = lc;
        lc += dr;
        lr += dq;
        if (lc >= W) { lc -= W; ++lr; }
        if (s_bad[this_lr] != 0) continue;
        const int32_t r = s_row[this_lr];
        const int64_t off = (int64_t)r * W + this_lc;
        const int64_t poff = (int64_t)r * G.ps + this_lc;
        const float2 bc = s_bc[this_lr];
        const float th = G.param[poff];
        const float gr = __ldg(G.grad + (int64_t)r * G.gs + this_lc);
        const float mm = G.m[off];
        const float vv = G.v[off];
        float tn, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, lrf, th, gr, mm, vv, bc, K, tn, mn, vn, ex, clipped);
        if (!T::kCoupled && (role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE)) {
          if (role == GS_ROLE_OPACITY) {
            c_clo += clipped;
            s_exo += (double)ex;
          } else {
            c_cls += clipped;
            s_exs += (double)ex;
          }
        }
        if (role == GS_ROLE_OPACITY) {
          c_apre += th > P.active_logit;
          c_apost += tn > P.active_logit;
        }
        G.param[poff] = tn;
        G.m[off] = mn;
        G.v[off] = vn;
      }
    }
    __syncthreads();
  }

  // ---- deterministic statistics reduction -----------------------------------
  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce<GS_STEP_STATS>(acc, is_max, s_red);
  if (tid == 0) {
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f) P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter))
    final_reduce<GS_STEP_STATS>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out, is_max, s_red);
}

struct StepWorkspace {
  unsigned int counter;
  unsigned int pad[15];
};

int max_step_blocks() { return gs_sm_count() * kStepBlocksPerSM; }

template <int MODE, bool STRICT>
void launch_mode(const StepParams& P, int grid, cudaStream_t s) {
  step_kernel<MODE, STRICT><<<grid, kThreads, 0, s>>>(P);
}

template <bool STRICT>
void launch_dispatch(int mode, const StepParams& P, int grid, cudaStream_t s) {
  switch (mode) {
    case GS_MODE_COUPLED_ADAM: launch_mode<GS_MODE_COUPLED_ADAM, STRICT>(P, grid, s); break;
    case GS_MODE_SPARSE_ADAM: launch_mode<GS_MODE_SPARSE_ADAM, STRICT>(P, grid, s); break;
    case GS_MODE_ADAMW_CONST: launch_mode<GS_MODE_ADAMW_CONST, STRICT>(P, grid, s); break;
    case GS_MODE_ADAMW_CONST_CLIP: launch_mode<GS_MODE_ADAMW_CONST_CLIP, STRICT>(P, grid, s); break;
    default: launch_mode<GS_MODE_ADAMW_GS, STRICT>(P, grid, s); break;
  }
}

}  // namespace gs

extern "C" size_t gs_step_workspace_bytes(void) {
  return sizeof(gs::StepWorkspace) +
         (size_t)gs::max_step_blocks() * GS_STEP_STATS * sizeof(double);
}

extern "C" int gs_step(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                       const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                       int32_t* clock, double* stats_out, void* ws, size_t ws_bytes,
                       void* stream) {
  using namespace gs;
  if (!groups || !cfg || n_groups < 1 || n_groups > GS_MAX_GROUPS || !clock || !stats_out ||
      max_rows < 0 || max_rows >= (int64_t)INT32_MAX) {
    gs_set_error("gs_step: invalid arguments");
    return GS_ERR_ARG;
  }
  if (cfg->mode < GS_MODE_COUPLED_ADAM || cfg->mode > GS_MODE_ADAMW_GS) {
    gs_set_error("gs_step: unknown mode %d", cfg->mode);
    return GS_ERR_ARG;
  }
  const bool dense = cfg->mode == GS_MODE_COUPLED_ADAM;
  if (!dense && (!rows || !n_rows_dev)) {
    gs_set_error("gs_step: sparse modes need the index list and its device count");
    return GS_ERR_ARG;
  }
  if (cfg->check == GS_CHECK_STRICT && !cfg->abort_flag) {
    gs_set_error("gs_step: strict check needs abort_flag");
    return GS_ERR_ARG;
  }
  if (!cfg->bias_lut || cfg->lut_len < 2) {
    gs_set_error("gs_step: bias-correction LUT missing");
    return GS_ERR_ARG;
  }
  if (cfg->mode == GS_MODE_ADAMW_GS && !(cfg->n_pixels_rounded > 0.0)) {
    gs_set_error("gs_step: adamw-gs needs N_I' > 0");
    return GS_ERR_ARG;
  }
  if (!ws || ws_bytes < gs_step_workspace_bytes()) {
    gs_set_error("gs_step: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  StepParams P{};
  for (int i = 0; i < n_groups; ++i) {
    const gs_group& g = groups[i];
    if (!g.param || !g.grad || !g.exp_avg || !g.exp_avg_sq || g.width < 1 || g.width > 4096 ||
        (g.param_stride != 0 && g.param_stride < g.width) ||
        (g.grad_stride != 0 && g.grad_stride < g.width)) {
      gs_set_error("gs_step: group %d invalid", i);
      return GS_ERR_ARG;
    }
    P.g[i] = GroupDev{g.param, g.grad, g.exp_avg, g.exp_avg_sq, (int)g.width, g.role, g.lr, 0,
                      g.param_stride ? g.param_stride : g.width,
                      g.grad_stride ? g.grad_stride : g.width};
  }
  P.n_groups = n_groups;
  P.check = cfg->check;
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
    gs_set_error("gs_step: bad densification-statistics arguments");
    return GS_ERR_ARG;
  }
  P.rows = rows;
  P.n_rows_dev = n_rows_dev;
  P.max_rows = max_rows;
  P.clock = clock;
  P.stats_out = stats_out;
  auto* hdr = reinterpret_cast<StepWorkspace*>(ws);
  P.counter = &hdr->counter;
  P.partials = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + sizeof(StepWorkspace));

  const int64_t chunks = (max_rows + kThreads - 1) / kThreads;
  int grid = (int)std::min<int64_t>(std::max<int64_t>(chunks, 1), max_step_blocks());
  cudaStream_t s = (cudaStream_t)stream;
  if (cfg->check == GS_CHECK_STRICT)
    launch_dispatch<true>(cfg->mode, P, grid, s);
  else
    launch_dispatch<false>(cfg->mode, P, grid, s);
  return gs_check_launch("gs_step");
}
