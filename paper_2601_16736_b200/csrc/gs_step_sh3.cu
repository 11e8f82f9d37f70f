// K2 fast path — the fused AdamW-GS step specialised at compile time for a
// fixed attribute layout (3DGS SH-3: xyz 3 | f_dc 3 | f_rest 45 | opacity 1 |
// scaling 3 | rotation 4), row-record optimizer state (gs_step_rows.cu).
//
// One warp owns a chunk of 32 visible rows.  Every loop below is unrolled
// over the compile-time layout, so roles, widths, record offsets and the
// penalty code paths cost no branches:
//
//   pass A  lane l loads, for every group g and k < W_g, the gradient of
//           element e = 32k + l of the chunk's (row, column) sequence of g
//           (row e / W_g, column e % W_g) — 59 coalesced loads per lane kept
//           in registers — plus theta of the opacity / scale elements, and
//           ORs a per-row bad mask (non-finite gradient, tau / kappa outside
//           the activation domain where a penalty is active).  One warp
//           reduction gives the 32-row validity mask: no gradient is read
//           twice and no row is partially written.
//   clocks  lane r bumps the clock of row r and fetches its bias factors.
//   pass B  group by group, batches of elements: load theta and the (m, v)
//           pair from the record, update (gs_common.cuh::update_element,
//           bit-identical to oracle step_fp32), store.  The opacity group has
//           exactly one element per lane and the scale group three, so the
//           DAR terms are computed lane-parallel.
#include <stdlib.h>

#include "gs_common.cuh"

namespace gs {

struct LayoutSH3 {
  static constexpr int G = 6;
  static constexpr int P = 59;
  __host__ __device__ static constexpr int W(int i) {
    return i == 2 ? 45 : i == 3 ? 1 : i == 5 ? 4 : 3;
  }
  __host__ __device__ static constexpr int OFF(int i) {
    return i == 0 ? 0 : i == 1 ? 3 : i == 2 ? 6 : i == 3 ? 51 : i == 4 ? 52 : 55;
  }
  __host__ __device__ static constexpr int ROLE(int i) {
    return i == 0 ? GS_ROLE_POSITION : i == 3 ? GS_ROLE_OPACITY : i == 4 ? GS_ROLE_SCALE
                                                                         : GS_ROLE_PLAIN;
  }
};

struct FixedGroup {
  float* param;
  const float* grad;
  float lr;
  int pad;
};

struct FixedParams {
  FixedGroup g[GS_MAX_GROUPS];
  float active_logit;
  StepConsts K;
  const float* lut;
  int lut_len;
  int global_t;
  const int32_t* nv_dev;
  double nv_host;
  const int32_t* abort_flag;
  const int32_t* rows;
  const int32_t* n_rows_dev;
  int64_t max_rows;
  float* record;
  int64_t stride;
  double* stats_out;
  double* partials;
  unsigned int* counter;
};

constexpr int kFixedThreads = 256;

// Element i of a chunk of R rows, enumerated group-major:
//   [group 0: R x W_0][group 1: R x W_1] ... ; group g starts at R * OFF_g.
// With R a multiple of 32 every group boundary is a multiple of 32, so the
// group of i is uniform across a warp.
template <class L>
__device__ __forceinline__ int group_of(int i, int R) {
  int g = 0;
#pragma unroll
  for (int k = 1; k < L::G; ++k) g += (i >= R * L::OFF(k)) ? 1 : 0;
  return g;
}

template <class L, int MODE, bool STRICT, int R, int MINB>
__global__ void __launch_bounds__(kFixedThreads, MINB) step_fixed_kernel(const FixedParams P) {
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NT = kFixedThreads;
  constexpr int E = R * L::P;              // elements per chunk
  constexpr int J = (E + NT - 1) / NT;     // elements per thread per chunk
  __shared__ int32_t s_row[R];
  __shared__ int s_bad[R];
  __shared__ float2 s_bc[R];
  __shared__ double s_red[GS_STEP_STATS * (NT / 32)];

  const int t = threadIdx.x;
  int64_t n_rows = kDense ? P.max_rows : (int64_t)(*P.n_rows_dev);
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  StepConsts Kc = P.K;
  if (kCoupled) {
    const float nv = P.nv_dev ? (float)(*P.nv_dev) : (float)P.nv_host;
    Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
    if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
  }
  const StepConsts& K = kCoupled ? Kc : P.K;

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  const int64_t n_chunks = (n_rows + R - 1) / R;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const int64_t base = chunk * R;
    const int nvalid = (int)(n_rows - base < R ? n_rows - base : R);
    __syncthreads();  // previous chunk's shared-memory readers are done
    int32_t my_row = 0;
    int my_clock = 0;
    if (t < R) {
      my_row = t < nvalid ? (kDense ? (int32_t)(base + t) : __ldg(P.rows + base + t)) : 0;
      s_row[t] = my_row;
      s_bad[t] = t < nvalid ? 0 : 4;
      if (t < nvalid)
        my_clock = reinterpret_cast<const int*>(P.record + (int64_t)my_row * P.stride)[2 * L::P];
    }
    __syncthreads();

    // ---- phase L: issue every load of this thread's elements ----------------
    float th[J], gr[J];
    float2 mv[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int i = t + NT * j;
      th[j] = gr[j] = 0.f;
      mv[j] = make_float2(0.f, 0.f);
      if (i < E) {
        const int g = group_of<L>(i, R);
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          if (g == gg) {
            const int W = L::W(gg);
            const int local = i - R * L::OFF(gg);
            const int r = local / W;
            const int c = local - r * W;
            if (r < nvalid) {
              const int32_t row = s_row[r];
              const int64_t off = (int64_t)row * W + c;
              th[j] = P.g[gg].param[off];
              gr[j] = __ldg(P.g[gg].grad + off);
              mv[j] = reinterpret_cast<const float2*>(P.record + (int64_t)row * P.stride)[L::OFF(gg) + c];
            }
          }
        }
      }
    }
    // bias factors of the clock after this step (used only if the row is valid)
    float2 my_bc = make_float2(1.f, 1.f);
    if (t < nvalid)
      my_bc = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : my_clock + 1, 0.0, 0.0);

    // ---- validity: non-finite gradient (bit 0), activation domain (bit 1) -----
    if (!STRICT) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int i = t + NT * j;
        if (i < E) {
          const int g = group_of<L>(i, R);
#pragma unroll
          for (int gg = 0; gg < L::G; ++gg) {
            if (g == gg) {
              const int W = L::W(gg);
              const int local = i - R * L::OFF(gg);
              const int r = local / W;
              const int role = L::ROLE(gg);
              const float lam = role == GS_ROLE_OPACITY ? K.lam_op
                                : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
              int bad = isfinite(gr[j]) ? 0 : 1;
              if (lam != 0.f && domain_bad(role, th[j])) bad |= 2;
              if (r < nvalid && bad) atomicOr(&s_bad[r], bad);
            }
          }
        }
      }
    }
    __syncthreads();
    if (t < nvalid) {
      ++c_vis;
      const int bad = s_bad[t];
      if (bad == 0) {
        reinterpret_cast<int*>(P.record + (int64_t)my_row * P.stride)[2 * L::P] = my_clock + 1;
        s_bc[t] = my_bc;
        ++c_step;
      } else if (bad & 1) {
        ++c_badg;
      } else {
        ++c_badd;
      }
    }
    __syncthreads();

    // ---- phase U: update and store ----------------------------------------------
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int i = t + NT * j;
      if (i < E) {
        const int g = group_of<L>(i, R);
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          if (g == gg) {
            const int W = L::W(gg);
            const int role = L::ROLE(gg);
            const int local = i - R * L::OFF(gg);
            const int r = local / W;
            const int c = local - r * W;
            if (r < nvalid && s_bad[r] == 0) {
              const int32_t row = s_row[r];
              float tn, mn, vn, ex;
              bool clipped;
              update_element<MODE>(role, P.g[gg].lr, th[j], gr[j], mv[j].x, mv[j].y, s_bc[r], K,
                                   tn, mn, vn, ex, clipped);
              if (!kCoupled && role == GS_ROLE_OPACITY) {
                c_clo += clipped;
                s_exo += (double)ex;
              } else if (!kCoupled && role == GS_ROLE_SCALE) {
                c_cls += clipped;
                s_exs += (double)ex;
              }
              if (role == GS_ROLE_OPACITY) {
                c_apre += th[j] > P.active_logit;
                c_apost += tn > P.active_logit;
              }
              P.g[gg].param[(int64_t)row * W + c] = tn;
              reinterpret_cast<float2*>(P.record + (int64_t)row * P.stride)[L::OFF(gg) + c] =
                  make_float2(mn, vn);
            }
          }
        }
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
  if (last_block_arrive(P.counter)) {
    if (threadIdx.x < GS_STEP_STATS) {
      double s = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b)
        s += P.partials[(size_t)b * GS_STEP_STATS + threadIdx.x];
      P.stats_out[threadIdx.x] = s;
    }
  }
}

static int g_fixed_variant = -1;

int fixed_variant() {
  if (g_fixed_variant < 0) {
    const char* e = getenv("GS_FIXED_VARIANT");
    g_fixed_variant = e ? atoi(e) : 0;
  }
  return g_fixed_variant;
}

template <class L, int MODE, bool STRICT, int R, int MINB>
void launch_fixed_v(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_fixed_kernel<L, MODE, STRICT, R, MINB><<<grid, kFixedThreads, 0, s>>>(P);
}

template <class L, int MODE, bool STRICT>
void launch_fixed(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  switch (fixed_variant()) {
    case 1: launch_fixed_v<L, MODE, STRICT, 32, 4>(P, max_rows, s); return;
    case 2: launch_fixed_v<L, MODE, STRICT, 32, 3>(P, max_rows, s); return;
    case 3: launch_fixed_v<L, MODE, STRICT, 64, 3>(P, max_rows, s); return;
    default: launch_fixed_v<L, MODE, STRICT, 64, 2>(P, max_rows, s); return;
  }
}

template <class L, bool STRICT>
void dispatch_fixed(int mode, const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  switch (mode) {
    case GS_MODE_COUPLED_ADAM: launch_fixed<L, GS_MODE_COUPLED_ADAM, STRICT>(P, max_rows, s); break;
    case GS_MODE_SPARSE_ADAM: launch_fixed<L, GS_MODE_SPARSE_ADAM, STRICT>(P, max_rows, s); break;
    case GS_MODE_ADAMW_CONST: launch_fixed<L, GS_MODE_ADAMW_CONST, STRICT>(P, max_rows, s); break;
    case GS_MODE_ADAMW_CONST_CLIP:
      launch_fixed<L, GS_MODE_ADAMW_CONST_CLIP, STRICT>(P, max_rows, s);
      break;
    default: launch_fixed<L, GS_MODE_ADAMW_GS, STRICT>(P, max_rows, s); break;
  }
}

template <class L>
bool layout_matches(const gs_group* groups, int n_groups) {
  if (n_groups != L::G) return false;
  for (int i = 0; i < L::G; ++i) {
    if (groups[i].width != L::W(i) || groups[i].role != L::ROLE(i)) return false;
  }
  return true;
}

}  // namespace gs

// Called by gs_step_rows (gs_step_rows.cu) after argument validation; returns
// 1 if a compiled fixed layout handled the launch, 0 otherwise.
int gs_step_fixed_try(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                      const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                      float* record, int64_t record_stride, double* stats_out, double* partials,
                      unsigned int* counter, void* stream) {
  using namespace gs;
  const char* off = getenv("GS_DISABLE_FIXED");
  if (off && off[0] == '1') return 0;
  if (!layout_matches<LayoutSH3>(groups, n_groups)) return 0;
  FixedParams P{};
  for (int i = 0; i < n_groups; ++i)
    P.g[i] = FixedGroup{groups[i].param, groups[i].grad, groups[i].lr, 0};
  P.active_logit = cfg->active_logit;
  P.K = make_consts(cfg);
  P.lut = cfg->bias_lut;
  P.lut_len = cfg->lut_len;
  P.global_t = cfg->global_t;
  P.nv_dev = cfg->n_visible_norm;
  P.nv_host = cfg->n_visible_host;
  P.abort_flag = cfg->abort_flag;
  P.rows = rows;
  P.n_rows_dev = n_rows_dev;
  P.max_rows = max_rows;
  P.record = record;
  P.stride = record_stride;
  P.stats_out = stats_out;
  P.partials = partials;
  P.counter = counter;
  cudaStream_t s = (cudaStream_t)stream;
  if (cfg->check == GS_CHECK_STRICT)
    dispatch_fixed<LayoutSH3, true>(cfg->mode, P, max_rows, s);
  else
    dispatch_fixed<LayoutSH3, false>(cfg->mode, P, max_rows, s);
  return 1;
}
