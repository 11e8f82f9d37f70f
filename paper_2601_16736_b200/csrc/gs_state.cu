// State kernels around the step:
//   gs_check_grads  strict all-row finite check (gradients.py:50-58,
//                   optimizer.py:181-184) + visible-row activation domain
//                   (primitives.py:44-48,78-84)
//   gs_rsr_apply    re-state regularisation (optimizer.py:327-340)
//   gs_reset_rows   relocation reset (optimizer.py:159-165)
//   gs_stats_all    classify_active + moment_stats (primitives.py:228-238,
//                   optimizer.py:489-506)
#include "gs_common.cuh"

namespace gs {

struct GroupPtrs {
  float* param;
  const float* grad;
  float* m;
  float* v;
  int width;
  int role;
  float lr;
  int64_t ps;  // param row stride (elements)
  int64_t gs;  // grad row stride
};

__host__ __forceinline__ GroupPtrs group_ptrs(const gs_group& g, bool with_grad, bool with_state,
                                              float lr) {
  return GroupPtrs{g.param, with_grad ? g.grad : nullptr, with_state ? g.exp_avg : nullptr,
                   with_state ? g.exp_avg_sq : nullptr, (int)g.width, g.role, lr,
                   g.param_stride ? g.param_stride : g.width,
                   g.grad_stride ? g.grad_stride : g.width};
}

static bool strides_ok(const gs_group& g) {
  return (g.param_stride == 0 || g.param_stride >= g.width) &&
         (g.grad_stride == 0 || g.grad_stride >= g.width);
}

struct GroupSet {
  GroupPtrs g[GS_MAX_GROUPS];
  int n;
};

static int fill_groups(const gs_group* groups, int32_t n_groups, GroupSet& S, const char* who,
                       bool need_grad, bool need_state = true) {
  if (!groups || n_groups < 1 || n_groups > GS_MAX_GROUPS) {
    gs_set_error("%s: bad group list", who);
    return GS_ERR_ARG;
  }
  S.n = n_groups;
  for (int i = 0; i < n_groups; ++i) {
    const gs_group& g = groups[i];
    if ((need_state && (!g.exp_avg || !g.exp_avg_sq)) || (need_grad && !g.grad) || g.width < 1 ||
        g.width > 4096 || !strides_ok(g)) {
      gs_set_error("%s: group %d invalid", who, i);
      return GS_ERR_ARG;
    }
    S.g[i] = group_ptrs(g, true, true, g.lr);
  }
  return GS_OK;
}

// ---------------------------------------------------------------------------
// strict check: one flat pass per group over all n_rows * width gradients
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mark_row(uint8_t* bad_rows, int64_t row, int bad) {
  atomicOr(reinterpret_cast<unsigned int*>(bad_rows + (row & ~3ll)),
           (unsigned int)bad << (8 * (row & 3)));
}

// grec != nullptr: the gradients of all groups form one row record (group g
// at column offset sum of the earlier widths, row stride grs, 16-byte rows):
// the finite check is one pass with 16-byte loads, `lpr` lanes per row (a
// power of two >= the row's 16-byte pieces), no index division.  Otherwise
// each group is checked on its own: dense groups as one flat array (the row
// is derived only for a non-finite value), strided groups element-wise.
__global__ void __launch_bounds__(kThreads)
    check_grads_kernel(const GroupSet S, int64_t n_rows, const int32_t* __restrict__ rows,
                       const int32_t* __restrict__ n_list_dev, double lam_op, double lam_sc,
                       uint8_t* __restrict__ bad_rows, int32_t* __restrict__ abort_flag,
                       const float* __restrict__ grec, int64_t grs, int P, int lpr) {
  int flag = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_list = rows ? (int64_t)(*n_list_dev) : 0;
  if (grec) {
    const int lane = threadIdx.x & 31;
    const int sub = lane / lpr;           // row within the warp's group of rows
    const int q0 = lane - sub * lpr;      // first 16-byte piece of this lane
    const int rows_per_warp = 32 / lpr;
    const int64_t warps = stride / 32;
    const int nq = (P + 3) / 4;
    constexpr int U = 4;  // row groups in flight per warp
    const int64_t step = warps * rows_per_warp;
    for (int64_t r0 = (tid0 / 32) * rows_per_warp; r0 < n_rows; r0 += U * step) {
      float4 x[U];
      int64_t row[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // issue all loads first
        row[u] = r0 + u * step + sub;
        x[u] = (row[u] < n_rows && q0 < nq)
                   ? __ldg(reinterpret_cast<const float4*>(grec + row[u] * grs) + q0)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (row[u] >= n_rows) continue;
        const float* rp = grec + row[u] * grs;
        int bad = 0;
        for (int q = q0; q < nq; q += lpr) {  // one pass unless a row has > 32 pieces
          const float4 y = q == q0 ? x[u] : __ldg(reinterpret_cast<const float4*>(rp) + q);
          const int c = 4 * q;
          bad |= !isfinite(y.x) | ((c + 1 < P) & !isfinite(y.y)) |
                 ((c + 2 < P) & !isfinite(y.z)) | ((c + 3 < P) & !isfinite(y.w));
        }
        if (bad) {
          flag |= 1;
          if (bad_rows) mark_row(bad_rows, row[u], 1);
        }
      }
    }
  }
  for (int gi = 0; gi < S.n; ++gi) {
    const GroupPtrs G = S.g[gi];
    const int W = G.width;
    const int64_t total = grec ? 0 : n_rows * W;
    if (G.gs == W) {
      // dense: 16-byte loads from the first aligned element, 4 in flight per thread
      const int64_t head = total == 0 ? 0 :
          std::min<int64_t>(total, (16 - (reinterpret_cast<uintptr_t>(G.grad) & 15u)) / 4 & 3);
      const int64_t nq4 = (total - head) / 4;
      const float4* g4 = reinterpret_cast<const float4*>(G.grad + head);
      auto check_elem = [&](int64_t e, float val) {
        if (!isfinite(val)) {
          flag |= 1;
          if (bad_rows) mark_row(bad_rows, e / W, 1);
        }
      };
      for (int64_t e = tid0; e < head; e += stride) check_elem(e, __ldg(G.grad + e));
      for (int64_t q = tid0; q < nq4; q += 4 * stride) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = q + u * stride < nq4 ? __ldg(g4 + q + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!(isfinite(x[u].x) && isfinite(x[u].y) && isfinite(x[u].z) && isfinite(x[u].w))) {
            const int64_t e = head + 4 * (q + u * stride);
            check_elem(e, x[u].x);
            check_elem(e + 1, x[u].y);
            check_elem(e + 2, x[u].z);
            check_elem(e + 3, x[u].w);
          }
        }
      }
      for (int64_t e = head + 4 * nq4 + tid0; e < total; e += stride) check_elem(e, __ldg(G.grad + e));
    } else {
      for (int64_t e = tid0; e < total; e += stride) {
        const int64_t row = e / W;
        if (!isfinite(__ldg(G.grad + row * G.gs + (e - row * W)))) {
          flag |= 1;
          if (bad_rows) mark_row(bad_rows, row, 1);
        }
      }
    }
    const double lam = G.role == GS_ROLE_OPACITY ? lam_op : G.role == GS_ROLE_SCALE ? lam_sc : 0.0;
    if (lam != 0.0 && G.param != nullptr) {
      const int64_t tot = n_list * W;
      const bool narrow = tot < (int64_t)UINT32_MAX;  // 32-bit index arithmetic
      for (int64_t e = tid0; e < tot; e += stride) {
        const int64_t li = narrow ? (int64_t)((uint32_t)e / (uint32_t)W) : e / W;
        const int64_t row = __ldg(rows + li);
        if (domain_bad(G.role, G.param[row * G.ps + (e - li * W)])) {
          flag |= 2;
          if (bad_rows) mark_row(bad_rows, row, 2);
        }
      }
    }
  }
  flag = __reduce_or_sync(0xffffffffu, flag);
  if ((threadIdx.x & 31) == 0 && flag) atomicOr(abort_flag, flag);
}

// ---------------------------------------------------------------------------
// RSR / reset: chunk of kThreads rows per CTA, flattened (row, col) per group
// ---------------------------------------------------------------------------
template <bool RESET>
__global__ void __launch_bounds__(kThreads)
    scatter_state_kernel(const GroupSet S, const int32_t* __restrict__ rows, int64_t k,
                         int64_t n_rows, double a1, double a2, int32_t* __restrict__ clock) {
  __shared__ int32_t s_row[kThreads];
  const int tid = threadIdx.x;
  const int64_t n_chunks = (k + kThreads - 1) / kThreads;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const int64_t base = chunk * kThreads;
    const int nvalid = (int)(k - base < kThreads ? k - base : kThreads);
    if (tid < nvalid) {
      const int32_t r = __ldg(rows + base + tid);
      const bool ok = r >= 0 && (int64_t)r < n_rows;  // ids outside the rows are skipped
      s_row[tid] = ok ? r : -1;
      if (RESET && clock && ok) clock[r] = 0;
    }
    __syncthreads();
    for (int gi = 0; gi < S.n; ++gi) {
      const GroupPtrs G = S.g[gi];
      const int W = G.width;
      const int E = nvalid * W;
      const int dq = kThreads / W, dr = kThreads % W;
      int lr = tid / W, lc = tid % W;
      for (int e = tid; e < E; e += kThreads) {
        const int64_t off = (int64_t)s_row[lr] * W + lc;
        if (s_row[lr] < 0) {
        } else if (RESET) {
          G.m[off] = 0.0f;
          G.v[off] = 0.0f;
        } else {
          // m *= alpha1 in float64, rounded once (optimizer.py:338-339)
          G.m[off] = __double2float_rn(__dmul_rn((double)G.m[off], a1));
          G.v[off] = __double2float_rn(__dmul_rn((double)G.v[off], a2));
        }
        lc += dr;
        lr += dq;
        if (lc >= W) { lc -= W; ++lr; }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// all-row statistics
// ---------------------------------------------------------------------------
constexpr int kStatsFields = 2 + 5 * GS_MAX_GROUPS;

struct StatsWorkspace {
  unsigned int counter;
  unsigned int pad[15];
};

__global__ void __launch_bounds__(kThreads)
    stats_all_kernel(const GroupSet S, int64_t n_rows, const uint8_t* __restrict__ alive,
                     float active_logit, double* __restrict__ out, double* partials,
                     unsigned int* counter) {
  __shared__ double s_red[kStatsFields * (kThreads / 32)];
  double acc[kStatsFields];
  bool is_max[kStatsFields];
#pragma unroll
  for (int f = 0; f < kStatsFields; ++f) {
    acc[f] = 0.0;
    is_max[f] = f >= 2 && (((f - 2) % 5) == 1 || ((f - 2) % 5) == 4);
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t r = tid0; r < n_rows; r += stride) {
    const bool al = alive == nullptr || alive[r] != 0;
    acc[0] += al;
  }
#pragma unroll
  for (int gi = 0; gi < GS_MAX_GROUPS; ++gi) {
    if (gi >= S.n) break;
    const GroupPtrs G = S.g[gi];
    const int64_t total = n_rows * G.width;
    double s_sq = 0.0, m_sq = 0.0, n_pos = 0.0, s_rt = 0.0, m_rt = 0.0;
    for (int64_t e = tid0; e < total; e += stride) {
      if (alive != nullptr && alive[e / G.width] == 0) continue;
      const double vv = (double)__ldg(G.v + e);
      const double sq = sqrt(vv);
      s_sq += sq;
      m_sq = fmax(m_sq, sq);
      if (sq > 0.0) {
        const double rt = __ddiv_rn(fabs((double)__ldg(G.m + e)), sq);
        n_pos += 1.0;
        s_rt += rt;
        m_rt = fmax(m_rt, rt);
      }
      if (G.role == GS_ROLE_OPACITY && G.width == 1 && G.param != nullptr)
        acc[1] += __ldg(G.param + e * G.ps) > active_logit;
    }
    acc[2 + 5 * gi + 0] = s_sq;
    acc[2 + 5 * gi + 1] = m_sq;
    acc[2 + 5 * gi + 2] = n_pos;
    acc[2 + 5 * gi + 3] = s_rt;
    acc[2 + 5 * gi + 4] = m_rt;
  }
  block_reduce<kStatsFields>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
    for (int f = 0; f < kStatsFields; ++f) partials[(size_t)blockIdx.x * kStatsFields + f] = acc[f];
  }
  if (last_block_arrive(counter)) {
    double tmp[kStatsFields];
    final_reduce<kStatsFields>(partials, gridDim.x, kStatsFields, tmp, is_max, s_red);
    if (threadIdx.x == 0)
      for (int f = 0; f < 2 + 5 * S.n; ++f) out[f] = tmp[f];
  }
}

int stats_blocks() { return gs_sm_count() * 3; }

// ---------------------------------------------------------------------------
// row-record state (see gs_step_rows.cu): slot s < P holds (m, v), slot P the
// int32 clock.  A warp owns a row; lanes stride over its slots.
// ---------------------------------------------------------------------------
template <bool RESET, bool VEC4>
__global__ void __launch_bounds__(kThreads)
    scatter_rows_kernel(float* __restrict__ record, int64_t stride, int P,
                        const int32_t* __restrict__ rows, int64_t k, int64_t n_rows, double a1,
                        double a2) {
  // VEC4: a lane moves one 16-byte piece (two slots) of a row, so a row is
  // one warp-wide access of 8(P+1) bytes; RPI rows per warp iteration keep
  // RPI rows' loads in flight before any store.  Ids outside [0, n_rows)
  // are skipped.
  constexpr int RPI = VEC4 ? 4 : 2;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  auto one = [&](float* rec, int s) {  // float2 slot s
    float2* p = reinterpret_cast<float2*>(rec + 2 * s);
    if (RESET) {
      if (s < P) *p = make_float2(0.f, 0.f);
      else if (s == P) reinterpret_cast<int*>(rec)[2 * s] = 0;  // clock = 0, pad kept
    } else if (s < P) {
      const float2 x = *p;  // m *= alpha1 in float64, rounded once (optimizer.py:338-339)
      *p = make_float2(__double2float_rn(__dmul_rn((double)x.x, a1)),
                       __double2float_rn(__dmul_rn((double)x.y, a2)));
    }
  };
  const int nq = (P + 1) / 2;  // 16-byte pieces of a row (VEC4: P + 1 even)
  const int s = 2 * lane;      // VEC4: first slot of the lane's piece
  for (int64_t i0 = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * RPI; i0 < k;
       i0 += RPI * warps) {
    float* rec[RPI];
    bool ok[RPI];
#pragma unroll
    for (int u = 0; u < RPI; ++u) {
      const int64_t r = i0 + u < k ? (int64_t)__ldg(rows + i0 + u) : -1;
      ok[u] = r >= 0 && r < n_rows;
      rec[u] = record + (ok[u] ? r : 0) * stride;
    }
    if (VEC4) {
      if (lane >= nq) continue;
      if (RESET) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          if (!ok[u]) continue;
          if (s + 1 < P) {
            reinterpret_cast<float4*>(rec[u])[lane] = z;
          } else {
            one(rec[u], s);
            one(rec[u], s + 1);
          }
        }
      } else {
        float4 x[RPI];
#pragma unroll
        for (int u = 0; u < RPI; ++u)
          x[u] = ok[u] ? reinterpret_cast<const float4*>(rec[u])[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          if (!ok[u]) continue;
          float4 y = x[u];
          y.x = __double2float_rn(__dmul_rn((double)x[u].x, a1));
          y.y = __double2float_rn(__dmul_rn((double)x[u].y, a2));
          if (s + 1 < P) {
            y.z = __double2float_rn(__dmul_rn((double)x[u].z, a1));
            y.w = __double2float_rn(__dmul_rn((double)x[u].w, a2));
          }  // else slot P (clock, pad) is written back unchanged
          reinterpret_cast<float4*>(rec[u])[lane] = y;
        }
      }
    } else {
      for (int sl = lane; sl <= P; sl += 32) {
#pragma unroll
        for (int u = 0; u < RPI; ++u)
          if (ok[u]) one(rec[u], sl);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    stats_rows_kernel(const GroupSet S, const float* __restrict__ record, int64_t stride,
                      int64_t n_rows, const uint8_t* __restrict__ alive, float active_logit,
                      double* __restrict__ out, double* partials, unsigned int* counter) {
  __shared__ double s_red[kStatsFields * (kThreads / 32)];
  double acc[kStatsFields];
  bool is_max[kStatsFields];
#pragma unroll
  for (int f = 0; f < kStatsFields; ++f) {
    acc[f] = 0.0;
    is_max[f] = f >= 2 && (((f - 2) % 5) == 1 || ((f - 2) % 5) == 4);
  }
  const int64_t stride_t = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t r = tid0; r < n_rows; r += stride_t) acc[0] += alive == nullptr || alive[r] != 0;
  int off = 0;
#pragma unroll
  for (int gi = 0; gi < GS_MAX_GROUPS; ++gi) {
    if (gi >= S.n) break;
    const GroupPtrs G = S.g[gi];
    const int W = G.width;
    const int64_t total = n_rows * W;
    double s_sq = 0.0, m_sq = 0.0, n_pos = 0.0, s_rt = 0.0, m_rt = 0.0;
    for (int64_t e = tid0; e < total; e += stride_t) {
      const int64_t row = e / W;
      const int col = (int)(e - row * W);
      if (alive != nullptr && alive[row] == 0) continue;
      const float2 x = __ldg(reinterpret_cast<const float2*>(record + row * stride + 2 * (off + col)));
      const double sq = sqrt((double)x.y);
      s_sq += sq;
      m_sq = fmax(m_sq, sq);
      if (sq > 0.0) {
        const double rt = __ddiv_rn(fabs((double)x.x), sq);
        n_pos += 1.0;
        s_rt += rt;
        m_rt = fmax(m_rt, rt);
      }
      if (G.role == GS_ROLE_OPACITY && W == 1 && G.param != nullptr)
        acc[1] += __ldg(G.param + row * G.ps) > active_logit;
    }
    acc[2 + 5 * gi + 0] = s_sq;
    acc[2 + 5 * gi + 1] = m_sq;
    acc[2 + 5 * gi + 2] = n_pos;
    acc[2 + 5 * gi + 3] = s_rt;
    acc[2 + 5 * gi + 4] = m_rt;
    off += W;
  }
  block_reduce<kStatsFields>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
    for (int f = 0; f < kStatsFields; ++f) partials[(size_t)blockIdx.x * kStatsFields + f] = acc[f];
  }
  if (last_block_arrive(counter)) {
    double tmp[kStatsFields];
    final_reduce<kStatsFields>(partials, gridDim.x, kStatsFields, tmp, is_max, s_red);
    if (threadIdx.x == 0)
      for (int f = 0; f < 2 + 5 * S.n; ++f) out[f] = tmp[f];
  }
}

// One-pass K4 on the row record: a warp reads 4 consecutive record rows per
// iteration (4 x 8(P+1) contiguous bytes in flight per warp; lane q takes
// the 16-byte piece of slots 2q, 2q+1 of each), so nothing is divided by a
// width.  A lane's slots belong to fixed groups across rows, so it keeps
// J x 2 accumulator sets; the block folds them in a fixed (warp, lane)
// order and the last CTA folds the blocks: deterministic for a given grid.
// sqrt(v) and |m| / sqrt(v) come from a float64 reciprocal square root
// (fp32 seed + two Newton steps, ~1 ulp of float64) instead of float64
// sqrt and division: the statistics agree with the reference's float64
// values to ~1e-16 relative at a fraction of the float64 instruction cost.
__device__ __forceinline__ double rsqrt_f64(float vf) {
  const double v = (double)vf;
  double r = (double)rsqrtf(vf);
  r = r * fma(-0.5 * v * r, r, 1.5);
  r = r * fma(-0.5 * v * r, r, 1.5);
  return r;
}

template <int J>
__global__ void __launch_bounds__(kThreads, 3)  // 3 CTAs/SM: 0.82 ms on c3 (2: 1.02, 4: 0.90)
    stats_rows_vec_kernel(const GroupSet S, int P, const float* __restrict__ record,
                          int64_t stride, int64_t n_rows, const uint8_t* __restrict__ alive,
                          float active_logit, double* __restrict__ out, double* partials,
                          unsigned int* counter) {
  constexpr int NW = kThreads / 32;
  constexpr int NF = 5;  // sum sqrt v, max sqrt v, n(v > 0), sum |m|/sqrt v, max |m|/sqrt v
  constexpr int RPI = 4;  // record rows per warp iteration
  __shared__ signed char s_grp[128];
  __shared__ double s_acc[NW][32][2 * J][NF];
  __shared__ double s_red[kStatsFields * NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 128) {
    int g = -1, off = 0;
    for (int i = 0; i < S.n; ++i) {
      if ((int)threadIdx.x >= off && (int)threadIdx.x < off + S.g[i].width) g = i;
      off += S.g[i].width;
    }
    s_grp[threadIdx.x] = (signed char)((int)threadIdx.x < P ? g : -1);
  }
  __syncthreads();
  int opac = -1;
  for (int i = 0; i < S.n; ++i)
    if (S.g[i].role == GS_ROLE_OPACITY && S.g[i].width == 1 && S.g[i].param != nullptr) opac = i;
  double a[2 * J][NF];
#pragma unroll
  for (int k = 0; k < 2 * J; ++k)
#pragma unroll
    for (int f = 0; f < NF; ++f) a[k][f] = 0.0;
  double n_alive = 0.0, n_active = 0.0;
  const int nq = (P + 1) / 2;  // 16-byte pieces holding slots < P
  const int64_t warps = (int64_t)gridDim.x * NW;
  for (int64_t r0 = ((int64_t)blockIdx.x * NW + warp) * RPI; r0 < n_rows; r0 += warps * RPI) {
    // every load of the iteration is independent: records, alive bytes and
    // opacities are issued together (the record rows are read whether alive
    // or not, and masked afterwards)
    float4 x[RPI][J];
    bool live[RPI];
    float tau[RPI];
#pragma unroll
    for (int i = 0; i < RPI; ++i) {
      const int64_t r = r0 + i < n_rows ? r0 + i : n_rows - 1;
      const float4* row = reinterpret_cast<const float4*>(record + r * stride);
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int q = lane + 32 * j;
        x[i][j] = q < nq ? __ldg(row + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      live[i] = r0 + i < n_rows && (alive == nullptr || alive[r] != 0);
      tau[i] = opac >= 0 ? __ldg(S.g[opac].param + r * S.g[opac].ps) : 0.f;
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < RPI; ++i) {
        if (!live[i]) continue;
        n_alive += 1.0;
        n_active += tau[i] > active_logit;
      }
    }
#pragma unroll
    for (int i = 0; i < RPI; ++i) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int q = lane + 32 * j;
        const float mm[2] = {x[i][j].x, x[i][j].z}, vv[2] = {x[i][j].y, x[i][j].w};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!live[i] || q >= nq || 2 * q + h >= P) continue;
          double* A = a[2 * j + h];
          if (vv[h] > 0.0f) {
            const double rs = rsqrt_f64(vv[h]);
            const double sq = (double)vv[h] * rs;
            const double rt = fabs((double)mm[h]) * rs;
            A[0] += sq;
            A[1] = fmax(A[1], sq);
            A[2] += 1.0;
            A[3] += rt;
            A[4] = fmax(A[4], rt);
          } else if (vv[h] != 0.0f) {  // negative / NaN v: the reference's sqrt gives NaN
            const double sq = sqrt((double)vv[h]);
            A[0] += sq;
            A[1] = fmax(A[1], sq);
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2 * J; ++k)
#pragma unroll
    for (int f = 0; f < NF; ++f) s_acc[warp][lane][k][f] = a[k][f];
  n_alive = warp_sum(n_alive);
  n_active = warp_sum(n_active);
  if (lane == 0) {
    s_red[warp] = n_alive;
    s_red[NW + warp] = n_active;
  }
  __syncthreads();
  // block fold: thread f owns output field f and walks (warp, lane, set) in
  // a fixed order
  const int nf = 2 + 5 * S.n;
  if ((int)threadIdx.x < nf) {
    const int f = threadIdx.x;
    double o = 0.0;
    if (f < 2) {
      for (int w = 0; w < NW; ++w) o += s_red[f * NW + w];
    } else {
      const int g = (f - 2) / 5, fld = (f - 2) % 5;
      const bool mx = fld == 1 || fld == 4;
      for (int w = 0; w < NW; ++w)
        for (int l = 0; l < 32; ++l)
#pragma unroll
          for (int k = 0; k < 2 * J; ++k) {
            const int sl = 2 * (l + 32 * (k / 2)) + (k & 1);
            if (sl < 128 && s_grp[sl] == g) {
              const double x = s_acc[w][l][k][fld];
              o = mx ? fmax(o, x) : o + x;
            }
          }
    }
    partials[(size_t)blockIdx.x * kStatsFields + f] = o;
    __threadfence();  // every writer publishes its partial before the last-block count
  } else if ((int)threadIdx.x < kStatsFields) {
    partials[(size_t)blockIdx.x * kStatsFields + threadIdx.x] = 0.0;
    __threadfence();
  }
  bool is_max[kStatsFields];
#pragma unroll
  for (int f = 0; f < kStatsFields; ++f)
    is_max[f] = f >= 2 && (((f - 2) % 5) == 1 || ((f - 2) % 5) == 4);
  if (last_block_arrive(counter)) {
    double tmp[kStatsFields];
    final_reduce<kStatsFields>(partials, gridDim.x, kStatsFields, tmp, is_max, s_red);
    if (threadIdx.x == 0)
      for (int f = 0; f < 2 + 5 * S.n; ++f) out[f] = tmp[f];
  }
}

// AIU (optimizer.py:425-450): picked invisible rows take one extra step with
// their frozen moments and clock, state untouched.  picked row i is
// inv_idx[jlist[i]]; lr_eta is fl32(lr * eta) per group (the reference does
// not apply mu_lr_scale here, optimizer.py:449).  Rows with clock 0 are
// skipped (:444).  A warp owns a row; lanes stride over its elements.
__global__ void __launch_bounds__(kThreads)
    aiu_rows_kernel(const GroupSet S, int P, float* __restrict__ record, int64_t stride,
                    const int32_t* __restrict__ inv_idx, const int32_t* __restrict__ jlist,
                    const int32_t* __restrict__ k_dev, const float* __restrict__ lut,
                    int lut_len, float eps, int32_t* __restrict__ picked_out) {
  // a warp per picked row; slot -> (group, column) from a shared table
  // (measured: interleaving 4 rows' index / clock / LUT chains per warp was
  // slower, 0.22 against 0.18 ms for 420k rows)
  __shared__ signed char s_g[128];
  __shared__ unsigned char s_c[128];
  if (threadIdx.x < 128) {
    int g = -1, c = 0, off = 0;
    for (int i = 0; i < S.n; ++i) {
      if ((int)threadIdx.x >= off && (int)threadIdx.x < off + S.g[i].width) {
        g = i;
        c = (int)threadIdx.x - off;
      }
      off += S.g[i].width;
    }
    s_g[threadIdx.x] = (signed char)g;
    s_c[threadIdx.x] = (unsigned char)c;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t k = *k_dev;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t i = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); i < k; i += warps) {
    const int32_t row = __ldg(inv_idx + __ldg(jlist + i));
    if (lane == 0 && picked_out) picked_out[i] = row;
    const float* rec = record + (int64_t)row * stride;
    const int t = reinterpret_cast<const int*>(rec)[2 * P];
    if (t <= 0) continue;  // never stepped: skipped (optimizer.py:444)
    const float2 bc = bias_factors(lut, lut_len, t, 0.0, 0.0);
    for (int sl = lane; sl < P; sl += 32) {
      const int gi = s_g[sl], c = s_c[sl];
      const float2 mv = reinterpret_cast<const float2*>(rec)[sl];
      const float mh = __fmul_rn(mv.x, bc.x);
      const float vh = __fmul_rn(mv.y, bc.y);
      const float den = __fadd_rn(__fsqrt_rn(vh), eps);
      const float upd = __fdiv_rn(__fmul_rn(S.g[gi].lr, mh), den);
      float* p = S.g[gi].param + (int64_t)row * S.g[gi].ps + c;
      *p = __fsub_rn(*p, upd);
    }
  }
}

// Densification statistics of the listed rows (DensifyStats.observe,
// pipeline.py:77-82) for the dense coupled-adam step, which updates every row
// but observes only the visible ones: thread per listed row.
__global__ void __launch_bounds__(kThreads)
    densify_rows_kernel(const float* __restrict__ grad, int64_t grad_stride, int width,
                        const int32_t* __restrict__ rows, const int32_t* __restrict__ n_list,
                        DensifyArgs D, const int32_t* __restrict__ abort_flag) {
  const int64_t n = (abort_flag && *abort_flag) ? 0 : *n_list;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads) {
    const int32_t r = __ldg(rows + i);
    densify_row(D, (uint32_t)r, grad + (int64_t)r * grad_stride, width, 1);
  }
}

static int record_args(const float* record, int64_t stride, int P, const char* who) {
  if (!record || P < 1 || stride < 2 * (P + 1) || (stride & 1) ||
      (reinterpret_cast<uintptr_t>(record) & 7u)) {
    gs_set_error("%s: bad record (stride %lld, P %d)", who, (long long)stride, P);
    return GS_ERR_ARG;
  }
  return GS_OK;
}

}  // namespace gs

static bool rows_vec4(const float* record, int64_t stride, int P) {
  return (P + 1) % 2 == 0 && stride % 4 == 0 && (reinterpret_cast<uintptr_t>(record) & 15u) == 0;
}

extern "C" int gs_rsr_apply_rows(float* record, int64_t record_stride, int32_t n_elems,
                                 const int32_t* rows, int64_t k, int64_t n_rows, double alpha1,
                                 double alpha2, void* stream) {
  using namespace gs;
  int rc = record_args(record, record_stride, n_elems, "gs_rsr_apply_rows");
  if (rc) return rc;
  if (!(alpha1 >= 0.0 && alpha1 < 1.0 && alpha2 >= 0.0 && alpha2 < 1.0)) {
    gs_set_error("gs_rsr_apply_rows: RSR factors must lie in [0, 1)");
    return GS_ERR_ARG;
  }
  if (k < 0 || (k > 0 && !rows)) {
    gs_set_error("gs_rsr_apply_rows: bad index list");
    return GS_ERR_ARG;
  }
  if (k == 0) return GS_OK;
  const int64_t need = (k + 31) / 32;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)gs_sm_count() * 8));
  if (rows_vec4(record, record_stride, n_elems))
    scatter_rows_kernel<false, true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        record, record_stride, n_elems, rows, k, n_rows, alpha1, alpha2);
  else
    scatter_rows_kernel<false, false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        record, record_stride, n_elems, rows, k, n_rows, alpha1, alpha2);
  return gs_check_launch("gs_rsr_apply_rows");
}

extern "C" int gs_reset_rows_rows(float* record, int64_t record_stride, int32_t n_elems,
                                  const int32_t* rows, int64_t k, int64_t n_rows, void* stream) {
  using namespace gs;
  int rc = record_args(record, record_stride, n_elems, "gs_reset_rows_rows");
  if (rc) return rc;
  if (k < 0 || (k > 0 && !rows)) {
    gs_set_error("gs_reset_rows_rows: bad index list");
    return GS_ERR_ARG;
  }
  if (k == 0) return GS_OK;
  const int64_t need = (k + 31) / 32;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)gs_sm_count() * 8));
  if (rows_vec4(record, record_stride, n_elems))
    scatter_rows_kernel<true, true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        record, record_stride, n_elems, rows, k, n_rows, 0.0, 0.0);
  else
    scatter_rows_kernel<true, false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        record, record_stride, n_elems, rows, k, n_rows, 0.0, 0.0);
  return gs_check_launch("gs_reset_rows_rows");
}

extern "C" int gs_stats_all_rows(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                                 const float* record, int64_t record_stride,
                                 const uint8_t* alive, float active_logit, double* out, void* ws,
                                 size_t ws_bytes, void* stream) {
  using namespace gs;
  GroupSet S{};
  if (!groups || n_groups < 1 || n_groups > GS_MAX_GROUPS) {
    gs_set_error("gs_stats_all_rows: bad group list");
    return GS_ERR_ARG;
  }
  S.n = n_groups;
  int P = 0;
  for (int i = 0; i < n_groups; ++i) {
    S.g[i] = group_ptrs(groups[i], false, false, 0.f);
    if (groups[i].width < 1 || !strides_ok(groups[i])) {
      gs_set_error("gs_stats_all_rows: group %d invalid", i);
      return GS_ERR_ARG;
    }
    P += (int)groups[i].width;
  }
  int rc = record_args(record, record_stride, P, "gs_stats_all_rows");
  if (rc) return rc;
  if (!out || n_rows < 0 || !ws || ws_bytes < gs_stats_workspace_bytes(n_groups)) {
    gs_set_error("gs_stats_all_rows: bad output / workspace");
    return GS_ERR_WORKSPACE;
  }
  auto* hdr = reinterpret_cast<StatsWorkspace*>(ws);
  auto* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + sizeof(StatsWorkspace));
  cudaStream_t s = (cudaStream_t)stream;
  if (record_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(record) & 15u) == 0 && P <= 127) {
    // one pass, a warp per 4 record rows per iteration
    const int64_t need = (n_rows + 4 * (kThreads / 32) - 1) / (4 * (kThreads / 32));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, stats_blocks()));
    if ((P + 1) / 2 <= 32)
      stats_rows_vec_kernel<1><<<grid, kThreads, 0, s>>>(S, P, record, record_stride, n_rows, alive,
                                                        active_logit, out, partials, &hdr->counter);
    else
      stats_rows_vec_kernel<2><<<grid, kThreads, 0, s>>>(S, P, record, record_stride, n_rows, alive,
                                                        active_logit, out, partials, &hdr->counter);
    return gs_check_launch("gs_stats_all_rows");
  }
  const int64_t need = (n_rows * 4 + kThreads - 1) / kThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, stats_blocks()));
  stats_rows_kernel<<<grid, kThreads, 0, s>>>(
      S, record, record_stride, n_rows, alive, active_logit, out, partials, &hdr->counter);
  return gs_check_launch("gs_stats_all_rows");
}

extern "C" int gs_check_grads(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                              const int32_t* rows, const int32_t* n_list_dev,
                              double lambda_opacity, double lambda_scale, uint8_t* bad_rows_out,
                              int32_t* abort_flag, void* stream) {
  using namespace gs;
  GroupSet S{};
  int rc = fill_groups(groups, n_groups, S, "gs_check_grads", true, false);
  if (rc) return rc;
  if (!abort_flag || n_rows < 0) {
    gs_set_error("gs_check_grads: abort_flag required");
    return GS_ERR_ARG;
  }
  if (bad_rows_out && (reinterpret_cast<uintptr_t>(bad_rows_out) & 3u)) {
    gs_set_error("gs_check_grads: bad_rows_out must be 4-byte aligned");
    return GS_ERR_ALIGN;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(abort_flag, 0, sizeof(int32_t), s) != cudaSuccess)
    return gs_check_launch("gs_check_grads memset");
  if (bad_rows_out && n_rows > 0 &&
      cudaMemsetAsync(bad_rows_out, 0, (size_t)n_rows, s) != cudaSuccess)
    return gs_check_launch("gs_check_grads memset");
  if (n_rows == 0) return GS_OK;
  int grid = gs_sm_count() * 8;
  if (rows && !n_list_dev) {
    gs_set_error("gs_check_grads: rows given without their device count");
    return GS_ERR_ARG;
  }
  // one gradient record?  (group g at offset sum of earlier widths, one stride)
  const float* grec = groups[0].grad;
  const int64_t grs = S.g[0].gs;
  int P = 0;
  for (int i = 0; i < n_groups && grec; ++i) {
    if (groups[i].grad != groups[0].grad + P || S.g[i].gs != grs) grec = nullptr;
    P += (int)groups[i].width;
  }
  // the 16-byte path needs 16-byte rows; the record may extend past P (pad)
  const int nq = (P + 3) / 4;
  if (grec && (grs < 4 * nq || grs % 4 != 0 || (reinterpret_cast<uintptr_t>(grec) & 15u)))
    grec = nullptr;
  int lpr = 1;
  while (lpr < nq && lpr < 32) lpr <<= 1;
  check_grads_kernel<<<grid, kThreads, 0, s>>>(S, n_rows, rows, n_list_dev, lambda_opacity,
                                               lambda_scale, bad_rows_out, abort_flag, grec, grs,
                                               P, lpr);
  return gs_check_launch("gs_check_grads");
}

extern "C" int gs_rsr_apply(const gs_group* groups, int32_t n_groups, const int32_t* rows,
                            int64_t k, int64_t n_rows, double alpha1, double alpha2,
                            void* stream) {
  using namespace gs;
  GroupSet S{};
  int rc = fill_groups(groups, n_groups, S, "gs_rsr_apply", false);
  if (rc) return rc;
  if (!(alpha1 >= 0.0 && alpha1 < 1.0 && alpha2 >= 0.0 && alpha2 < 1.0)) {
    gs_set_error("gs_rsr_apply: RSR factors must lie in [0, 1)");
    return GS_ERR_ARG;
  }
  if (k < 0 || (k > 0 && !rows)) {
    gs_set_error("gs_rsr_apply: bad index list");
    return GS_ERR_ARG;
  }
  if (k == 0) return GS_OK;
  const int64_t chunks = (k + kThreads - 1) / kThreads;
  int grid = (int)std::min<int64_t>(chunks, (int64_t)gs_sm_count() * 8);
  scatter_state_kernel<false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(S, rows, k, n_rows,
                                                                           alpha1, alpha2, nullptr);
  return gs_check_launch("gs_rsr_apply");
}

extern "C" int gs_reset_rows(const gs_group* groups, int32_t n_groups, int32_t* clock,
                             const int32_t* rows, int64_t k, int64_t n_rows, void* stream) {
  using namespace gs;
  GroupSet S{};
  int rc = fill_groups(groups, n_groups, S, "gs_reset_rows", false);
  if (rc) return rc;
  if (k < 0 || (k > 0 && !rows)) {
    gs_set_error("gs_reset_rows: bad index list");
    return GS_ERR_ARG;
  }
  if (k == 0) return GS_OK;
  const int64_t chunks = (k + kThreads - 1) / kThreads;
  int grid = (int)std::min<int64_t>(chunks, (int64_t)gs_sm_count() * 8);
  scatter_state_kernel<true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(S, rows, k, n_rows, 0.0,
                                                                          0.0, clock);
  return gs_check_launch("gs_reset_rows");
}

extern "C" size_t gs_stats_workspace_bytes(int32_t n_groups) {
  (void)n_groups;
  return sizeof(gs::StatsWorkspace) +
         (size_t)gs::stats_blocks() * gs::kStatsFields * sizeof(double);
}

extern "C" int gs_stats_all(const gs_group* groups, int32_t n_groups, int64_t n_rows,
                            const uint8_t* alive, float active_logit, double* out, void* ws,
                            size_t ws_bytes, void* stream) {
  using namespace gs;
  GroupSet S{};
  int rc = fill_groups(groups, n_groups, S, "gs_stats_all", false);
  if (rc) return rc;
  if (!out || n_rows < 0) {
    gs_set_error("gs_stats_all: bad arguments");
    return GS_ERR_ARG;
  }
  if (!ws || ws_bytes < gs_stats_workspace_bytes(n_groups)) {
    gs_set_error("gs_stats_all: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  auto* hdr = reinterpret_cast<StatsWorkspace*>(ws);
  auto* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + sizeof(StatsWorkspace));
  const int64_t need = (n_rows * 4 + kThreads - 1) / kThreads;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, stats_blocks()));
  stats_all_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(S, n_rows, alive, active_logit,
                                                                out, partials, &hdr->counter);
  return gs_check_launch("gs_stats_all");
}

extern "C" int gs_aiu_apply_rows(const gs_group* groups, int32_t n_groups, float* record,
                                 int64_t record_stride, const int32_t* inv_idx,
                                 const int32_t* jlist, const int32_t* k_dev, int64_t max_k,
                                 const float* bias_lut, int32_t lut_len, float eps,
                                 int32_t* picked_out, void* stream) {
  using namespace gs;
  GroupSet S{};
  if (!groups || n_groups < 1 || n_groups > GS_MAX_GROUPS) {
    gs_set_error("gs_aiu_apply_rows: bad group list");
    return GS_ERR_ARG;
  }
  S.n = n_groups;
  int P = 0;
  for (int i = 0; i < n_groups; ++i) {
    if (!groups[i].param || groups[i].width < 1 || !strides_ok(groups[i])) {
      gs_set_error("gs_aiu_apply_rows: group %d invalid", i);
      return GS_ERR_ARG;
    }
    // lr carries fl32(lr * eta), set by the caller
    S.g[i] = group_ptrs(groups[i], false, false, groups[i].lr);
    P += (int)groups[i].width;
  }
  int rc = record_args(record, record_stride, P, "gs_aiu_apply_rows");
  if (rc) return rc;
  if (P > 128) {
    gs_set_error("gs_aiu_apply_rows: at most 128 elements per row (%d)", P);
    return GS_ERR_ARG;
  }
  if (!inv_idx || !jlist || !k_dev || !bias_lut || lut_len < 2 || max_k < 0) {
    gs_set_error("gs_aiu_apply_rows: bad index / LUT arguments");
    return GS_ERR_ARG;
  }
  if (max_k == 0) return GS_OK;
  const int64_t need = (max_k + 7) / 8;  // a warp per row
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)gs_sm_count() * 8));
  aiu_rows_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(
      S, P, record, record_stride, inv_idx, jlist, k_dev, bias_lut, lut_len, eps, picked_out);
  return gs_check_launch("gs_aiu_apply_rows");
}

// ---------------------------------------------------------------------------
// MCMC relocation (pipeline.py:197-233): every dead row takes its target's
// attributes, the target and its respawns share the blend-preserving opacity
// tau_new (computed on the host in float64 with the reference's formula,
// 1 - (1 - o)^(1/(k+1)), since the host draws the targets anyway), and the
// respawned rows restart with zero moments and clock (reset_rows,
// optimizer.py:159-165).  A warp owns a dead row.  Dead rows are distinct and
// never targets, and the kernel never reads tau, so the writes race with no
// read: a target shared by several respawns receives the same value from each.
// ---------------------------------------------------------------------------
namespace gs {

__global__ void __launch_bounds__(kThreads)
    relocate_rows_kernel(const GroupSet S, int opacity_group, const int32_t* __restrict__ dead,
                         const int32_t* __restrict__ targets, const float* __restrict__ tau_new,
                         int64_t k, float* __restrict__ record, int64_t stride, int rec_elems) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t i = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); i < k; i += warps) {
    const int64_t d = __ldg(dead + i);
    const int64_t t = __ldg(targets + i);
    for (int gi = 0; gi < S.n; ++gi) {
      const GroupPtrs& G = S.g[gi];
      if (gi == opacity_group) {
        if (lane == 0) {
          const float tn = __ldg(tau_new + i);
          G.param[d * G.ps] = tn;
          G.param[t * G.ps] = tn;
        }
        continue;
      }
      for (int c = lane; c < G.width; c += 32) G.param[d * G.ps + c] = G.param[t * G.ps + c];
    }
    float* rec = record + d * stride;
    for (int c = lane; c < rec_elems; c += 32) rec[c] = 0.0f;  // (m, v) pairs, clock, pad
  }
}

}  // namespace gs

extern "C" int gs_relocate_rows(const gs_group* groups, int32_t n_groups, int32_t opacity_group,
                                const int32_t* dead, const int32_t* targets,
                                const float* tau_new, int64_t k, float* record,
                                int64_t record_stride, void* stream) {
  using namespace gs;
  GroupSet S{};
  if (!groups || n_groups < 1 || n_groups > GS_MAX_GROUPS || opacity_group < 0 ||
      opacity_group >= n_groups || groups[opacity_group].width != 1) {
    gs_set_error("gs_relocate_rows: bad group list / opacity group");
    return GS_ERR_ARG;
  }
  S.n = n_groups;
  int P = 0;
  for (int i = 0; i < n_groups; ++i) {
    if (!groups[i].param || groups[i].width < 1 || !strides_ok(groups[i])) {
      gs_set_error("gs_relocate_rows: group %d invalid", i);
      return GS_ERR_ARG;
    }
    S.g[i] = group_ptrs(groups[i], false, false, 0.f);
    P += (int)groups[i].width;
  }
  int rc = record_args(record, record_stride, P, "gs_relocate_rows");
  if (rc) return rc;
  if (k < 0 || (k > 0 && (!dead || !targets || !tau_new))) {
    gs_set_error("gs_relocate_rows: bad row lists");
    return GS_ERR_ARG;
  }
  if (k == 0) return GS_OK;
  const int64_t warps_needed = k;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((warps_needed + kThreads / 32 - 1) / (kThreads / 32),
                           (int64_t)gs_sm_count() * 8));
  relocate_rows_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(
      S, opacity_group, dead, targets, tau_new, k, record, record_stride, 2 * (P + 1));
  return gs_check_launch("gs_relocate_rows");
}

extern "C" int gs_densify_rows(const float* grad, int64_t grad_stride, int32_t width,
                               const int32_t* rows, const int32_t* n_list_dev, int64_t max_rows,
                               float* accum, int32_t* count, float scale,
                               const int32_t* abort_flag, void* stream) {
  using namespace gs;
  if (!grad || width < 1 || grad_stride < width || !rows || !n_list_dev || max_rows < 0 ||
      !accum || !count) {
    gs_set_error("gs_densify_rows: bad arguments");
    return GS_ERR_ARG;
  }
  if (max_rows == 0) return GS_OK;
  const int64_t need = (max_rows + kThreads - 1) / kThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)gs_sm_count() * 4));
  densify_rows_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(
      grad, grad_stride, width, rows, n_list_dev, DensifyArgs{accum, count, scale, 0}, abort_flag);
  return gs_check_launch("gs_densify_rows");
}
