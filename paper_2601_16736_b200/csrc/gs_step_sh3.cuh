// Shared by gs_step_sh3.cu (dispatch + C ABI) and gs_step_sh3_m*.cu (one
// translation unit per step mode, compiled in parallel).
#pragma once
// K2 fast path: the fused AdamW-GS step, specialised at compile time for the
// 3DGS SH-3 attribute layout (xyz 3 | f_dc 3 | f_rest 45 | opacity 1 |
// scaling 3 | rotation 4) with row-record optimizer state.  gs_step_rows
// (gs_step_rows.cu) calls gs_step_fixed_try first.
//
// Every kernel here walks chunks of 32 visible rows.  The group loop is
// unrolled over the compile-time layout, so widths, roles, record offsets and
// the penalty code paths cost no branches.  The arithmetic is
// gs_common.cuh::update_element, bit-identical to oracle step_fp32.  A row
// with a non-finite gradient, or tau / kappa outside the activation domain
// where a penalty is active, is skipped whole.
//
// Shipped kernels:
//   step_tma4_kernel (gs_step_sh3_tma.cuh)  default for device-resident
//       parameter / gradient / moment records: 2-D TMA row gathers and
//       scatters (tile::gather4 / tile::scatter4), loader / consumer / storer
//       warps, 3-stage ring, in-place update in shared memory.
//   step_ring_kernel<..., REC=1>  records the TMA kernel cannot take
//       (host-mapped gradients, compact 240-byte rows, GS_FIXED_VARIANT=21):
//       3 producer warps cp.async the chunk's moment records, theta rows and
//       gradient rows (16-byte pieces, array by array; row ids by shuffle),
//       plus the row ids and bias factors, into a 2-stage ring (full / empty
//       mbarriers).  8 consumer warps check, update and store, with one
//       named barrier per chunk (epoch-tagged row flags).
//   step_ws_kernel<...>  per-attribute theta / gradient tensors.  The same
//       ring with 4-byte element gathers in chunk element order and three
//       consumer barriers per chunk (cheaper there than per-element row-id
//       shuffles).
// Measured alternatives (phase-separated, the first cp.async rings, other
// ring shapes, 1-D bulk copies) build only with -DGS_BUILD_VARIANTS=1
// (gs_set_fixed_variant); their results are bit-identical.
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
  uint32_t ps;  // param / grad row strides (elements; == width unless record views)
  uint32_t gs;
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
  DensifyArgs D;
  const int32_t* rows;
  const int32_t* n_rows_dev;
  int64_t max_rows;
  float* record;
  int64_t stride;
  // row-interleaved parameter / gradient records (REC kernels): the group
  // pointers are prec + OFF(g) / grec + OFF(g) with row strides prs / grs
  const float* prec;
  const float* grec;
  uint32_t prs;
  uint32_t grs;
  int grec_ca;  // gradient record copies through L1 (.ca): host-mapped gradients
  int tma_ok;   // records and the state record allow 16-byte bulk copies
  int wide;     // records past 2^32 elements of row offset: 64-bit ring kernel only
  double* stats_out;
  double* partials;
  unsigned int* counter;
  // two-phase fused compaction (step_tma4_kernel MASK 3 / 4): the visible
  // ids of every CTA's mask range, the per-CTA counts and the grid barrier
  int32_t* tp_ids;
  int32_t* tp_counts;
  unsigned int* tp_bar;
  int mask_slices;  // streaming fused kernel: 0 = by size, 1 = per-CTA slices, 2 = tiles grid-stride
  unsigned int* tile_ctr;  // streaming fused kernel: the dynamic tail's claim counter (null: off)
  int dyn_eighths;         // eighths of the tiles in the dynamic tail
};

constexpr int kFixedThreads = 256;

// Rounds of group g in a chunk of R rows: ceil(R * W_g / NT) (compile-time).
template <class L, int R, int NT>
struct ChunkShape {
  __host__ __device__ static constexpr int rounds(int g) { return (R * L::W(g) + NT - 1) / NT; }
  __host__ __device__ static constexpr int first(int g) {
    int s = 0;
    for (int k = 0; k < g; ++k) s += rounds(k);
    return s;
  }
  static constexpr int total = first(L::G);
};

// Chunk elements are enumerated group by group; element k*NT + t of group g
// is (row (k*NT + t) / W_g, column (k*NT + t) % W_g) of the chunk.  The group
// loop is unrolled, so widths, roles, record offsets and the parameter
// pointers are compile-time per round, and a round's warp-uniform predicate
// (k*NT + t < R*W_g) is the only control flow.
#if GS_BUILD_VARIANTS  // measured alternatives; -DGS_BUILD_VARIANTS=1
template <class L, int MODE, bool STRICT, int R, int MINB, int NT>
__global__ void __launch_bounds__(NT, MINB) step_fixed_kernel(const FixedParams P) {
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  using S = ChunkShape<L, R, NT>;
  constexpr int NR = S::total;  // element rounds per thread per chunk
  __shared__ uint32_t s_row[R];
  __shared__ int s_bad[R];
  __shared__ float2 s_bc[R];
  __shared__ int s_any_bad;
  __shared__ double s_red[GS_STEP_STATS * (NT / 32)];

  const int t = threadIdx.x;
  float2* const rec_base = reinterpret_cast<float2*>(P.record);
  const uint32_t rec_stride2 = (uint32_t)(P.stride / 2);  // float2 per record
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
    int my_clock = 0;
    float2* my_rec = nullptr;
    if (t == 0) s_any_bad = 0;
    if (t < R) {
      const int32_t my_row = t < nvalid ? (kDense ? (int32_t)(base + t) : __ldg(P.rows + base + t)) : 0;
      my_rec = rec_base + (size_t)my_row * rec_stride2;
      s_row[t] = (uint32_t)my_row;
      s_bad[t] = t < nvalid ? 0 : 4;
      if (t < nvalid) my_clock = reinterpret_cast<const int*>(my_rec)[2 * L::P];
    }
    __syncthreads();

    // ---- phase L: every load of this thread's elements, all groups ------------
    float th[NR], gr[NR];
    float2 mv[NR];
#pragma unroll
    for (int gg = 0; gg < L::G; ++gg) {
      const int W = L::W(gg);
#pragma unroll
      for (int k = 0; k < S::rounds(gg); ++k) {
        const int q = S::first(gg) + k;
        const int i = k * NT + t;
        const int r = i / W;
        th[q] = gr[q] = 0.f;
        mv[q] = make_float2(0.f, 0.f);
        if (i < R * W && r < nvalid) {
          const int c = i - r * W;
          // 32-bit element offset: the host guarantees n_rows * W < 2^32
          const uint32_t row = s_row[r];
          const uint32_t off = row * (uint32_t)W + (uint32_t)c;
          th[q] = P.g[gg].param[off];
          gr[q] = __ldg(P.g[gg].grad + off);
          mv[q] = rec_base[(size_t)row * rec_stride2 + L::OFF(gg) + c];
        }
      }
    }
    float2 my_bc = make_float2(1.f, 1.f);
    if (t < nvalid)
      my_bc = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : my_clock + 1, 0.0, 0.0);

    // ---- validity: non-finite gradient (bit 0), activation domain (bit 1) -----
    if (!STRICT) {
#pragma unroll
      for (int gg = 0; gg < L::G; ++gg) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
        for (int k = 0; k < S::rounds(gg); ++k) {
          const int q = S::first(gg) + k;
          const int i = k * NT + t;
          const int r = i / W;
          int bad = isfinite(gr[q]) ? 0 : 1;
          if ((role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
              domain_bad(role, th[q]))
            bad |= 2;
          if (bad && i < R * W && r < nvalid) {
            atomicOr(&s_bad[r], bad);
            s_any_bad = 1;
          }
        }
      }
    }
    __syncthreads();
    const bool any_bad = s_any_bad != 0 || nvalid < R;  // block-uniform
    if (t < nvalid) {
      ++c_vis;
      const int bad = s_bad[t];
      if (bad == 0) {
        reinterpret_cast<int*>(my_rec)[2 * L::P] = my_clock + 1;
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
    for (int gg = 0; gg < L::G; ++gg) {
      const int W = L::W(gg);
      const int role = L::ROLE(gg);
      float* const par = P.g[gg].param;
      const float lr = P.g[gg].lr;
#pragma unroll
      for (int k = 0; k < S::rounds(gg); ++k) {
        const int q = S::first(gg) + k;
        const int i = k * NT + t;
        const int r = i / W;
        // common case (no bad / missing row in the chunk): no per-element check
        if (i < R * W && (!any_bad || (r < nvalid && s_bad[r] == 0))) {
          const int c = i - r * W;
          const uint32_t row = s_row[r];
          const uint32_t off = row * (uint32_t)W + (uint32_t)c;
          float tn, mn, vn, ex;
          bool clipped;
          update_element<MODE>(role, lr, th[q], gr[q], mv[q].x, mv[q].y, s_bc[r], K, tn, mn, vn,
                               ex, clipped);
          if (!kCoupled && role == GS_ROLE_OPACITY) {
            c_clo += clipped;
            s_exo += (double)ex;
          } else if (!kCoupled && role == GS_ROLE_SCALE) {
            c_cls += clipped;
            s_exs += (double)ex;
          }
          if (role == GS_ROLE_OPACITY) {
            c_apre += th[q] > P.active_logit;
            c_apost += tn > P.active_logit;
          }
          par[off] = tn;
          rec_base[(size_t)row * rec_stride2 + L::OFF(gg) + c] = make_float2(mn, vn);
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
  if (last_block_arrive(P.counter))
    final_reduce<GS_STEP_STATS>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out, is_max, s_red);
}
#endif  // GS_BUILD_VARIANTS (phase-separated kernel)

// ---------------------------------------------------------------------------
// Pipelined variant: a persistent CTA walks its chunks through an S-stage
// shared-memory ring filled with cp.async (LDGSTS).  While chunk c is
// validated, updated and written back, the gathers of chunks c+1 .. c+S-1
// are in flight, so every SM keeps ~(S-1) chunks of loads outstanding
// without holding them in registers.
//   * records: whole 8*(P+1)-byte rows, 16-byte cp.async.cg pieces;
//   * theta / grad: 4-byte cp.async.ca gathers in chunk element order;
//   * write-back: theta with scattered 4-byte stores, the updated record
//     (m, v pairs + clock) from shared memory with 16-byte stores.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
// 16-byte piece with an L2 prefetch-size hint (the L2 fills the whole 256-B
// (or 128-B) aligned span around the piece from DRAM in one request)
template <int HINT>
__device__ __forceinline__ void cp_async16_h(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (HINT & 1)
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else if (HINT & 4)
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_ca(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#if GS_BUILD_VARIANTS
template <class L, int R>
struct PipeStage {
  static constexpr int kSlots = L::P + 1;                  // record slots per row
  static constexpr int kRec = R * kSlots * 8;              // bytes of records
  static constexpr int kTh = R * L::P * 4;                 // theta bytes
  static constexpr int kBytes = kRec + 2 * kTh;
};

template <class L, int MODE, bool STRICT, int R, int S, int MINB>
__global__ void __launch_bounds__(kFixedThreads, MINB) step_pipe_kernel(const FixedParams P) {
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NT = kFixedThreads;
  constexpr int SLOTS = L::P + 1;
  using SH = ChunkShape<L, R, NT>;
  using ST = PipeStage<L, R>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_bad[R];
  __shared__ float2 s_bc[R];
  __shared__ uint32_t s_rows[S + 1][R];  // row ids, one slot more than stages (no reuse race)
  __shared__ double s_red[GS_STEP_STATS * (NT / 32)];

  auto rec_of = [&](int st) { return reinterpret_cast<float2*>(smem + st * ST::kBytes); };
  auto th_of = [&](int st) { return reinterpret_cast<float*>(smem + st * ST::kBytes + ST::kRec); };
  auto g_of = [&](int st) {
    return reinterpret_cast<float*>(smem + st * ST::kBytes + ST::kRec + ST::kTh);
  };
  auto row_of = [&](int64_t k) { return s_rows[k % (S + 1)]; };

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
  // this CTA's k-th chunk
  auto chunk_id = [&](int64_t k) { return (int64_t)blockIdx.x + k * gridDim.x; };
  auto chunk_rows = [&](int64_t ch) -> int {
    const int64_t rem = n_rows - ch * R;
    return rem <= 0 ? 0 : (rem < R ? (int)rem : R);
  };
  auto load_row_id = [&](int64_t ch) -> uint32_t {
    if (t >= R || t >= chunk_rows(ch)) return 0u;
    const int64_t i = ch * R + t;
    return kDense ? (uint32_t)i : (uint32_t)__ldg(P.rows + i);
  };
  // issue the gathers of this CTA's k-th chunk into stage st (row ids in smem)
  auto issue = [&](int64_t kc, int st) {
    const int64_t ch = chunk_id(kc);
    const int nv = chunk_rows(ch);
    const uint32_t* rows = row_of(kc);
    float2* srec = rec_of(st);
    // records: 16-byte pieces, SLOTS*8/16 per row
    constexpr int kPieces = SLOTS * 8 / 16;
    for (int p = t; p < nv * kPieces; p += NT) {
      const int r = p / kPieces;
      const int k = p - r * kPieces;
      const float* src = P.record + (int64_t)rows[r] * P.stride + 4 * k;
      cp_async16(reinterpret_cast<float*>(srec + r * SLOTS) + 4 * k, src);
    }
    float* sth = th_of(st);
    float* sg = g_of(st);
#pragma unroll
    for (int gg = 0; gg < L::G; ++gg) {
      const int W = L::W(gg);
#pragma unroll
      for (int k = 0; k < SH::rounds(gg); ++k) {
        const int i = k * NT + t;
        const int r = i / W;
        if (i < R * W && r < nv) {
          const int c = i - r * W;
          const uint32_t off = rows[r] * (uint32_t)W + (uint32_t)c;
          const int e = R * L::OFF(gg) + i;
          cp_async4(sth + e, P.g[gg].param + off);
          cp_async4(sg + e, P.g[gg].grad + off);
        }
      }
    }
  };

  // ---- prologue: row ids + gathers of the first S-1 chunks ---------------------
  uint32_t pf_row = 0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (t < R) row_of(s)[t] = load_row_id(chunk_id(s));
  }
  pf_row = load_row_id(chunk_id(S - 1));
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (chunk_id(s) < n_chunks) issue(s, s);
    cp_async_commit();
  }

  for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
    const int st = (int)(k % S);
    const int st_next = (int)((k + S - 1) % S);
    const int64_t ch = chunk_id(k);
    const int nvalid = chunk_rows(ch);
    // A. row ids of chunk k+S-1 (its id slot was last read two iterations
    //    ago); prefetch the ids of chunk k+S
    if (t < R) row_of(k + S - 1)[t] = pf_row;
    pf_row = load_row_id(chunk_id(k + S));
    __syncthreads();  // B: stage st_next free (chunk k-1 written back), ids visible
    if (t < R) s_bad[t] = t < nvalid ? 0 : 4;
    // C. gathers of chunk k+S-1
    if (chunk_id(k + S - 1) < n_chunks) issue(k + S - 1, st_next);
    cp_async_commit();
    // D. chunk k landed
    cp_async_wait<S - 1>();
    __syncthreads();

    float2* srec = rec_of(st);
    float* sth = th_of(st);
    float* sg = g_of(st);
    const uint32_t* srow = row_of(k);
    // E. validity
    if (!STRICT) {
#pragma unroll
      for (int gg = 0; gg < L::G; ++gg) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
        for (int kk = 0; kk < SH::rounds(gg); ++kk) {
          const int i = kk * NT + t;
          const int r = i / W;
          if (i < R * W && r < nvalid) {
            const int e = R * L::OFF(gg) + i;
            int bad = isfinite(sg[e]) ? 0 : 1;
            if ((role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
                domain_bad(role, sth[e]))
              bad |= 2;
            if (bad) atomicOr(&s_bad[r], bad);
          }
        }
      }
      __syncthreads();
    }
    // F. clocks and bias factors (thread r owns row r)
    if (t < nvalid) {
      ++c_vis;
      const int bad = s_bad[t];
      if (bad == 0) {
        int* clk = reinterpret_cast<int*>(srec + t * SLOTS + L::P);
        const int tn = *clk + 1;
        *clk = tn;
        s_bc[t] = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : tn, 0.0, 0.0);
        ++c_step;
      } else if (bad & 1) {
        ++c_badg;
      } else {
        ++c_badd;
      }
    }
    __syncthreads();
    // G. update: theta to global, (m, v) into the staged record
#pragma unroll
    for (int gg = 0; gg < L::G; ++gg) {
      const int W = L::W(gg);
      const int role = L::ROLE(gg);
      float* const par = P.g[gg].param;
      const float lr = P.g[gg].lr;
#pragma unroll
      for (int kk = 0; kk < SH::rounds(gg); ++kk) {
        const int i = kk * NT + t;
        const int r = i / W;
        if (i < R * W && r < nvalid && s_bad[r] == 0) {
          const int c = i - r * W;
          const int e = R * L::OFF(gg) + i;
          float2* slot = srec + r * SLOTS + L::OFF(gg) + c;
          const float2 mv = *slot;
          const float th = sth[e];
          float tn, mn, vn, ex;
          bool clipped;
          update_element<MODE>(role, lr, th, sg[e], mv.x, mv.y, s_bc[r], K, tn, mn, vn, ex,
                               clipped);
          if (!kCoupled && role == GS_ROLE_OPACITY) {
            c_clo += clipped;
            s_exo += (double)ex;
          } else if (!kCoupled && role == GS_ROLE_SCALE) {
            c_cls += clipped;
            s_exs += (double)ex;
          }
          if (role == GS_ROLE_OPACITY) {
            c_apre += th > P.active_logit;
            c_apost += tn > P.active_logit;
          }
          par[srow[r] * (uint32_t)W + (uint32_t)c] = tn;
          *slot = make_float2(mn, vn);
        }
      }
    }
    __syncthreads();
    // H. record write-back, 16-byte pieces, valid rows only
    {
      constexpr int kPieces = SLOTS * 8 / 16;
      for (int p = t; p < nvalid * kPieces; p += NT) {
        const int r = p / kPieces;
        if (s_bad[r] != 0) continue;
        const int kk = p - r * kPieces;
        const float4 v = reinterpret_cast<const float4*>(srec + r * SLOTS)[kk];
        reinterpret_cast<float4*>(P.record + (int64_t)srow[r] * P.stride)[kk] = v;
      }
    }
  }
  cp_async_wait<0>();

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

template <class L, int MODE, bool STRICT, int R, int S, int MINB>
void launch_pipe(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  constexpr int bytes = S * PipeStage<L, R>::kBytes;
  smem_opt_in<step_pipe_kernel<L, MODE, STRICT, R, S, MINB>>(bytes);
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_pipe_kernel<L, MODE, STRICT, R, S, MINB><<<grid, kFixedThreads, bytes, s>>>(P);
}

// ---------------------------------------------------------------------------
// pipe2: the cp.async ring with three barriers per chunk.  Row ids ride one
// slot ahead of the data ring; the bad-row flags are double-buffered so they
// can be re-armed without an extra barrier; the updated (m, v) pairs and the
// clock go straight to global memory (the staged record is read-only).
// ---------------------------------------------------------------------------
template <class L, int MODE, bool STRICT, int R, int S, int MINB>
__global__ void __launch_bounds__(kFixedThreads, MINB) step_pipe2_kernel(const FixedParams P) {
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NT = kFixedThreads;
  constexpr int SLOTS = L::P + 1;
  using SH = ChunkShape<L, R, NT>;
  using ST = PipeStage<L, R>;
  static_assert(NT % 32 == 0 && (R * 1) % 32 == 0, "warp-uniform group boundaries");
  // Each group's elements start at thread (R * OFF_g) mod NT instead of 0, so
  // the small groups land on different warps and every warp gets the same
  // number of 32-element pieces per chunk (balanced barriers).
  auto rot_of = [](int gg) { return (R * L::OFF(gg)) & (NT - 1); };
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_bad[2][R];
  __shared__ float2 s_bc[2][R];
  __shared__ int s_any[2];
  __shared__ uint32_t s_rows[S + 1][R];
  __shared__ double s_red[GS_STEP_STATS * (NT / 32)];

  const int t = threadIdx.x;
  float2* const rec_base = reinterpret_cast<float2*>(P.record);
  const uint32_t rec_stride2 = (uint32_t)(P.stride / 2);
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
  auto chunk_id = [&](int64_t k) { return (int64_t)blockIdx.x + k * gridDim.x; };
  auto chunk_rows = [&](int64_t k) -> int {
    const int64_t rem = n_rows - chunk_id(k) * R;
    return rem <= 0 ? 0 : (rem < R ? (int)rem : R);
  };
  auto load_row_id = [&](int64_t k) -> uint32_t {
    if (t >= R || t >= chunk_rows(k)) return 0u;
    const int64_t i = chunk_id(k) * R + t;
    return kDense ? (uint32_t)i : (uint32_t)__ldg(P.rows + i);
  };
  auto stage = [&](int st) { return smem + st * ST::kBytes; };
  auto issue = [&](int64_t kc, int st) {
    const int nv = chunk_rows(kc);
    const uint32_t* rows = s_rows[kc % (S + 1)];
    float2* srec = reinterpret_cast<float2*>(stage(st));
    constexpr int kPieces = SLOTS * 8 / 16;
    for (int p = t; p < nv * kPieces; p += NT) {
      const int r = p / kPieces;
      const int k = p - r * kPieces;
      cp_async16(reinterpret_cast<float*>(srec + r * SLOTS) + 4 * k,
                 P.record + (size_t)rows[r] * P.stride + 4 * k);
    }
    float* sth = reinterpret_cast<float*>(stage(st) + ST::kRec);
    float* sg = sth + R * L::P;
#pragma unroll
    for (int gg = 0; gg < L::G; ++gg) {
      const int W = L::W(gg);
#pragma unroll
      for (int k = 0; k < SH::rounds(gg); ++k) {
        const int i = k * NT + ((t - rot_of(gg)) & (NT - 1));
        const int r = i / W;
        if (i < R * W && r < nv) {
          const uint32_t off = rows[r] * (uint32_t)W + (uint32_t)(i - r * W);
          const int e = R * L::OFF(gg) + i;
          cp_async4(sth + e, P.g[gg].param + off);
          cp_async4(sg + e, P.g[gg].grad + off);
        }
      }
    }
  };

  // prologue: ids of chunks 0..S-1 (the last one prefetched in a register),
  // gathers of chunks 0..S-2, bad flags of chunk 0
  uint32_t pf_row = 0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s)
    if (t < R) s_rows[s % (S + 1)][t] = load_row_id(s);
  pf_row = load_row_id(S - 1);
  if (t < R) s_bad[0][t] = t < chunk_rows(0) ? 0 : 4;
  if (t == 0) s_any[0] = chunk_rows(0) < R;
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (chunk_id(s) < n_chunks) issue(s, s);
    cp_async_commit();
  }

  for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
    const int st = (int)(k % S);
    const int b = (int)(k & 1);
    const int nvalid = chunk_rows(k);
    // A. ids of chunk k+S-1 (slot last read in iteration k-2); prefetch k+S
    if (t < R) s_rows[(k + S - 1) % (S + 1)][t] = pf_row;
    pf_row = load_row_id(k + S);
    // #1: chunk k landed; iteration k-1 finished (stage (k-1)%S free)
    cp_async_wait<S - 2>();
    __syncthreads();
    if (chunk_id(k + S - 1) < n_chunks) issue(k + S - 1, (int)((k + S - 1) % S));
    cp_async_commit();

    const float2* srec = reinterpret_cast<const float2*>(stage(st));
    const float* sth = reinterpret_cast<const float*>(stage(st) + ST::kRec);
    const float* sg = sth + R * L::P;
    const uint32_t* srow = s_rows[k % (S + 1)];
    // E. validity; thread r prepares row r's clock and bias factors
    if (!STRICT) {
#pragma unroll
      for (int gg = 0; gg < L::G; ++gg) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
        for (int kk = 0; kk < SH::rounds(gg); ++kk) {
          const int i = kk * NT + ((t - rot_of(gg)) & (NT - 1));
          const int r = i / W;
          if (i < R * W && r < nvalid) {
            const int e = R * L::OFF(gg) + i;
            int bad = isfinite(sg[e]) ? 0 : 1;
            if ((role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
                domain_bad(role, sth[e]))
              bad |= 2;
            if (bad) {
              atomicOr(&s_bad[b][r], bad);
              s_any[b] = 1;
            }
          }
        }
      }
    }
    int tn = 0;
    float2 bc = make_float2(1.f, 1.f);
    if (t < nvalid) {
      tn = reinterpret_cast<const int*>(srec + t * SLOTS + L::P)[0] + 1;
      bc = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : tn, 0.0, 0.0);
    }
    __syncthreads();  // #2: bad flags final
    const bool any_bad = s_any[b] != 0;
    if (t < nvalid) {
      ++c_vis;
      const int bad = s_bad[b][t];
      if (bad == 0) {
        reinterpret_cast<int*>(rec_base + (size_t)srow[t] * rec_stride2 + L::P)[0] = tn;
        s_bc[b][t] = bc;
        ++c_step;
      } else if (bad & 1) {
        ++c_badg;
      } else {
        ++c_badd;
      }
    }
    // re-arm the other flag buffer for chunk k+1 (last read in iteration k-1)
    if (t < R) s_bad[b ^ 1][t] = t < chunk_rows(k + 1) ? 0 : 4;
    if (t == 0) s_any[b ^ 1] = chunk_rows(k + 1) < R;
    __syncthreads();  // #3: bias factors visible
    // G. update: theta and (m, v) straight to global.  The common case (a
    //    full chunk without bad rows) runs without any per-element predicate
    //    on the full rounds; otherwise every element checks its row.
    auto update = [&](int gg, int i, int r) {
      const int W = L::W(gg);
      const int role = L::ROLE(gg);
      const int c = i - r * W;
      const int e = R * L::OFF(gg) + i;
      const uint32_t row = srow[r];
      const float2 mv = srec[r * SLOTS + L::OFF(gg) + c];
      const float th = sth[e];
      float tnv, mn, vn, ex;
      bool clipped;
      update_element<MODE>(role, P.g[gg].lr, th, sg[e], mv.x, mv.y, s_bc[b][r], K, tnv, mn, vn,
                           ex, clipped);
      if (!kCoupled && role == GS_ROLE_OPACITY) {
        c_clo += clipped;
        s_exo += (double)ex;
      } else if (!kCoupled && role == GS_ROLE_SCALE) {
        c_cls += clipped;
        s_exs += (double)ex;
      }
      if (role == GS_ROLE_OPACITY) {
        c_apre += th > P.active_logit;
        c_apost += tnv > P.active_logit;
      }
      P.g[gg].param[row * (uint32_t)W + (uint32_t)c] = tnv;
      rec_base[(size_t)row * rec_stride2 + L::OFF(gg) + c] = make_float2(mn, vn);
    };
    if (!any_bad) {
#pragma unroll
      for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
        for (int kk = 0; kk < SH::rounds(gg); ++kk) {
          const int i = kk * NT + ((t - rot_of(gg)) & (NT - 1));
          const bool full = (kk + 1) * NT <= R * L::W(gg);  // compile-time
          if (full || i < R * L::W(gg)) update(gg, i, i / L::W(gg));
        }
      }
    } else {
#pragma unroll
      for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
        for (int kk = 0; kk < SH::rounds(gg); ++kk) {
          const int i = kk * NT + ((t - rot_of(gg)) & (NT - 1));
          const int r = i / L::W(gg);
          if (i < R * L::W(gg) && r < nvalid && s_bad[b][r] == 0) update(gg, i, r);
        }
      }
    }
  }
  cp_async_wait<0>();

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

template <class L, int MODE, bool STRICT, int R, int S, int MINB>
void launch_pipe2(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  constexpr int bytes = S * PipeStage<L, R>::kBytes;
  smem_opt_in<step_pipe2_kernel<L, MODE, STRICT, R, S, MINB>>(bytes);
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_pipe2_kernel<L, MODE, STRICT, R, S, MINB><<<grid, kFixedThreads, bytes, s>>>(P);
}

#endif  // GS_BUILD_VARIANTS (pipe / pipe2)
// ---------------------------------------------------------------------------
// Warp-specialised variant: kProd producer warps fill an S-stage ring with
// cp.async gathers (row ids, 16-byte record pieces, 4-byte theta / grad
// elements) and signal a per-stage "full" mbarrier through
// cp.async.mbarrier.arrive.noinc; kCons consumer warps wait on it, validate,
// update and store, synchronising only among themselves (named barrier 1),
// and release the stage through an "empty" mbarrier.  Producers never wait
// on a block barrier, so gathers for the next chunks stay in flight while
// the consumers compute.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(s),
      "l"(gmem), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem), "r"(s),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <class L, int R>
struct WsStage {
  static constexpr int kSlots = L::P + 1;
  static constexpr int kPL = (L::P + 3) & ~3;  // staged theta / grad row (16-byte pieces)
  static constexpr int kRec = R * kSlots * 8;
  static constexpr int kTh = R * kPL * 4;
  static constexpr int kBytes = kRec + 2 * kTh + R * 4;  // + row ids
};

template <class L, int MODE, bool STRICT, int R, int S, int NPW, int NCW, int MINB, bool REC,
          bool BULKST = false>
__global__ void __launch_bounds__((NPW + NCW) * 32, MINB) step_ws_kernel(const FixedParams P) {
  // BULKST (records only): results are written into the stage in place and
  // every good row leaves with two bulk stores (parameter row, moment record)
  static_assert(REC || !BULKST, "bulk stores need row-contiguous records");
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NC = NCW * 32;  // consumer threads
  constexpr int NP = NPW * 32;  // producer threads
  constexpr int SLOTS = L::P + 1;
  using SH = ChunkShape<L, R, NC>;
  using ST = WsStage<L, R>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];
  __shared__ int s_bad[S][R];
  __shared__ int s_any[S];
  __shared__ float2 s_bc[S][R];
  __shared__ uint32_t s_crow[S][R];  // consumers' copy of the row ids
  __shared__ double s_red[GS_STEP_STATS * ((NPW + NCW))];

  const int tid = threadIdx.x;
  const bool producer = tid >= NC;
  int64_t n_rows = kDense ? P.max_rows : (int64_t)(*P.n_rows_dev);
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  const int64_t n_chunks = (n_rows + R - 1) / R;
  auto chunk_id = [&](int64_t k) { return (int64_t)blockIdx.x + k * gridDim.x; };
  auto chunk_rows = [&](int64_t k) -> int {
    const int64_t rem = n_rows - chunk_id(k) * R;
    return rem <= 0 ? 0 : (rem < R ? (int)rem : R);
  };
  auto stage = [&](int st) { return smem + st * ST::kBytes; };
  constexpr int PL = ST::kPL;
  // staged theta / grad of chunk element i (row r) of group gg: group-major
  // for per-attribute gathers, row-major (one 16-byte-piece copy per record
  // row) for record views
  auto sidx = [](int gg, int i, int r) -> int {
    return REC ? r * PL + L::OFF(gg) + (i - r * L::W(gg)) : R * L::OFF(gg) + i;
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], NP);
      mbar_init(&empty_bar[s], NC);
    }
  }
  if (tid < R * S) s_bad[tid / R][tid % R] = 0;
  if (tid < S) s_any[tid] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  if (producer) {
    // ------------------------------------------------------------------ producer
    const int pt = tid - NC;
    // row id of row pt of chunk k (producer lanes pt < R), prefetched one
    // chunk ahead so the gathers never wait on the index list
    auto fetch_id = [&](int64_t k) -> uint32_t {
      if (pt >= R || pt >= chunk_rows(k)) return 0u;
      const int64_t i = chunk_id(k) * R + pt;
      return kDense ? (uint32_t)i : (uint32_t)__ldg(P.rows + i);
    };
    uint32_t next_id = fetch_id(0);
    for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
      const int st = (int)(k % S);
      const uint32_t my_id = next_id;
      next_id = fetch_id(k + 1);
      if (k >= S) mbar_wait(&empty_bar[st], (unsigned)(((k / S) - 1) & 1));
      const int nv = chunk_rows(k);
      unsigned char* sb = stage(st);
      uint32_t* srows = reinterpret_cast<uint32_t*>(sb + ST::kRec + 2 * ST::kTh);
      if (pt < R) srows[pt] = my_id;
      named_sync(2, NP);  // producer-only: ids visible to the other producer lanes
      float2* srec = reinterpret_cast<float2*>(sb);
      constexpr int kPieces = SLOTS * 8 / 16;
      for (int p = pt; p < nv * kPieces; p += NP) {
        const int r = p / kPieces;
        const int kk = p - r * kPieces;
        cp_async16(reinterpret_cast<float*>(srec + r * SLOTS) + 4 * kk,
                   P.record + (size_t)srows[r] * P.stride + 4 * kk);
      }
      float* sth = reinterpret_cast<float*>(sb + ST::kRec);
      float* sg = sth + R * PL;
      if (REC) {
        constexpr int kRowPieces = PL / 4;
        for (int p = pt; p < nv * kRowPieces; p += NP) {
          const int r = p / kRowPieces;
          const int q = p - r * kRowPieces;
          cp_async16(sth + r * PL + 4 * q, P.prec + srows[r] * P.prs + 4 * q);
          if (P.grec_ca)
            cp_async16_ca(sg + r * PL + 4 * q, P.grec + srows[r] * P.grs + 4 * q);
          else
            cp_async16(sg + r * PL + 4 * q, P.grec + srows[r] * P.grs + 4 * q);
        }
      } else {
        using PS = ChunkShape<L, R, NP>;
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          const int W = L::W(gg);
#pragma unroll
          for (int kk = 0; kk < PS::rounds(gg); ++kk) {
            const int i = kk * NP + ((pt + NP - (R * L::OFF(gg)) % NP) % NP);
            const int r = i / W;
            if (i < R * W && r < nv) {
              const uint32_t c = (uint32_t)(i - r * W);
              const int e = R * L::OFF(gg) + i;
              cp_async4(sth + e, P.g[gg].param + srows[r] * P.g[gg].ps + c);
              cp_async4(sg + e, P.g[gg].grad + srows[r] * P.g[gg].gs + c);
            }
          }
        }
      }
      mbar_arrive_cp_async(&full_bar[st]);
    }
  } else {
    // ------------------------------------------------------------------ consumers
    const int t = tid;
    StepConsts Kc = P.K;
    if (kCoupled) {
      const float nv = P.nv_dev ? (float)(*P.nv_dev) : (float)P.nv_host;
      Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
      if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
    }
    const StepConsts& K = kCoupled ? Kc : P.K;
    float2* const rec_base = reinterpret_cast<float2*>(P.record);
    const uint32_t rec_stride2 = (uint32_t)(P.stride / 2);
    for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
      const int st = (int)(k % S);
      const int nvalid = chunk_rows(k);
      // row ids straight from the index list (visible after the first named
      // barrier below); the producers keep their own copy in the stage
      if (t < R)
        s_crow[st][t] = t < nvalid ? (kDense ? (uint32_t)(chunk_id(k) * R + t)
                                             : (uint32_t)__ldg(P.rows + chunk_id(k) * R + t))
                                   : 0u;
      mbar_wait(&full_bar[st], (unsigned)((k / S) & 1));
      unsigned char* sbw = stage(st);
      const unsigned char* sb = sbw;
      const float2* srec = reinterpret_cast<const float2*>(sb);
      const float* sth = reinterpret_cast<const float*>(sb + ST::kRec);
      const float* sg = sth + R * PL;
      float2* const srec_w = reinterpret_cast<float2*>(sbw);
      float* const sth_w = reinterpret_cast<float*>(sbw + ST::kRec);
      const uint32_t* srow = s_crow[st];
      if (!STRICT) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          const int W = L::W(gg);
          const int role = L::ROLE(gg);
          const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / W;
            if (i < R * W && r < nvalid) {
              const int e = sidx(gg, i, r);
              int bad = isfinite(sg[e]) ? 0 : 1;
              if ((role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
                  domain_bad(role, sth[e]))
                bad |= 2;
              if (bad) {
                atomicOr(&s_bad[st][r], bad);
                s_any[st] = 1;
              }
            }
          }
        }
      }
      int tn = 0;
      float2 bc = make_float2(1.f, 1.f);
      if (t < nvalid) {
        tn = reinterpret_cast<const int*>(srec + t * SLOTS + L::P)[0] + 1;
        bc = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : tn, 0.0, 0.0);
      }
      named_sync(1, NC);  // bad flags final
      const bool any_bad = s_any[st] != 0 || nvalid < R;
      if (t < nvalid) {
        ++c_vis;
        const int bad = s_bad[st][t];
        if (bad == 0) {
          if (!BULKST)
            reinterpret_cast<int*>(rec_base + (size_t)s_crow[st][t] * rec_stride2 + L::P)[0] = tn;
          s_bc[st][t] = bc;
          if (P.D.group >= 0) {
#pragma unroll
            for (int gg = 0; gg < L::G; ++gg)
              if (gg == P.D.group)
                densify_row(P.D, s_crow[st][t], sg + sidx(gg, t * L::W(gg), t), L::W(gg), 1);
          }
          ++c_step;
        } else if (bad & 1) {
          ++c_badg;
        } else {
          ++c_badd;
        }
      }
      named_sync(1, NC);  // bias factors visible
      if (BULKST && t < nvalid && s_bad[st][t] == 0)
        reinterpret_cast<int*>(srec_w + t * SLOTS + L::P)[0] = tn;
      auto update = [&](int gg, int i, int r) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const int c = i - r * W;
        const int e = sidx(gg, i, r);
        const uint32_t row = srow[r];
        const float2 mv = srec[r * SLOTS + L::OFF(gg) + c];
        const float th = sth[e];
        float tnv, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, P.g[gg].lr, th, sg[e], mv.x, mv.y, s_bc[st][r], K, tnv, mn,
                             vn, ex, clipped);
        if (!kCoupled && role == GS_ROLE_OPACITY) {
          c_clo += clipped;
          s_exo += (double)ex;
        } else if (!kCoupled && role == GS_ROLE_SCALE) {
          c_cls += clipped;
          s_exs += (double)ex;
        }
        if (role == GS_ROLE_OPACITY) {
          c_apre += th > P.active_logit;
          c_apost += tnv > P.active_logit;
        }
        if (BULKST) {
          sth_w[e] = tnv;
          srec_w[r * SLOTS + L::OFF(gg) + c] = make_float2(mn, vn);
        } else {
          P.g[gg].param[row * P.g[gg].ps + (uint32_t)c] = tnv;
          rec_base[(size_t)row * rec_stride2 + L::OFF(gg) + c] = make_float2(mn, vn);
        }
      };
      if (!any_bad) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const bool full = (kk + 1) * NC <= R * L::W(gg);  // compile-time
            if (full || i < R * L::W(gg)) update(gg, i, i / L::W(gg));
          }
        }
      } else {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / L::W(gg);
            if (i < R * L::W(gg) && r < nvalid && s_bad[st][r] == 0) update(gg, i, r);
          }
        }
      }
      if (BULKST) {
        fence_proxy_async_smem();  // generic-proxy smem writes -> bulk-store reads
        named_sync(1, NC);         // the chunk's rows are final in shared memory
        if (t < R) {
          // stage released one chunk later, once the stores have read it
          if (t < nvalid && s_bad[st][t] == 0) {
            const uint32_t row = srow[t];
            bulk_s2g(P.g[0].param + (size_t)row * P.prs, sth + t * PL, (uint32_t)(PL * 4));
            bulk_s2g(P.record + (size_t)row * P.stride, srec + t * SLOTS, (uint32_t)(SLOTS * 8));
          }
          bulk_commit();
          s_bad[st][t] = 0;
          if (t == 0) s_any[st] = 0;
          bulk_wait_read1();
          if (k > 0) mbar_arrive(&empty_bar[(int)((k - 1) % S)]);
        } else {
          mbar_arrive(&empty_bar[st]);
        }
      } else {
        named_sync(1, NC);  // all reads of this stage's flags / data done
        if (t < R) s_bad[st][t] = 0;
        if (t == 0) s_any[st] = 0;
        mbar_arrive(&empty_bar[st]);
      }
    }
    if (BULKST) bulk_wait0();
  }
  cp_async_wait<0>();

  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce_n<GS_STEP_STATS, (NPW + NCW)>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f)
      P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter))
    final_reduce_n<GS_STEP_STATS, (NPW + NCW)>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out,
                                               is_max, s_red);
}

template <class L, int MODE, bool STRICT, int R, int S, int NPW, int NCW, int MINB,
          bool REC = false, bool BULKST = false>
void launch_ws(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  constexpr int bytes = S * WsStage<L, R>::kBytes;
  smem_opt_in<step_ws_kernel<L, MODE, STRICT, R, S, NPW, NCW, MINB, REC, BULKST>>(bytes);
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_ws_kernel<L, MODE, STRICT, R, S, NPW, NCW, MINB, REC, BULKST>
      <<<grid, (NPW + NCW) * 32, bytes, s>>>(P);
}

// ---------------------------------------------------------------------------
// Record kernel (the default for parameter/gradient records): the gather
// ring of step_ws_kernel with the synchronisation cut to one named barrier
// per chunk.
//   * producers: each warp owns whole rows (r = warp, warp + NPW, ...); every
//     lane holds the chunk's row id of its own index and the owner warp
//     broadcasts it with a shuffle — no shared-memory row-id hand-off and no
//     producer barrier.  A row is 60 16-byte pieces (30 moment record, 15
//     theta, 15 gradient): two per lane.
//   * consumers: the clock and bias factors of row t are fetched before the
//     check pass, so the LUT latency hides behind it; bad-row flags carry the
//     stage's use count (epoch) instead of being reset, so after the single
//     barrier nothing else needs a block-wide ordering point.
// ---------------------------------------------------------------------------
template <class L, int MODE, bool STRICT, int R, int S, int NPW, int NCW, int MINB, bool FLAT,
          bool REC, int HINT>
__global__ void __launch_bounds__((NPW + NCW) * 32, MINB) step_ring_kernel(const FixedParams P) {
  static_assert(REC || FLAT, "per-attribute gathers use the flattened producer");
  static_assert(R == 32, "one lane per row id");
  static_assert(S >= 2, "stage reuse relies on the next chunk's barrier");
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NC = NCW * 32;
  constexpr int NP = NPW * 32;
  constexpr int SLOTS = L::P + 1;
  using SH = ChunkShape<L, R, NC>;
  using ST = WsStage<L, R>;
  constexpr int PL = ST::kPL;
  constexpr int kRecPieces = SLOTS * 8 / 16;
  constexpr int kRowPieces = PL / 4;
  constexpr int kPiecesPerRow = kRecPieces + 2 * kRowPieces;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];
  __shared__ int s_badg[S][R];  // == epoch: non-finite gradient in this use of the stage
  __shared__ int s_badd[S][R];  // == epoch: activation-domain violation
  __shared__ int s_any[S];
  __shared__ float2 s_bc[S][R];
  __shared__ uint32_t s_crow[S][R];
  __shared__ double s_red[GS_STEP_STATS * (NPW + NCW)];

  const int tid = threadIdx.x;
  const bool producer = tid >= NC;
  // 32-bit chunk bookkeeping: row ids are int32 and the fixed-layout
  // dispatch keeps max_rows * row stride below 2^32 (rows_kind)
  int n_rows = kDense ? (int)P.max_rows : *P.n_rows_dev;
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  const int n_chunks = (n_rows + R - 1) / R;
  const int G = (int)gridDim.x;  // chunks are taken grid-stride: c = blockIdx.x + k * G
  auto chunk_rows = [&](int c) -> int {
    const int rem = n_rows - c * R;
    return rem <= 0 ? 0 : (rem < R ? rem : R);
  };
  auto stage = [&](int st) { return smem + st * ST::kBytes; };
  // row offsets into the parameter / gradient arrays: 32-bit unless the
  // cloud is past rows * stride >= 2^32 (HINT & 32, chosen by the dispatch)
  auto roff = [](uint32_t row, uint32_t stride) {
    if constexpr ((HINT & 32) != 0)
      return (size_t)row * stride;
    else
      return row * stride;
  };
  // staged theta / grad: row-major for records, group-major for per-attribute gathers
  auto sidx = [](int gg, int i, int r) -> int {
    return REC ? r * PL + L::OFF(gg) + (i - r * L::W(gg)) : R * L::OFF(gg) + i;
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], NP);
      mbar_init(&empty_bar[s], NC);
    }
  }
  if (tid < R * S) {
    s_badg[tid / R][tid % R] = 0;
    s_badd[tid / R][tid % R] = 0;
  }
  if (tid < S) s_any[tid] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  if (producer) {
    // ------------------------------------------------------------------ producer
    const int pt = tid - NC;
    const int lane = pt & 31;
    const int warp = pt >> 5;
    auto fetch_id = [&](int c) -> uint32_t {
      if (lane >= chunk_rows(c)) return 0u;
      const int i = c * R + lane;
      return kDense ? (uint32_t)i : (uint32_t)__ldg(P.rows + i);
    };
    uint32_t next_id = fetch_id((int)blockIdx.x);
    int st = 0;
    unsigned ph = 0;  // parity of this use of stage st
    for (int c = (int)blockIdx.x, k = 0; c < n_chunks; c += G, ++k) {
      const uint32_t my_id = next_id;
      next_id = fetch_id(c + G);
      if (k >= S) mbar_wait(&empty_bar[st], ph ^ 1u);
      const int nv = chunk_rows(c);
      unsigned char* sb = stage(st);
      float* srec = reinterpret_cast<float*>(sb);
      float* sth = reinterpret_cast<float*>(sb + ST::kRec);
      float* sg = sth + R * PL;
      if (FLAT) {
        // array by array over the chunk (all moment records, then theta, then
        // gradients), 16-byte pieces spread over all producer threads; the row
        // id of each piece comes from its lane in every warp by shuffle
        auto id_of = [&](int r) { return __shfl_sync(0xffffffffu, my_id, r & 31); };
#pragma unroll
        for (int j = 0; j < (R * kRecPieces + NP - 1) / NP; ++j) {
          const int p = j * NP + pt;
          const int r = p / kRecPieces;
          const uint32_t row = id_of(r);
          if (r < nv) {
            const int q = p - r * kRecPieces;
            cp_async16_h<HINT>(srec + r * (2 * SLOTS) + 4 * q, P.record + (size_t)row * P.stride + 4 * q);
          }
        }
        if (REC) {
#pragma unroll
          for (int j = 0; j < (R * kRowPieces + NP - 1) / NP; ++j) {
            const int p = j * NP + pt;
            const int r = p / kRowPieces;
            const uint32_t row = id_of(r);
            if (r < nv) {
              const int q = p - r * kRowPieces;
              cp_async16_h<HINT>(sth + r * PL + 4 * q, P.prec + roff(row, P.prs) + 4 * q);
            }
          }
#pragma unroll
          for (int j = 0; j < (R * kRowPieces + NP - 1) / NP; ++j) {
            const int p = j * NP + pt;
            const int r = p / kRowPieces;
            const uint32_t row = id_of(r);
            if (r < nv) {
              const int q = p - r * kRowPieces;
              if (P.grec_ca)
                cp_async16_ca(sg + r * PL + 4 * q, P.grec + roff(row, P.grs) + 4 * q);
              else
                cp_async16_h<HINT>(sg + r * PL + 4 * q, P.grec + roff(row, P.grs) + 4 * q);
            }
          }
        } else {
          // per-attribute tensors: 4-byte elements in chunk element order,
          // rotated per group like the consumers (balanced warps)
          using PS = ChunkShape<L, R, NP>;
#pragma unroll
          for (int gg = 0; gg < L::G; ++gg) {
            const int W = L::W(gg);
#pragma unroll
            for (int kk = 0; kk < PS::rounds(gg); ++kk) {
              const int i = kk * NP + ((pt + NP - (R * L::OFF(gg)) % NP) % NP);
              const int r = i / W;
              const uint32_t row = id_of(r);
              if (i < R * W && r < nv) {
                const uint32_t c = (uint32_t)(i - r * W);
                const int e = R * L::OFF(gg) + i;
                cp_async4(sth + e, P.g[gg].param + row * P.g[gg].ps + c);
                cp_async4(sg + e, P.g[gg].grad + row * P.g[gg].gs + c);
              }
            }
          }
        }
      }
      if (warp == 0 && lane < nv) {
        // row ids and bias factors ride the stage too, so the consumers
        // touch no global memory before their barrier; the clock read here
        // stalls only this producer warp, which runs chunks ahead
        if (!kDense) cp_async4(&s_crow[st][lane], P.rows + c * R + lane);
        const int tb = kDense ? P.global_t
                              : __ldg(reinterpret_cast<const int*>(P.record + (size_t)my_id * P.stride +
                                                                   2 * L::P)) + 1;
        cp_async8(&s_bc[st][lane], P.lut + 2 * (tb < P.lut_len ? tb : P.lut_len - 1));
      }
      for (int r = warp; !FLAT && r < nv; r += NPW) {  // warp-uniform
        const uint32_t row = __shfl_sync(0xffffffffu, my_id, r);
#pragma unroll
        for (int j = 0; j < (kPiecesPerRow + 31) / 32; ++j) {
          const int p = lane + 32 * j;
          if (p < kRecPieces) {
            cp_async16_h<HINT>(srec + r * (2 * SLOTS) + 4 * p, P.record + (size_t)row * P.stride + 4 * p);
          } else if (p < kRecPieces + kRowPieces) {
            const int q = p - kRecPieces;
            cp_async16_h<HINT>(sth + r * PL + 4 * q, P.prec + roff(row, P.prs) + 4 * q);
          } else if (p < kPiecesPerRow) {
            const int q = p - kRecPieces - kRowPieces;
            if (P.grec_ca)
              cp_async16_ca(sg + r * PL + 4 * q, P.grec + roff(row, P.grs) + 4 * q);
            else
              cp_async16_h<HINT>(sg + r * PL + 4 * q, P.grec + roff(row, P.grs) + 4 * q);
          }
        }
      }
      mbar_arrive_cp_async(&full_bar[st]);
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    }
  } else {
    // ------------------------------------------------------------------ consumers
    const int t = tid;
    StepConsts Kc = P.K;
    if (kCoupled) {
      const float nv = P.nv_dev ? (float)(*P.nv_dev) : (float)P.nv_host;
      Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
      if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
    }
    const StepConsts& K = kCoupled ? Kc : P.K;
    float2* const rec_base = reinterpret_cast<float2*>(P.record);
    const uint32_t rec_stride2 = (uint32_t)(P.stride / 2);
    int st = 0;
    int ep = 1;  // this use of stage st (epoch tag of its row flags)
    for (int c = (int)blockIdx.x; c < n_chunks; c += G) {
      const int nvalid = chunk_rows(c);
      if (kDense && t < R) s_crow[st][t] = (uint32_t)(c * R + t);
      mbar_wait(&full_bar[st], (unsigned)((ep - 1) & 1));
      const unsigned char* sb = stage(st);
      const float2* srec = reinterpret_cast<const float2*>(sb);
      const float* sth = reinterpret_cast<const float*>(sb + ST::kRec);
      const float* sg = sth + R * PL;
      const uint32_t* srow = s_crow[st];
      // row ids (sparse modes) and bias factors were staged by the producers
      const int tn = t < nvalid ? reinterpret_cast<const int*>(srec + t * SLOTS + L::P)[0] + 1 : 0;
      if (!STRICT && REC) {
        // gradients: the staged rows' 16-byte pieces (pad columns ignored);
        // activation domain: the opacity / scale columns of theta, on the
        // top threads (the gradient pieces leave them one piece short)
        constexpr int kQ = PL / 4;
#pragma unroll
        for (int j = 0; j < (R * kQ + NC - 1) / NC; ++j) {
          const int p = j * NC + t;
          const int r = p / kQ;
          if (p < R * kQ && r < nvalid) {
            const int q = p - r * kQ;
            const float4 v = reinterpret_cast<const float4*>(sg + r * PL)[q];
            const bool bad = !isfinite(v.x) || (4 * q + 1 < L::P && !isfinite(v.y)) ||
                             (4 * q + 2 < L::P && !isfinite(v.z)) ||
                             (4 * q + 3 < L::P && !isfinite(v.w));
            if (bad) {
              atomicMax(&s_badg[st][r], ep);
              s_any[st] = ep;
            }
          }
        }
        int dbase = 0;
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          const int role = L::ROLE(gg);
          if (role != GS_ROLE_OPACITY && role != GS_ROLE_SCALE) continue;
          const int W = L::W(gg);
          const float lam = role == GS_ROLE_OPACITY ? K.lam_op : K.lam_sc;
          if (lam != 0.f) {
#pragma unroll
            for (int kk = 0; kk < (R * W + NC - 1) / NC; ++kk) {
              const int i = kk * NC + (NC - 1 - t + NC - dbase % NC) % NC;
              const int r = i / W;
              if (i < R * W && r < nvalid && domain_bad(role, sth[r * PL + L::OFF(gg) + (i - r * W)])) {
                atomicMax(&s_badd[st][r], ep);
                s_any[st] = ep;
              }
            }
          }
          dbase += R * W;
        }
      } else if (!STRICT) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          const int W = L::W(gg);
          const int role = L::ROLE(gg);
          const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / W;
            if (i < R * W && r < nvalid) {
              const int e = sidx(gg, i, r);
              const bool bg = !isfinite(sg[e]);
              const bool bd = (role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
                              domain_bad(role, sth[e]);
              if (bg) atomicMax(&s_badg[st][r], ep);
              if (bd) atomicMax(&s_badd[st][r], ep);
              if (bg || bd) s_any[st] = ep;
            }
          }
        }
      }
      named_sync(1, NC);  // flags, row ids and bias factors of the chunk are final
      const bool any_bad = s_any[st] == ep || nvalid < R;
      auto row_ok = [&](int r) { return s_badg[st][r] != ep && s_badd[st][r] != ep; };
      if (t < nvalid) {
        ++c_vis;
        if (row_ok(t)) {
          int* const clk = reinterpret_cast<int*>(rec_base + (size_t)srow[t] * rec_stride2 + L::P);
          if (HINT & 2) __stcs(clk, tn); else *clk = tn;
          if (P.D.group >= 0) {
#pragma unroll
            for (int gg = 0; gg < L::G; ++gg)
              if (gg == P.D.group)
                densify_row(P.D, srow[t], sg + sidx(gg, t * L::W(gg), t), L::W(gg), 1);
          }
          ++c_step;
        } else if (s_badg[st][t] == ep) {
          ++c_badg;
        } else {
          ++c_badd;
        }
      }
      auto update = [&](int gg, int i, int r) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const int c = i - r * W;
        const int e = sidx(gg, i, r);
        const uint32_t row = srow[r];
        const float2 mv = srec[r * SLOTS + L::OFF(gg) + c];
        const float th = sth[e];
        float tnv, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, P.g[gg].lr, th, sg[e], mv.x, mv.y, s_bc[st][r], K, tnv, mn,
                             vn, ex, clipped);
        if (!kCoupled && role == GS_ROLE_OPACITY) {
          c_clo += clipped;
          s_exo += (double)ex;
        } else if (!kCoupled && role == GS_ROLE_SCALE) {
          c_cls += clipped;
          s_exs += (double)ex;
        }
        if (role == GS_ROLE_OPACITY) {
          c_apre += th > P.active_logit;
          c_apost += tnv > P.active_logit;
        }
        if (HINT & 2) {  // streaming (evict-first) stores
          __stcs(P.g[gg].param + roff(row, P.g[gg].ps) + (uint32_t)c, tnv);
          __stcs(rec_base + (size_t)row * rec_stride2 + L::OFF(gg) + c, make_float2(mn, vn));
        } else {
          P.g[gg].param[roff(row, P.g[gg].ps) + (uint32_t)c] = tnv;
          rec_base[(size_t)row * rec_stride2 + L::OFF(gg) + c] = make_float2(mn, vn);
        }
      };
      if (!any_bad) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const bool full = (kk + 1) * NC <= R * L::W(gg);  // compile-time
            if (full || i < R * L::W(gg)) update(gg, i, i / L::W(gg));
          }
        }
      } else {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / L::W(gg);
            if (i < R * L::W(gg) && r < nvalid && row_ok(r)) update(gg, i, r);
          }
        }
      }
      mbar_arrive(&empty_bar[st]);  // this thread's reads of the stage are done
      if (++st == S) {
        st = 0;
        ++ep;
      }
    }
  }
  cp_async_wait<0>();

  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce_n<GS_STEP_STATS, (NPW + NCW)>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f)
      P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter))
    final_reduce_n<GS_STEP_STATS, (NPW + NCW)>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out,
                                               is_max, s_red);
}

template <class L, int MODE, bool STRICT, int R, int S, int NPW, int NCW, int MINB, bool FLAT,
          bool REC = true, int HINT = 0>
void launch_ring(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  constexpr int bytes = S * WsStage<L, R>::kBytes;
  smem_opt_in<step_ring_kernel<L, MODE, STRICT, R, S, NPW, NCW, MINB, FLAT, REC, HINT>>(bytes);
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_ring_kernel<L, MODE, STRICT, R, S, NPW, NCW, MINB, FLAT, REC, HINT>
      <<<grid, (NPW + NCW) * 32, bytes, s>>>(P);
}

#if GS_BUILD_VARIANTS  // 1-D bulk-copy kernel (TMA op rate bound)
// ---------------------------------------------------------------------------
// TMA variant for row-interleaved records (parameters, gradients and the
// optimizer-state record all row-contiguous): one producer warp moves each
// visible row with three bulk copies (cp.async.bulk, SASS UBLKCP) — the
// 480-byte moment record, the 240-byte parameter row and the 240-byte
// gradient row — completing on the stage's "full" mbarrier by transaction
// count.  Consumers update in shared memory in place, then every good row is
// written back with two bulk stores (parameter row, moment record with the
// new clock); bad rows are never stored, so they stay untouched.  Compared
// with the cp.async gather variant this replaces ~60 16-byte copies and
// ~120 scattered 4/8-byte stores per row with 5 bulk operations.
// ---------------------------------------------------------------------------
template <class L, int R>
struct TmaStage {
  static constexpr int kSlots = L::P + 1;
  static constexpr int kPL = (L::P + 3) & ~3;
  static constexpr int kRecRow = kSlots * 8;  // moment record row incl. the clock slot
  static constexpr int kThRow = kPL * 4;      // parameter / gradient record row
  static constexpr int kRec = R * kRecRow;
  static constexpr int kTh = R * kThRow;
  static constexpr int kBytes = kRec + 2 * kTh;
  static_assert(kRecRow % 16 == 0 && kThRow % 16 == 0, "bulk copies move 16-byte multiples");
};

template <class L, int MODE, bool STRICT, int R, int S, int NCW, int MINB>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB) step_tma_kernel(const FixedParams P) {
  static_assert(R == 32, "one producer lane per row");
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NC = NCW * 32;
  using SH = ChunkShape<L, R, NC>;
  using ST = TmaStage<L, R>;
  constexpr int SLOTS = ST::kSlots;
  constexpr int PL = ST::kPL;
  extern __shared__ __align__(16) unsigned char smem[];  // bulk copies need 16-byte alignment
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];
  __shared__ int s_bad[S][R];
  __shared__ int s_any[S];
  __shared__ float2 s_bc[S][R];
  __shared__ uint32_t s_crow[S][R];
  __shared__ double s_red[GS_STEP_STATS * (NCW + 1)];

  const int tid = threadIdx.x;
  const bool producer = tid >= NC;
  int64_t n_rows = kDense ? P.max_rows : (int64_t)(*P.n_rows_dev);
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  const int64_t n_chunks = (n_rows + R - 1) / R;
  auto chunk_id = [&](int64_t k) { return (int64_t)blockIdx.x + k * gridDim.x; };
  auto chunk_rows = [&](int64_t k) -> int {
    const int64_t rem = n_rows - chunk_id(k) * R;
    return rem <= 0 ? 0 : (rem < R ? (int)rem : R);
  };
  auto stage = [&](int st) { return smem + st * ST::kBytes; };
  auto sidx = [](int gg, int i, int r) -> int { return r * PL + L::OFF(gg) + (i - r * L::W(gg)); };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NC);
    }
  }
  if (tid < R * S) s_bad[tid / R][tid % R] = 0;
  if (tid < S) s_any[tid] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0;
  double s_exo = 0.0, s_exs = 0.0;

  if (producer) {
    // ------------------------------------------------------------------ producer
    const int lane = tid - NC;
    auto fetch_id = [&](int64_t k) -> uint32_t {
      if (lane >= chunk_rows(k)) return 0u;
      const int64_t i = chunk_id(k) * R + lane;
      return kDense ? (uint32_t)i : (uint32_t)__ldg(P.rows + i);
    };
    uint32_t next_id = fetch_id(0);
    for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
      const int st = (int)(k % S);
      const uint32_t row = next_id;
      next_id = fetch_id(k + 1);
      if (k >= S) mbar_wait(&empty_bar[st], (unsigned)(((k / S) - 1) & 1));
      const int nv = chunk_rows(k);
      unsigned char* sb = stage(st);
      if (lane == 0)
        mbar_arrive_expect_tx(&full_bar[st], (uint32_t)nv * (ST::kRecRow + 2 * ST::kThRow));
      __syncwarp();
      if (lane < nv) {
        bulk_g2s(sb + lane * ST::kRecRow, P.record + (size_t)row * P.stride, ST::kRecRow,
                 &full_bar[st]);
        bulk_g2s(sb + ST::kRec + lane * ST::kThRow, P.prec + (size_t)row * P.prs, ST::kThRow,
                 &full_bar[st]);
        bulk_g2s(sb + ST::kRec + ST::kTh + lane * ST::kThRow, P.grec + (size_t)row * P.grs,
                 ST::kThRow, &full_bar[st]);
      }
    }
  } else {
    // ------------------------------------------------------------------ consumers
    const int t = tid;
    StepConsts Kc = P.K;
    if (kCoupled) {
      const float nv = P.nv_dev ? (float)(*P.nv_dev) : (float)P.nv_host;
      Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
      if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
    }
    const StepConsts& K = kCoupled ? Kc : P.K;
    float* const prec = const_cast<float*>(P.prec);
    for (int64_t k = 0; chunk_id(k) < n_chunks; ++k) {
      const int st = (int)(k % S);
      const int nvalid = chunk_rows(k);
      if (t < R)
        s_crow[st][t] = t < nvalid ? (kDense ? (uint32_t)(chunk_id(k) * R + t)
                                             : (uint32_t)__ldg(P.rows + chunk_id(k) * R + t))
                                   : 0u;
      mbar_wait(&full_bar[st], (unsigned)((k / S) & 1));
      unsigned char* sb = stage(st);
      float2* srec = reinterpret_cast<float2*>(sb);
      float* sth = reinterpret_cast<float*>(sb + ST::kRec);
      const float* sg = reinterpret_cast<const float*>(sb + ST::kRec + ST::kTh);
      const uint32_t* srow = s_crow[st];
      if (!STRICT) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
          const int W = L::W(gg);
          const int role = L::ROLE(gg);
          const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.f;
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / W;
            if (i < R * W && r < nvalid) {
              const int e = sidx(gg, i, r);
              int bad = isfinite(sg[e]) ? 0 : 1;
              if ((role == GS_ROLE_OPACITY || role == GS_ROLE_SCALE) && lam != 0.f &&
                  domain_bad(role, sth[e]))
                bad |= 2;
              if (bad) {
                atomicOr(&s_bad[st][r], bad);
                s_any[st] = 1;
              }
            }
          }
        }
      }
      int tn = 0;
      float2 bc = make_float2(1.f, 1.f);
      if (t < nvalid) {
        tn = reinterpret_cast<const int*>(srec + t * SLOTS + L::P)[0] + 1;
        bc = bias_factors(P.lut, P.lut_len, kDense ? P.global_t : tn, 0.0, 0.0);
      }
      named_sync(1, NC);  // bad flags final
      const bool any_bad = s_any[st] != 0 || nvalid < R;
      if (t < nvalid) {
        ++c_vis;
        const int bad = s_bad[st][t];
        if (bad == 0) {
          s_bc[st][t] = bc;
          if (P.D.group >= 0) {
#pragma unroll
            for (int gg = 0; gg < L::G; ++gg)
              if (gg == P.D.group)
                densify_row(P.D, srow[t], sg + sidx(gg, t * L::W(gg), t), L::W(gg), 1);
          }
          ++c_step;
        } else if (bad & 1) {
          ++c_badg;
        } else {
          ++c_badd;
        }
      }
      named_sync(1, NC);  // bias factors visible; the clock slots are read
      if (t < nvalid && s_bad[st][t] == 0) reinterpret_cast<int*>(srec + t * SLOTS + L::P)[0] = tn;
      auto update = [&](int gg, int i, int r) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const int c = i - r * W;
        const int e = sidx(gg, i, r);
        float2& mv = srec[r * SLOTS + L::OFF(gg) + c];
        const float th = sth[e];
        float tnv, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, P.g[gg].lr, th, sg[e], mv.x, mv.y, s_bc[st][r], K, tnv, mn,
                             vn, ex, clipped);
        if (!kCoupled && role == GS_ROLE_OPACITY) {
          c_clo += clipped;
          s_exo += (double)ex;
        } else if (!kCoupled && role == GS_ROLE_SCALE) {
          c_cls += clipped;
          s_exs += (double)ex;
        }
        if (role == GS_ROLE_OPACITY) {
          c_apre += th > P.active_logit;
          c_apost += tnv > P.active_logit;
        }
        sth[e] = tnv;
        mv = make_float2(mn, vn);
      };
      if (!any_bad) {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const bool full = (kk + 1) * NC <= R * L::W(gg);  // compile-time
            if (full || i < R * L::W(gg)) update(gg, i, i / L::W(gg));
          }
        }
      } else {
#pragma unroll
        for (int gg = 0; gg < L::G; ++gg) {
#pragma unroll
          for (int kk = 0; kk < SH::rounds(gg); ++kk) {
            const int i = kk * NC + ((t + NC - (R * L::OFF(gg)) % NC) % NC);
            const int r = i / L::W(gg);
            if (i < R * L::W(gg) && r < nvalid && s_bad[st][r] == 0) update(gg, i, r);
          }
        }
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> bulk-store reads
      named_sync(1, NC);         // the chunk's rows are final in shared memory
      if (t < R) {
        // row t's stores; the stage is released one chunk later, once they
        // have read shared memory (wait_group.read 1), so the store latency
        // overlaps the next chunk's update instead of stalling this one
        if (t < nvalid && s_bad[st][t] == 0) {
          const uint32_t row = srow[t];
          bulk_s2g(prec + (size_t)row * P.prs, sth + t * PL, ST::kThRow);
          bulk_s2g(P.record + (size_t)row * P.stride, srec + t * SLOTS, ST::kRecRow);
        }
        bulk_commit();  // one (possibly empty) group per chunk
        s_bad[st][t] = 0;
        if (t == 0) s_any[st] = 0;
        bulk_wait_read1();
        if (k > 0) mbar_arrive(&empty_bar[(int)((k - 1) % S)]);
      } else {
        mbar_arrive(&empty_bar[st]);
      }
    }
    bulk_wait0();
  }

  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce_n<GS_STEP_STATS, (NCW + 1)>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f)
      P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter))
    final_reduce_n<GS_STEP_STATS, (NCW + 1)>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out,
                                             is_max, s_red);
}

template <class L, int MODE, bool STRICT, int R, int S, int NCW, int MINB>
void launch_tma(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  constexpr int bytes = S * TmaStage<L, R>::kBytes;
  smem_opt_in<step_tma_kernel<L, MODE, STRICT, R, S, NCW, MINB>>(bytes);
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_tma_kernel<L, MODE, STRICT, R, S, NCW, MINB><<<grid, (NCW + 1) * 32, bytes, s>>>(P);
}

#endif  // GS_BUILD_VARIANTS (1-D bulk copies)

}  // namespace gs

#include "gs_step_sh3_tma.cuh"

namespace gs {

int fixed_variant();  // gs_step_sh3.cu: GS_FIXED_VARIANT / gs_set_fixed_variant

#if GS_BUILD_VARIANTS
template <class L, int MODE, bool STRICT, int R, int MINB, int NT = kFixedThreads>
void launch_fixed_v(const FixedParams& P, int64_t max_rows, cudaStream_t s) {
  const int64_t chunks = (max_rows + R - 1) / R;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)gs_sm_count() * MINB));
  step_fixed_kernel<L, MODE, STRICT, R, MINB, NT><<<grid, NT, 0, s>>>(P);
}

// Measured alternatives of the record and per-attribute kernels (results
// identical).  Returns false for an unknown variant.
template <class L, int MODE, bool STRICT>
bool launch_variant(const FixedParams& P, int64_t max_rows, int kind, int v, cudaStream_t s) {
  if (kind == 2) {
    switch (v) {
      case 8: launch_ws<L, MODE, STRICT, 32, 3, 3, 8, 2, true>(P, max_rows, s); return true;
      case 9: launch_tma<L, MODE, STRICT, 32, 6, 12, 1>(P, max_rows, s); return true;
      case 10: launch_tma<L, MODE, STRICT, 32, 3, 4, 2>(P, max_rows, s); return true;
      case 11: launch_ws<L, MODE, STRICT, 32, 3, 3, 8, 2, true, true>(P, max_rows, s); return true;
      case 12: launch_tma<L, MODE, STRICT, 32, 3, 8, 2>(P, max_rows, s); return true;
      case 13: launch_ring<L, MODE, STRICT, 32, 3, 3, 8, 2, false>(P, max_rows, s); return true;
      case 14: launch_ring<L, MODE, STRICT, 32, 3, 2, 8, 2, true>(P, max_rows, s); return true;
      case 16: launch_ring<L, MODE, STRICT, 32, 2, 2, 6, 3, true>(P, max_rows, s); return true;
      case 17: launch_ring<L, MODE, STRICT, 32, 3, 3, 8, 2, true>(P, max_rows, s); return true;
      case 18: launch_ring<L, MODE, STRICT, 32, 2, 2, 8, 2, true>(P, max_rows, s); return true;
      case 19: launch_ring<L, MODE, STRICT, 32, 2, 4, 8, 2, true>(P, max_rows, s); return true;
      case 20: launch_ring<L, MODE, STRICT, 32, 2, 3, 8, 2, true, true, 0>(P, max_rows, s); return true;
      default: return false;
    }
  }
  switch (v) {
    case 1: launch_fixed_v<L, MODE, STRICT, 64, 2>(P, max_rows, s); return true;
    case 2: launch_pipe<L, MODE, STRICT, 32, 2, 3>(P, max_rows, s); return true;
    case 3: launch_pipe2<L, MODE, STRICT, 32, 2, 3>(P, max_rows, s); return true;
    case 4: launch_ws<L, MODE, STRICT, 32, 3, 2, 8, 2>(P, max_rows, s); return true;
    case 5: launch_pipe2<L, MODE, STRICT, 32, 3, 2>(P, max_rows, s); return true;
    case 6: launch_ws<L, MODE, STRICT, 32, 3, 2, 6, 2>(P, max_rows, s); return true;
    // ring kernel on per-attribute tensors: a shuffle per 4-byte element costs
    // the producers more than the barrier it saves (0.81 vs 0.78 ms on c3)
    case 7: launch_ring<L, MODE, STRICT, 32, 3, 3, 8, 2, true, false>(P, max_rows, s); return true;
    case 19: launch_ws<L, MODE, STRICT, 32, 3, 3, 8, 2>(P, max_rows, s); return true;  // 3 stages
    default: return false;
  }
}
#endif  // GS_BUILD_VARIANTS

// kind: 0 dense per-attribute rows, 1 strided rows (per-element gathers),
// 2 row-interleaved parameter + gradient records.  M: tensor maps of the
// records when the TMA kernel may run (device-resident, 16-byte strides,
// rows of >= 64 floats), else null.
template <class L, int MODE, bool STRICT>
void launch_fixed(const FixedParams& P, const TmaMaps* M, int64_t max_rows, int kind,
                  cudaStream_t s) {
  // the densification statistics run in the default kernels only
  const int v = P.D.group >= 0 ? 0 : fixed_variant();
#if GS_BUILD_VARIANTS
  if (v > 0 && v != 21 && launch_variant<L, MODE, STRICT>(P, max_rows, kind, v, s)) return;
#endif
  if (kind == 2) {
    // records: 2-D TMA row gathers / scatters (tile::gather4 / scatter4,
    // gs_step_sh3_tma.cuh) when the records allow them; the cp.async ring
    // otherwise (host-mapped gradients, compact 240-byte rows) or on request
    // (variant 21)
    if (M != nullptr && v != 21) {
      // shape: (stages, consumer warps, CTAs / SM).  3 x 8 x 2 measured best
      // on c3 (K2 0.532 ms, 0.86 of the copy peak; 2 stages 0.567 ms) and
      // on c5 at 100% visibility (0.94); profiles/r02/tma4_shape_sweep.txt.
      // GS_TMA4_SHAPE selects the measured alternatives (identical results).
#if GS_BUILD_VARIANTS
      static const int shape = getenv("GS_TMA4_SHAPE") ? atoi(getenv("GS_TMA4_SHAPE")) : 0;
      switch (shape) {
        case 1: launch_tma4<L, MODE, STRICT, 2, 8, 2>(P, *M, max_rows, s); return;
        case 2: launch_tma4<L, MODE, STRICT, 3, 12, 2>(P, *M, max_rows, s); return;
        case 3: launch_tma4<L, MODE, STRICT, 2, 8, 3>(P, *M, max_rows, s); return;
        case 4: launch_tma4<L, MODE, STRICT, 3, 6, 2>(P, *M, max_rows, s); return;
        case 5: launch_tma4<L, MODE, STRICT, 3, 10, 2>(P, *M, max_rows, s); return;
        default: break;
      }
#endif
      // short lists (under 16 chunks per CTA slot whatever the count): the
      // bias warp, so the loader's per-chunk work is only the TMA issue
      // (c1 K2 0.0258 against 0.0277 ms; c3 0.566 against 0.544 ms,
      // profiles/r02/small_clouds.txt).  GS_TMA4_BW=0/1 forces one.
      static const int force = getenv("GS_TMA4_BW") ? atoi(getenv("GS_TMA4_BW")) : -1;
      const bool bw = force >= 0 ? force != 0
                                 : (max_rows + 31) / 32 < (int64_t)kBalancedChunksPerCta * 2 *
                                                              gs_sm_count();
      if (bw) launch_tma4<L, MODE, STRICT, 3, 8, 2, 0, true>(P, *M, max_rows, s);
      else launch_tma4<L, MODE, STRICT, 3, 8, 2>(P, *M, max_rows, s);
      return;
    }
    if (P.wide) {  // > 2^32 parameter-record elements: 64-bit row offsets
      launch_ring<L, MODE, STRICT, 32, 2, 3, 8, 2, true, true, 1 | 32>(P, max_rows, s);
      return;
    }
    // 2 stages beat 3 on every workload measured (c3 K2 0.595 vs 0.627 ms,
    // profiles/r01/ring_stage_sweep.txt); 2 or 4 producer warps do worse;
    // L2::256B prefetch-size hint on the gathers: 0.595 -> 0.592 ms (c3)
    launch_ring<L, MODE, STRICT, 32, 2, 3, 8, 2, true, true, 1>(P, max_rows, s);
    return;
  }
  launch_ws<L, MODE, STRICT, 32, 2, 3, 8, 2>(P, max_rows, s);
}

// Fused K1 + K2 on records (the fused check): the TMA kernel's loader
// compacts the visibility mask itself (mask_kind 1: uint8, 2: int32 radii;
// 3 / 4: the same, two-phase compaction with balanced shares, for clouds
// under 16 mask tiles per CTA slot: c1 step 0.0316 against 0.0345 ms for
// K1 + K2, c2 0.105 against 0.111; ties from 400k rows to 3M).
// low_vis: the bias warp variant, for sparse masks where the loader's scan
// is the bottleneck (c5 at 1%: 0.190 against 0.223 ms); on dense masks the
// loader-staged bias factors win (c3: 0.534 against 0.580 ms)
// (profiles/r02/fused_k1_variants.txt).  GS_TMA4_BW=0/1 forces one.
template <class L, int MODE>
void launch_fixed_masked(const FixedParams& P, const TmaMaps& M, int64_t n_rows, int mask_kind,
                         const void* mask, bool low_vis, cudaStream_t s) {
  static const int force = getenv("GS_TMA4_BW") ? atoi(getenv("GS_TMA4_BW")) : -1;
  const bool bw = force >= 0 ? force != 0 : low_vis;
#if GS_BUILD_VARIANTS
  static const int mtb = getenv("GS_TMA4_MTB") ? atoi(getenv("GS_TMA4_MTB")) : 1024;
  if (mask_kind == 1 && mtb == 512) {
    if (bw) launch_tma4<L, MODE, false, 3, 8, 2, 1, true, 512>(P, M, n_rows, s, mask);
    else launch_tma4<L, MODE, false, 3, 8, 2, 1, false, 512>(P, M, n_rows, s, mask);
    return;
  }
#endif
  if (mask_kind >= 3) {  // two-phase: the bias warp (c3-sized: 0.563 against 0.652 ms)
    if (force == 0) {
      if (mask_kind == 4) launch_tma4<L, MODE, false, 3, 8, 2, 4, false>(P, M, n_rows, s, mask);
      else launch_tma4<L, MODE, false, 3, 8, 2, 3, false>(P, M, n_rows, s, mask);
    } else {
      if (mask_kind == 4) launch_tma4<L, MODE, false, 3, 8, 2, 4, true>(P, M, n_rows, s, mask);
      else launch_tma4<L, MODE, false, 3, 8, 2, 3, true>(P, M, n_rows, s, mask);
    }
    return;
  }
  // sparse uint8 masks on big clouds (>= 64 one-KB tiles per CTA slot): 3
  // CTAs per SM (2 stages, 4 consumer warps, 512-byte mask tiles), i.e. 3
  // mask-scanning loaders per SM, the loader being the busy role there
  // (c5 at 1%: 0.190 against 0.196 ms, at 3%: 0.476 against 0.504; on the
  // 6.25M-row shard the extra CTAs lose, 0.039 against 0.037;
  // profiles/r02/small_clouds.txt).  GS_LOWVIS_SHAPE=0/1 forces it off/on.
  static const int lv = getenv("GS_LOWVIS_SHAPE") ? atoi(getenv("GS_LOWVIS_SHAPE")) : -1;
  const bool big = (n_rows + 1023) / 1024 >= 64 * 2 * (int64_t)gs_sm_count();
  if (mask_kind == 1 && bw && (lv == 1 || (lv < 0 && big))) {
    launch_tma4<L, MODE, false, 2, 4, 3, 1, true, 512>(P, M, n_rows, s, mask);
    return;
  }
  if (mask_kind == 1 && bw && lv == 2) {
    launch_tma4<L, MODE, false, 2, 6, 3, 1, true, 512>(P, M, n_rows, s, mask);
    return;
  }
  if (mask_kind == 2) {
    if (bw) launch_tma4<L, MODE, false, 3, 8, 2, 2, true>(P, M, n_rows, s, mask);
    else launch_tma4<L, MODE, false, 3, 8, 2, 2, false>(P, M, n_rows, s, mask);
  } else {
    if (bw) launch_tma4<L, MODE, false, 3, 8, 2, 1, true>(P, M, n_rows, s, mask);
    else launch_tma4<L, MODE, false, 3, 8, 2, 1, false>(P, M, n_rows, s, mask);
  }
}

}  // namespace gs
