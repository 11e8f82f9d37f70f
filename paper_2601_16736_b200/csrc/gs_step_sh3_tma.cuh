// K2 on the row records with Blackwell 2-D TMA row gathers and scatters
// (cp.async.bulk.tensor.2d ... tile::gather4 / tile::scatter4, SASS UTMALDG /
// UTMASTG): the default SH-3 step for device-resident parameter, gradient and
// moment records (included by gs_step_sh3.cuh).
//
// A CTA walks chunks of 32 visible rows through an S-stage shared-memory
// ring (3 stages, 2 CTAs per SM by default; 2 stages, 3 CTAs per SM for
// sparse masks on big clouds).  Where the chunks come from (MASK, below):
// an index list (dealt grid-stride, the last round split evenly), a mask
// streamed through the loader (1-KB tiles grid-stride with an optional
// dynamic tail, or per-CTA slices on small clouds), or a mask compacted in
// two phases around a grid barrier.  Warp roles:
//   loader  (warp NCW)     per chunk, lanes 0..7 each issue three gather4
//                          operations (4 rows each) for the moment records
//                          (480 B of every 512-B row), the parameter rows and
//                          the gradient rows (256 B each), completing on the
//                          stage's "full" mbarrier by transaction bytes; every
//                          lane also stages its row id and the bias factors of
//                          its row's next clock (from the bias LUT).
//   consumers (warps 0..NCW-1)  check, then update the staged rows IN PLACE
//                          (theta, m, v, clock), then fence the async proxy
//                          and arrive on the stage's "done" mbarrier.
//   storer  (warp NCW+1)   lanes 0..7 scatter4 the parameter rows and the
//                          moment records back, wait until the bulk stores
//                          have read the stage, and hand it back to the
//                          loader ("empty" mbarrier).
//   bias    (warp NCW+2, BW only)  turns the landed clocks into bias factors,
//                          so the loader only scans masks and issues copies.
// The statistics: per-thread counters and sums, a block tree, per-CTA
// partials and a last-CTA fold in CTA order (deterministic).
// Rows past the end of the index list get row id n_rows: the gathers fill
// them with zeros and the scatters drop them (out of the tensor's bounds).
// A skipped (bad) row is left unchanged in the stage, so its scatter writes
// back the bytes it read.  Per-row math is gs_common.cuh::update_element in
// the same element order as step_ring_kernel, so results are bit-identical.
//
// Compared with the cp.async ring (60 16-byte LSU copies and ~120 scattered
// 4/8-byte stores per row), a 32-row chunk costs 24 + 16 TMA operations and
// the SM issue slots go to the arithmetic.  Probe on B200 (scripts/
// tma4_probe.cu, profiles/r02/tma4_probe*.txt): the data movement alone runs
// at 0.86 of the copy peak for 30% i.i.d. rows and 0.94 for all rows; the
// kernel reaches 0.86 / 0.94 (profiles/r02/tma4_shape_sweep.txt).
#pragma once

#include <cuda.h>

#include <type_traits>

namespace gs {

struct TmaMaps {
  CUtensorMap rec;  // moment record  [n_rows, stride] fp32, box {2*(P+1), 1}
  CUtensorMap prm;  // parameter record [n_rows, prs], box {64, 1}
  CUtensorMap grd;  // gradient record  [n_rows, grs], box {64, 1}
};

template <class L, int R>
struct Tma4Stage {
  static constexpr int kSlots = L::P + 1;   // float2 slots of a moment record row
  static constexpr int kRecRow = kSlots * 8;
  static constexpr int kPT = 64;            // staged parameter / gradient row (floats)
  static constexpr int kRec = R * kRecRow;
  static constexpr int kTh = R * kPT * 4;
  static constexpr int kBytes = kRec + 2 * kTh;
  static_assert(kPT >= L::P, "parameter row box");
  static_assert((4 * kRecRow) % 128 == 0 && (4 * kPT * 4) % 128 == 0 && kBytes % 128 == 0,
                "every 4-row TMA box lands 128-byte aligned");
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_gather4(void* smem, const CUtensorMap* map, int r0, int r1,
                                            int r2, int r3, uint64_t* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(s),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tma_scatter4(const CUtensorMap* map, const void* smem, int r0,
                                             int r1, int r2, int r3) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group"
      " [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(map),
      "r"(s), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

// MASK: 0 = the compacted index list (P.rows, *P.n_rows_dev rows; dense
// mode: every row), 1 = a uint8 visibility mask, 2 = int32 radii (> 0 is
// visible): the loader compacts the mask itself (fused K1, below);
// 3 / 4 = the same masks compacted in two phases (below): every CTA first
// compacts an even slice of the mask into P.tp_ids, a grid barrier
// publishes the per-CTA counts, then every CTA steps an even contiguous
// share of the visible rows (one wave of CTAs, all resident).
// BW: a fourth role, the bias warp (warp NCW+2), turns the staged clocks
// into bias factors after the gathers land, so the loader's per-chunk work
// is only the TMA issue (the mask-scanning loader); without it the loader
// reads each row's clock and LUT entry itself.
// Index lists shorter than this many chunks per CTA deal whole rounds of G
// chunks grid-stride and split the last, partial round evenly over the CTAs.
constexpr int kBalancedChunksPerCta = 16;

// A list of n positions over G CTAs: spans k < full of CTA b are the chunks
// (k * G + b) * 32 .. + 32; the last span is the CTA's even share of the
// remaining n - 32 * G * full positions (< 32 each, possibly empty).
struct TailSplit {
  int full;  // whole rounds of G chunks
  int n;
  __device__ int n_spans() const { return full + 1; }
  __device__ void span(int k, int b, int G, int& lo, int& hi) const {
    if (k < full) {
      lo = (k * G + b) * 32;
      hi = lo + 32;
    } else if (k == full) {
      const int base = full * G * 32;
      const int64_t rem = n - base;
      lo = base + (int)(rem * b / G);
      hi = base + (int)(rem * (b + 1) / G);
    } else {
      lo = hi = 0;
    }
  }
};
__device__ __forceinline__ TailSplit tail_split(int n, int G) { return TailSplit{n / (32 * G), n}; }

template <class L, int MODE, bool STRICT, int S, int NCW, int MINB, int MASK, bool BW = false,
          int MTB = 1024>
__global__ void __launch_bounds__((NCW + 2 + (BW ? 1 : 0)) * 32, MINB)
    step_tma4_kernel(const FixedParams P, const __grid_constant__ TmaMaps M, const void* vis_mask,
                     unsigned long long* trc) {
  constexpr int NWARPS = NCW + 2 + (BW ? 1 : 0);
  constexpr int R = 32;
  constexpr bool kDense = MODE == GS_MODE_COUPLED_ADAM;
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  constexpr int NC = NCW * 32;
  constexpr int SLOTS = L::P + 1;
  using SH = ChunkShape<L, R, NC>;
  using ST = Tma4Stage<L, R>;
  constexpr int PT = ST::kPT;
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t data_bar[BW ? S : 1];  // BW: the gathers of the stage landed
  __shared__ __align__(8) uint64_t done_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];
  __shared__ int s_badg[S][R];  // == epoch: non-finite gradient in this use of the stage
  __shared__ int s_badd[S][R];  // == epoch: activation-domain violation
  __shared__ int s_any[S];
  __shared__ float2 s_bc[S][R];
  __shared__ uint32_t s_crow[S][R];
  __shared__ int s_nv[S];  // rows of the chunk in the stage; -1 ends the CTA's chunk stream
  constexpr bool kStreamMask = MASK == 1 || MASK == 2;
  // pending visible ids (fused compaction): one tile's rows + a partial chunk
  constexpr int kPend = kStreamMask ? 2 * (MASK == 2 ? MTB / 4 : MTB) : 1;
  __shared__ uint32_t s_pend[kPend];
  // 6 KB of mask tiles in flight (4 KB at 3 CTAs per SM, to fit)
  constexpr int kMaskRing = kStreamMask ? (MINB >= 3 ? 4096 : 6144) / MTB : 1;
  __shared__ __align__(128) unsigned char s_mask[kMaskRing][kStreamMask ? MTB : 16];
  __shared__ __align__(8) uint64_t mask_bar[kMaskRing];
  __shared__ double s_red[GS_STEP_STATS * NWARPS];
  constexpr bool kTwoPhase = MASK >= 3;
  constexpr int kNT = NWARPS * 32;
  __shared__ int s_pref[kTwoPhase ? kNT + 1 : 1];  // exclusive prefix of the CTA counts
  __shared__ int s_wsum[kTwoPhase ? NWARPS : 1];
  // TMA boxes land 128-byte aligned (the host adds 128 bytes of slack)
  unsigned char* const smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) GS_STAMP(trc, 0);
  int n_rows = (kDense || MASK != 0) ? (int)P.max_rows : *P.n_rows_dev;
  if (STRICT && *P.abort_flag != 0) n_rows = 0;
  const int n_chunks = (n_rows + R - 1) / R;
  const int G = (int)gridDim.x;
  const int oob = (int)P.max_rows;  // row id past the tensors: zero-filled / dropped
  auto chunk_rows = [&](int c) -> int {
    const int rem = n_rows - c * R;
    return rem <= 0 ? 0 : (rem < R ? rem : R);
  };
  auto stage = [&](int st) { return smem + st * ST::kBytes; };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 32);  // the loader's (or bias warp's) lanes (+ tx without BW)
      if (BW) mbar_init(&data_bar[s], 1);  // loader lane 0 + tx
      mbar_init(&done_bar[s], NC);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kMaskRing; ++s) mbar_init(&mask_bar[s], 1);
  }
  if (tid < R * S) {
    s_badg[tid / R][tid % R] = 0;
    s_badd[tid / R][tid % R] = 0;
  }
  if (tid < S) s_any[tid] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  int tp_total = 0;  // two-phase: the mask's visible count
  if constexpr (kTwoPhase) {
    // ---- phase A (every thread): compact granules [g0, g1) of the mask
    // (16 bytes each: 16 uint8 rows or 4 radii) into P.tp_ids from row
    // g0 * Q on, in ascending row order, one block-wide scan per pass
    constexpr int kEsz = MASK == 3 ? 1 : 4;
    constexpr int Q = 16 / kEsz;
    const int64_t nr = n_rows;
    const int64_t ng = (nr + Q - 1) / Q;
    const int64_t g0 = ng * blockIdx.x / G, g1 = ng * (blockIdx.x + 1) / G;
    const unsigned char* gm = reinterpret_cast<const unsigned char*>(vis_mask);
    int run = 0;
    for (int64_t gb = g0; gb < g1; gb += kNT) {
      const int64_t g = gb + tid;
      uint32_t bits = 0;
      if (g < g1) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if ((g + 1) * Q <= nr) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(gm) + g);
          w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
        } else {  // ragged end of the mask: element reads, zero past the rows
          for (int by = 0; by < 16; ++by)
            if (g * 16 + by < nr * kEsz) w[by >> 2] |= (uint32_t)gm[g * 16 + by] << (8 * (by & 3));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (MASK == 3) {
#pragma unroll
            for (int e = 0; e < 4; ++e) bits |= (((w[j] >> (8 * e)) & 0xffu) != 0u) << (4 * j + e);
          } else {
            bits |= (uint32_t)((int)w[j] > 0) << j;
          }
        }
      }
      const int cnt = __popc(bits);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      int wpre = 0, tot = 0;
#pragma unroll
      for (int w2 = 0; w2 < NWARPS; ++w2) {
        const int x = s_wsum[w2];
        wpre += w2 < warp ? x : 0;
        tot += x;
      }
      int pos = run + wpre + incl - cnt;
      int32_t* dst = P.tp_ids + g0 * Q;
      for (uint32_t x = bits; x; x &= x - 1) dst[pos++] = (int32_t)(g * Q + __ffs(x) - 1);
      run += tot;
      __syncthreads();  // s_wsum is rewritten by the next pass
    }
    if (tid == 0) {
      P.tp_counts[blockIdx.x] = run;
      GS_STAMP(trc, 12);
    }
    grid_barrier(P.tp_bar);
    if (tid == 0) GS_STAMP(trc, 13);
    // ---- phase B: exclusive prefix of the G counts (G <= kNT), this CTA's
    // even share [p0, p1) of the visible positions
    const int cnt = tid < G ? __ldcg(P.tp_counts + tid) : 0;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int wpre = 0, tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < NWARPS; ++w2) {
      const int x = s_wsum[w2];
      wpre += w2 < warp ? x : 0;
      tot += x;
    }
    if (tid < G) s_pref[tid] = wpre + incl - cnt;
    if (tid == 0) s_pref[G] = tot;
    __syncthreads();
    tp_total = tot;
  }

  unsigned c_vis = 0, c_step = 0, c_badg = 0, c_badd = 0, c_apre = 0, c_apost = 0, c_clo = 0,
           c_cls = 0, c_runs = 0;
  double s_exo = 0.0, s_exs = 0.0;

  if (warp == NCW) {
    // ------------------------------------------------------------------ loader
    int st = 0, k = 0;
    unsigned ph = 0;
#ifdef GS_TRACE
    long long tr_t0 = clock64(), tr_empty = 0, tr_mask = 0;  // loader wait cycles
#define GS_TRACE_WAIT(acc, stmt)     \
  do {                               \
    const long long t_ = clock64();  \
    stmt;                            \
    acc += clock64() - t_;           \
  } while (0)
#else
#define GS_TRACE_WAIT(acc, stmt) stmt
#endif
    // one chunk into the next stage: lane i's row id (oob past nv), nv rows;
    // nv < 0 ends the stream (no data, the consumers and the storer exit)
    auto emit = [&](int my_id, int nv) {
      if (k >= S) GS_TRACE_WAIT(tr_empty, mbar_wait(&empty_bar[st], ph ^ 1u));
      unsigned char* sb = stage(st);
      uint64_t* tbar = BW ? &data_bar[st] : &full_bar[st];  // the gathers complete here
      if (nv > 0) {
        if (lane == 0) mbar_expect_tx(tbar, ST::kBytes);
        __syncwarp();
        const int q = (4 * lane) & 31;
        const int r0 = __shfl_sync(0xffffffffu, my_id, q);
        const int r1 = __shfl_sync(0xffffffffu, my_id, q + 1);
        const int r2 = __shfl_sync(0xffffffffu, my_id, q + 2);
        const int r3 = __shfl_sync(0xffffffffu, my_id, q + 3);
        // layout hint: rows that do not continue the previous row's run
        const int prev = __shfl_up_sync(0xffffffffu, my_id, 1);
        const unsigned starts =
            __ballot_sync(0xffffffffu, lane < nv && (lane == 0 || prev + 1 != my_id));
        if (lane == 0) c_runs += __popc(starts);
        if (lane < R / 4) {
          tma_gather4(sb + lane * 4 * ST::kRecRow, &M.rec, r0, r1, r2, r3, tbar);
          tma_gather4(sb + ST::kRec + lane * 4 * PT * 4, &M.prm, r0, r1, r2, r3, tbar);
          tma_gather4(sb + ST::kRec + ST::kTh + lane * 4 * PT * 4, &M.grd, r0, r1, r2, r3, tbar);
        }
        // row ids and the bias factors of the row's next clock ride the
        // stage, so the consumers touch no global memory before their
        // barrier (bias factors read by the consumers: c3 K2 0.585 ms
        // against 0.535)
        if (my_id != oob && BW) {
          s_crow[st][lane] = (uint32_t)my_id;
        } else if (my_id != oob) {
          s_crow[st][lane] = (uint32_t)my_id;
          const int tb = kDense ? P.global_t
                                : __ldg(reinterpret_cast<const int*>(P.record + (size_t)my_id * P.stride +
                                                                     2 * L::P)) + 1;
          s_bc[st][lane] = __ldg(reinterpret_cast<const float2*>(P.lut) + (tb < P.lut_len ? tb : P.lut_len - 1));
        }
      }
      if (lane == 0) s_nv[st] = nv;
      if (BW) {
        __syncwarp();  // row ids and the chunk size are written before lane 0 arrives
        if (lane == 0) {
          mbar_arrive(&data_bar[st]);
        }
      } else {
        mbar_arrive(&full_bar[st]);
      }
      if (k == 0 && lane == 0) GS_STAMP(trc, 1);
      ++k;
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    };
    if constexpr (MASK == 0) {
      if (n_chunks < kBalancedChunksPerCta * G) {
        // few chunks per CTA: whole rounds of G chunks grid-stride (the
        // CTAs stay on one window of the list: DRAM locality), then the
        // last partial round split evenly, so the CTAs finish together
        // (grid-stride alone leaves a chunk of imbalance: 5 vs 6 at c1)
        const TailSplit ts = tail_split(n_rows, G);
        auto fetch = [&](int k) -> int {
          int b, e;
          ts.span(k, (int)blockIdx.x, G, b, e);
          const int i = b + lane;
          return i < e ? (kDense ? i : __ldg(P.rows + i)) : oob;
        };
        int next_id = fetch(0);
        for (int k = 0; k < ts.n_spans(); ++k) {
          const int my_id = next_id;
          int b, e;
          ts.span(k, (int)blockIdx.x, G, b, e);
          next_id = fetch(k + 1);
          if (e > b) emit(my_id, e - b);
        }
      } else {
        auto fetch_id = [&](int c) -> int {
          if (c >= n_chunks || lane >= chunk_rows(c)) return oob;
          const int i = c * R + lane;
          return kDense ? i : __ldg(P.rows + i);
        };
        int next_id = fetch_id((int)blockIdx.x);
        for (int c = (int)blockIdx.x; c < n_chunks; c += G) {
          const int my_id = next_id;
          next_id = fetch_id(c + G);
          emit(my_id, chunk_rows(c));
        }
      }
    } else if constexpr (kTwoPhase) {
      // two-phase: positions [p0, p1) of the visible list; position p lives
      // in the slice of CTA c = max{c : pref[c] <= p} at row offset
      // g0(c) * Q, index p - pref[c]
      // positions dealt like the short index lists above: whole rounds of
      // G chunks grid-stride, the last round split evenly
      constexpr int Q = MASK == 3 ? 16 : 4;
      const int64_t ng = ((int64_t)n_rows + Q - 1) / Q;
      const TailSplit ts = tail_split(tp_total, G);
      int owner = 0;  // positions only grow: search from the last owner
      auto fetch = [&](int k) -> int {
        int b, e;
        ts.span(k, (int)blockIdx.x, G, b, e);
        const int p = b + lane;
        if (p >= e) return oob;
        int lo = owner, hi = G - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_pref[mid] <= p) lo = mid;
          else hi = mid - 1;
        }
        owner = lo;
        return __ldcg(P.tp_ids + ng * owner / G * Q + (p - s_pref[owner]));
      };
      int next_id = fetch(0);
      for (int k = 0; k < ts.n_spans(); ++k) {
        const int my_id = next_id;
        int b, e;
        ts.span(k, (int)blockIdx.x, G, b, e);
        next_id = fetch(k + 1);
        if (e > b) emit(my_id, e - b);
      }
    } else {
      // fused compaction: the CTA takes 1-KB mask tiles grid-stride (1024
      // uint8 rows or 256 int32 radii; small masks: tiles of its own slice,
      // below); lane 0 streams them into a
      // kMaskRing-deep shared-memory ring with 1-D bulk copies (mbarrier tx
      // counts); each lane takes 32 consecutive uint8 rows (two 16-byte
      // reads) or 16 radii, one warp scan per tile packs the
      // visible ids into a ring of pending ids, and every 32 of them leave
      // as one chunk (ids need no order: rows are independent).  The host
      // runs this path for 16-byte-aligned masks only.
      constexpr int kTileBytes = MTB;
      static_assert(MASK != 1 || MTB == 512 || MTB == 1024, "16 or 32 mask bytes per lane");
      constexpr int kEsz = MASK == 1 ? 1 : 4;
      constexpr int kRowsPerTile = kTileBytes / kEsz;
      constexpr int kLane = MASK == 1 ? MTB / 32 : 64;  // mask bytes per lane
      constexpr int kReads = kLane / 16;              // 16-byte smem reads per lane per tile
      const int64_t nr = n_rows;
      const int n_tiles = (int)((nr + kRowsPerTile - 1) / kRowsPerTile);
      const unsigned char* gmask = reinterpret_cast<const unsigned char*>(vis_mask);
      // small masks (under kBalancedChunksPerCta tiles per CTA): every CTA
      // scans its own contiguous 16-byte-aligned slice of the rows, in 1-KB
      // tiles (dealt grid-stride, a few tiles would leave most CTAs idle)
      constexpr int64_t kAlign = 16 / kEsz;  // rows per 16 mask bytes
      const bool range_mode =
          P.mask_slices == 0 ? n_tiles < kBalancedChunksPerCta * G : P.mask_slices == 1;
      int64_t r_lo = 0, r_hi = nr;
      if (range_mode) {
        const int64_t na = (nr + kAlign - 1) / kAlign;
        r_lo = na * blockIdx.x / G * kAlign;
        r_hi = na * (blockIdx.x + 1) / G * kAlign;
        r_hi = r_hi < nr ? r_hi : nr;
      }
      // the tile walk, specialised for the two dealings (index arithmetic on
      // the loader's critical path: c5 at 1% is loader-bound)
      // dynamic tail (sparse masks, tiles dealt grid-stride): the first
      // kStaticRounds rounds of G tiles are dealt grid-stride, the rest are
      // claimed one by one from a global counter (P.tile_ctr) by whichever
      // loader is free, so the CTAs finish together.  Lane 0 keeps claims in
      // flight (issued two tiles ahead of their use), so the atomic's latency
      // stays off the loader's path (two claims in flight); claims land in
      // s_claim (one per ring slot), -1 once the pool is empty.
      const int n_static = P.tile_ctr != nullptr && !range_mode
                               ? (int)((int64_t)n_tiles * (8 - P.dyn_eighths) / 8) / G * G
                               : n_tiles;
      const int n_dyn = n_tiles - n_static;
      __shared__ int s_claim[kStreamMask ? kMaskRing : 1];
      auto scan_tiles = [&](auto deal_tag) {
        constexpr int kDeal = decltype(deal_tag)::value;  // 0 grid-stride, 1 slices, 2 + dynamic tail
        constexpr bool kSlice = kDeal == 1;
        constexpr bool kDyn = kDeal == 2;
        const int my_static = kDyn ? n_static / G : 0;  // static tiles of this CTA (dynamic dealing)
        unsigned next_claim = 0, next_claim2 = 0;  // two claims in flight (lane 0)
        if constexpr (kDyn) {
          if (lane == 0) {
            next_claim = atomicAdd(P.tile_ctr, 1u);
            next_claim2 = atomicAdd(P.tile_ctr, 1u);
          }
        }
        auto tile_of = [&](int k2) -> int {  // dynamic dealing: tile number, -1 past the pool
          if (k2 < my_static) return (int)blockIdx.x + k2 * G;
          return s_claim[k2 % kMaskRing];
        };
        auto tile_start = [&](int k2) -> int64_t {
          if constexpr (kSlice) return r_lo + (int64_t)k2 * kRowsPerTile;
          else if constexpr (kDyn) return (int64_t)tile_of(k2) * kRowsPerTile;
          else return (int64_t)((int)blockIdx.x + k2 * G) * kRowsPerTile;
        };
        auto tile_end = [&](int64_t st) -> int64_t {
          return st + kRowsPerTile < r_hi ? st + kRowsPerTile : r_hi;
        };
        // bytes of the tile that arrive by bulk copy (16-byte multiple); rows
        // past them (the ragged end of the mask) are read from global memory
        auto bulk_bytes = [&](int64_t st) -> int {
          return (int)(((tile_end(st) - st) * kEsz) & ~(int64_t)15);
        };
        const int my_tiles =
            kDyn ? INT32_MAX
                 : kSlice ? (r_hi > r_lo ? (int)((r_hi - r_lo + kRowsPerTile - 1) / kRowsPerTile) : 0)
                          : ((int)blockIdx.x < n_tiles ? (n_tiles - 1 - (int)blockIdx.x) / G + 1 : 0);
        auto issue = [&](int k2) {  // tile number k2 of this CTA into slot k2 % kMaskRing
          if (k2 >= my_tiles) return;
          const int slot = k2 % kMaskRing;
          if constexpr (kDyn) {
            if (k2 >= my_static) {  // take the claim in flight, put the next one in flight
              int c = -1;
              if (lane == 0) {
                c = (int)next_claim < n_dyn ? n_static + (int)next_claim : -1;
                next_claim = next_claim2;
                if (c >= 0) next_claim2 = atomicAdd(P.tile_ctr, 1u);
                s_claim[slot] = c;
              }
              c = __shfl_sync(0xffffffffu, c, 0);
              if (c < 0) return;
            }
          }
          const int64_t st = tile_start(k2);
          const int b = bulk_bytes(st);
          if (lane == 0) {
            if (b > 0) {
              mbar_arrive_expect_tx(&mask_bar[slot], (uint32_t)b);
              bulk_g2s(s_mask[slot], gmask + st * kEsz, (uint32_t)b, &mask_bar[slot]);
            } else {
              mbar_arrive(&mask_bar[slot]);
            }
          }
        };
        // byte offset in the tile of the lane's 16-byte read q, and its first row
        // each lane owns contiguous rows (32 uint8 rows or 16 radii), so the
        // pending ids, and hence the chunks, stay in ascending row order within
        // a tile (index-coherent masks keep their DRAM locality)
        auto read_off = [&](int q) -> int {
          return MASK == 1 ? lane * kLane + 16 * q : (lane & (MTB / 64 - 1)) * 64 + 16 * q;
        };
        auto row_of_bit = [&](int k) -> int {  // bit k of the lane's mask -> row of the tile
          return MASK == 1 ? lane * kLane + k : (lane & (MTB / 64 - 1)) * 16 + k;
        };
        int head = 0, tail = 0;  // ring of pending ids: s_pend[head .. tail)
  #pragma unroll
        for (int k2 = 0; k2 < kMaskRing; ++k2) issue(k2);
        for (int k2 = 0; k2 < my_tiles; ++k2) {
          if constexpr (kDyn) {
            if (k2 >= my_static && s_claim[k2 % kMaskRing] < 0) break;  // the pool is empty
          }
          const int64_t st = tile_start(k2);
          const int slot = k2 % kMaskRing;
          GS_TRACE_WAIT(tr_mask, mbar_wait(&mask_bar[slot], (unsigned)((k2 / kMaskRing) & 1)));
          const int bb = bulk_bytes(st);
          const int64_t gend = tile_end(st) * kEsz;  // the tile's last mask byte + 1
          uint32_t bits = 0;
          if (MASK == 1 || lane < MTB / 64) {
  #pragma unroll
            for (int q = 0; q < kReads; ++q) {
              const int off = read_off(q);
              uint4 v;
              if (off + 16 <= bb) {
                v = *reinterpret_cast<const uint4*>(s_mask[slot] + off);
              } else {  // ragged end: global element reads (zero past the rows)
                uint32_t w[4] = {0u, 0u, 0u, 0u};
                const int64_t g0 = st * kEsz + off;
  #pragma unroll
                for (int by = 0; by < 16; ++by) {
                  const int64_t gb = g0 + by;
                  if (gb < gend) w[by >> 2] |= (uint32_t)gmask[gb] << (8 * (by & 3));
                }
                v = make_uint4(w[0], w[1], w[2], w[3]);
              }
              if constexpr (MASK == 1) {
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  #pragma unroll
                for (int j = 0; j < 4; ++j)
  #pragma unroll
                  for (int e = 0; e < 4; ++e)
                    bits |= (((w[j] >> (8 * e)) & 0xffu) != 0u) << (16 * q + 4 * j + e);
              } else {
                bits |= (uint32_t)((int)v.x > 0) << (4 * q) | (uint32_t)((int)v.y > 0) << (4 * q + 1) |
                        (uint32_t)((int)v.z > 0) << (4 * q + 2) | (uint32_t)((int)v.w > 0) << (4 * q + 3);
              }
            }
          }
          const int cnt = __popc(bits);
          int incl = cnt;
  #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int total = __shfl_sync(0xffffffffu, incl, 31);
          int pos = tail + incl - cnt;
          const int row0 = (int)st;
          for (uint32_t x = bits; x; x &= x - 1)
            s_pend[(pos++) & (kPend - 1)] = row0 + row_of_bit(__ffs(x) - 1);
          tail += total;
          __syncwarp();  // ids written; every lane is done with the slot
          issue(k2 + kMaskRing);
          while (tail - head >= R) {
            emit((int)s_pend[(head + lane) & (kPend - 1)], R);
            head += R;
          }
        }
        if (tail > head) emit(lane < tail - head ? (int)s_pend[(head + lane) & (kPend - 1)] : oob,
                              tail - head);
      };
      if (range_mode) scan_tiles(std::integral_constant<int, 1>{});
      else if (n_dyn > 0) scan_tiles(std::integral_constant<int, 2>{});
      else scan_tiles(std::integral_constant<int, 0>{});
    }
    emit(oob, -1);
    if (lane == 0) GS_STAMP(trc, 2);
#ifdef GS_TRACE
    if (lane == 0 && !kTwoPhase) {
      GS_TRACE_VAL(trc, 12, (unsigned long long)(clock64() - tr_t0));
      GS_TRACE_VAL(trc, 14, (unsigned long long)tr_empty);
      GS_TRACE_VAL(trc, 15, (unsigned long long)tr_mask);
    }
#endif
#undef GS_TRACE_WAIT
  } else if (BW && warp == NCW + 2) {
    // ------------------------------------------------------------ bias warp
    int st = 0;
    unsigned ph = 0;
    for (;;) {
      mbar_wait(&data_bar[st], ph);
      const int nv = s_nv[st];
      if (lane < nv) {
        const float2* srec = reinterpret_cast<const float2*>(stage(st));
        const int tb = kDense ? P.global_t
                              : reinterpret_cast<const int*>(srec + lane * SLOTS + L::P)[0] + 1;
        s_bc[st][lane] = __ldg(reinterpret_cast<const float2*>(P.lut) + (tb < P.lut_len ? tb : P.lut_len - 1));
      }
      mbar_arrive(&full_bar[st]);
      if (nv < 0) break;
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    }
  } else if (warp == NCW + 1) {
    // ------------------------------------------------------------------ storer
    int st = 0;
    unsigned ph = 0;
    for (;;) {
      mbar_wait(&done_bar[st], ph);
      const int nv = s_nv[st];
      if (nv < 0) break;
      const int my_id = lane < nv ? (int)s_crow[st][lane] : oob;
      const unsigned char* sb = stage(st);
      const int q = (4 * lane) & 31;
      const int r0 = __shfl_sync(0xffffffffu, my_id, q);
      const int r1 = __shfl_sync(0xffffffffu, my_id, q + 1);
      const int r2 = __shfl_sync(0xffffffffu, my_id, q + 2);
      const int r3 = __shfl_sync(0xffffffffu, my_id, q + 3);
      if (lane < R / 4 && 4 * lane < nv) {
        tma_scatter4(&M.rec, sb + lane * 4 * ST::kRecRow, r0, r1, r2, r3);
        tma_scatter4(&M.prm, sb + ST::kRec + lane * 4 * PT * 4, r0, r1, r2, r3);
        bulk_commit();
        bulk_wait_read0();  // the stage may be refilled once the stores have read it
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[st]);
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    }
    // every bulk store has read its stage (per-chunk wait above); the writes
    // themselves complete with the kernel, so the CTA does not wait for them
    if (lane == 0) GS_STAMP(trc, 5);
  } else {
    // ---------------------------------------------------------------- consumers
    const int t = tid;
    StepConsts Kc = P.K;
    if (kCoupled) {
      // the coupled normaliser N_v: given (sharded: the global count), or
      // the two-phase total of this mask
      const float nv = P.nv_dev ? (float)(*P.nv_dev)
                                : kTwoPhase ? (float)s_pref[G] : (float)P.nv_host;
      Kc.inv_nv = nv != 0.0f ? __frcp_rn(nv) : 0.0f;
      if (nv == 0.0f) Kc.lam_op = Kc.lam_sc = 0.0f;
    }
    const StepConsts& K = kCoupled ? Kc : P.K;
    int st = 0;
    int ep = 1;  // this use of stage st (epoch tag of its row flags)
    for (;;) {
      // BW: start on the landed gathers (data barrier); the bias factors
      // (full barrier, the bias warp) are awaited only after the check pass
      mbar_wait(BW ? &data_bar[st] : &full_bar[st], (unsigned)((ep - 1) & 1));
      const int nvalid = s_nv[st];
      if (tid == 0 && ep == 1 && st == 0) GS_STAMP(trc, 3);
      if (nvalid < 0) {
        mbar_arrive(&done_bar[st]);  // the storer reads the end marker too
        if (tid == 0) GS_STAMP(trc, 4);
        break;
      }
      unsigned char* sb = stage(st);
      float2* srec = reinterpret_cast<float2*>(sb);
      float* sth = reinterpret_cast<float*>(sb + ST::kRec);
      const float* sg = sth + R * PT;
      const uint32_t* srow = s_crow[st];
      const int tn = t < nvalid ? reinterpret_cast<const int*>(srec + t * SLOTS + L::P)[0] + 1 : 0;
      if (!STRICT) {
        // gradients in 16-byte pieces (columns >= P are pad and ignored);
        // activation domain on the opacity / scale columns of theta
        constexpr int kQ = (L::P + 3) / 4;
#pragma unroll
        for (int j = 0; j < (R * kQ + NC - 1) / NC; ++j) {
          const int p = j * NC + t;
          const int r = p / kQ;
          if (p < R * kQ && r < nvalid) {
            const int qq = p - r * kQ;
            const float4 v = reinterpret_cast<const float4*>(sg + r * PT)[qq];
            const bool bad = !isfinite(v.x) || (4 * qq + 1 < L::P && !isfinite(v.y)) ||
                             (4 * qq + 2 < L::P && !isfinite(v.z)) ||
                             (4 * qq + 3 < L::P && !isfinite(v.w));
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
              if (i < R * W && r < nvalid && domain_bad(role, sth[r * PT + L::OFF(gg) + (i - r * W)])) {
                atomicMax(&s_badd[st][r], ep);
                s_any[st] = ep;
              }
            }
          }
          dbase += R * W;
        }
      }
      if (BW) mbar_wait(&full_bar[st], (unsigned)((ep - 1) & 1));  // bias factors staged
      named_sync(1, NC);  // flags of the chunk are final; nobody has written the stage yet
      const bool any_bad = s_any[st] == ep || nvalid < R;
      auto row_ok = [&](int r) { return s_badg[st][r] != ep && s_badd[st][r] != ep; };
      // every thread reads the elements it updates before writing them, and
      // the element sets of different threads are disjoint, so in-place
      // updates need no further barrier
      auto update = [&](int gg, int i, int r) {
        const int W = L::W(gg);
        const int role = L::ROLE(gg);
        const int cc = i - r * W;
        const int e = r * PT + L::OFF(gg) + cc;
        float2* mvp = srec + r * SLOTS + L::OFF(gg) + cc;
        const float2 mv = *mvp;
        const float th = sth[e];
        float tnv, mn, vn, ex;
        bool clipped;
        update_element<MODE>(role, P.g[gg].lr, th, sg[e], mv.x, mv.y, s_bc[st][r], K, tnv, mn, vn,
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
        sth[e] = tnv;
        *mvp = make_float2(mn, vn);
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
      if (t < nvalid) {
        ++c_vis;
        if (row_ok(t)) {
          // the clock slot belongs to no element: thread t owns it
          reinterpret_cast<int*>(srec + t * SLOTS + L::P)[0] = tn;
          if (P.D.group >= 0) {
#pragma unroll
            for (int gg = 0; gg < L::G; ++gg)
              if (gg == P.D.group) densify_row(P.D, srow[t], sg + t * PT + L::OFF(gg), L::W(gg), 1);
          }
          ++c_step;
        } else if (s_badg[st][t] == ep) {
          ++c_badg;
        } else {
          ++c_badd;
        }
      }
      fence_proxy_async_smem();     // generic-proxy writes of the stage -> the bulk stores
      mbar_arrive(&done_bar[st]);
      if (++st == S) {
        st = 0;
        ++ep;
      }
    }
  }

  double acc[GS_STEP_STATS] = {(double)c_vis,  (double)c_step, (double)c_badg, (double)c_badd,
                               (double)c_apre, (double)c_apost, (double)c_clo, (double)c_cls,
                               s_exo,          s_exs,          (double)c_runs};
  const bool is_max[GS_STEP_STATS] = {false, false, false, false, false,
                                      false, false, false, false, false};
  block_reduce_n<GS_STEP_STATS, NWARPS>(acc, is_max, s_red);
  if (threadIdx.x == 0) {
    GS_STAMP(trc, 6);
    GS_TRACE_VAL(trc, 9, (unsigned long long)acc[0]);
#pragma unroll
    for (int f = 0; f < GS_STEP_STATS; ++f)
      P.partials[(size_t)blockIdx.x * GS_STEP_STATS + f] = acc[f];
  }
  if (last_block_arrive(P.counter)) {
    if (threadIdx.x == 0) GS_STAMP(trc, 7);
    if (threadIdx.x == 0 && P.tile_ctr != nullptr) *P.tile_ctr = 0u;  // every claim is done
    final_reduce_n<GS_STEP_STATS, NWARPS>(P.partials, gridDim.x, GS_STEP_STATS, P.stats_out,
                                             is_max, s_red);
    if (threadIdx.x == 0) GS_STAMP(trc, 8);
  }
#ifdef GS_TRACE
  if (threadIdx.x == 0 && trc) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    GS_TRACE_VAL(trc, 10, (unsigned long long)smid);
    GS_STAMP(trc, 11);
  }
#endif
}

// Largest grid of the two-phase kernel: one CTA count per thread of a CTA.
template <int NCW, bool BW>
constexpr int tma4_two_phase_max_grid() {
  return (NCW + 2 + (BW ? 1 : 0)) * 32;
}

// Host: tensor maps of the three records (cuTensorMapEncodeTiled through the
// runtime's driver entry point; no libcuda link dependency).
bool encode_tma_maps(const FixedParams& P, int64_t n_rows, int rec_box, TmaMaps* out);

template <class L, int MODE, bool STRICT, int S, int NCW, int MINB, int MASK = 0, bool BW = false,
          int MTB = 1024>
void launch_tma4(const FixedParams& P, const TmaMaps& M, int64_t max_rows, cudaStream_t s,
                 const void* vis_mask = nullptr) {
  constexpr int bytes = S * Tma4Stage<L, 32>::kBytes + 128;
  constexpr auto kern = step_tma4_kernel<L, MODE, STRICT, S, NCW, MINB, MASK, BW, MTB>;
  smem_opt_in<kern>(bytes);
  if constexpr (MASK >= 3) {
    // two-phase: one wave of CTAs (the grid barrier needs every CTA
    // resident), at least 256 mask rows each, launched cooperatively
    // resident CTAs of this kernel on the current device (cached per device)
    static std::atomic<int> resident_of[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int resident = dev < 64 ? resident_of[dev].load(std::memory_order_relaxed) : 0;
    if (resident <= 0) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NCW + 2 + (BW ? 1 : 0)) * 32,
                                                        bytes) != cudaSuccess)
        per_sm = 0;
      resident = per_sm * gs_sm_count();
      if (dev < 64 && resident > 0) resident_of[dev].store(resident, std::memory_order_relaxed);
    }
    if (resident <= 0) {
      gs_set_error("two-phase step kernel: no resident CTA (occupancy query failed)");
      gs_fail_launch();
      return;
    }
    const int64_t want = (max_rows + 255) / 256;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>({want, (int64_t)gs_sm_count() * MINB, (int64_t)resident,
                              (int64_t)tma4_two_phase_max_grid<NCW, BW>()}));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((NCW + 2 + (BW ? 1 : 0)) * 32);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P, M, vis_mask, trace_buf());
    if (e != cudaSuccess) {
      gs_set_error("two-phase step kernel (cooperative launch of %d CTAs): %s", grid,
                   cudaGetErrorString(e));
      gs_fail_launch();
    }
    return;
  }
  const int64_t tile = MASK == 1 ? MTB : MASK == 2 ? MTB / 4 : 32;
  int64_t work = (max_rows + tile - 1) / tile;
  // streamed masks under kBalancedChunksPerCta tiles per CTA slot: the
  // kernel gives every CTA a contiguous slice (>= 256 rows each)
  if ((MASK == 1 || MASK == 2) &&
      (P.mask_slices == 1 ||
       (P.mask_slices == 0 && work < (int64_t)kBalancedChunksPerCta * gs_sm_count() * MINB)))
    work = (max_rows + 255) / 256;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)gs_sm_count() * MINB));
  step_tma4_kernel<L, MODE, STRICT, S, NCW, MINB, MASK, BW, MTB>
      <<<grid, (NCW + 2 + (BW ? 1 : 0)) * 32, bytes, s>>>(P, M, vis_mask, trace_buf());
}

}  // namespace gs
