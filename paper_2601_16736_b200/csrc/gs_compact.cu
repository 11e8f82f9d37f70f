// K1 — visibility compaction (replaces np.flatnonzero(vis), optimizer.py:235,249).
//
// Reduce-then-scan over tiles of 8192 rows (32 per thread, two 16-byte
// mask loads in flight each):
//   count   each CTA popcounts its tile and writes one int; the last CTA to
//           finish scans the tile counts into exclusive offsets (no CTA ever
//           waits on another);
//   write   each CTA reads its offset and its tile's selection bitmap (the
//           count pass stores one bit per row; the mask is read once),
//           block-scans, stages its ascending indices in shared memory and
//           writes them coalesced.
// The result is bit-identical to np.flatnonzero.  A decoupled look-back
// single pass was measured first: with ~1200 co-resident tiles its prefix
// chain advanced one look-back window per L2 round trip and the CTAs spent
// their time at the barrier (~40 us at 6M rows), while the two passes here
// have no dependency chain.  (An earlier write pass summed all preceding tile
// counts per CTA: O(tiles^2), 58 us at 50M rows.)  Workspace: one int per
// tile and one bit per row, overwritten by every call, plus an arrival
// counter that must start at zero and is left at zero (graph-safe, no memset).
#include <stdio.h>

#include "gs_common.cuh"

namespace gs {

constexpr int kLoadItems = 16;                                  // rows per 16-byte mask load
constexpr int kCompactItems = 32;                               // rows per thread (2 loads)
constexpr int kCompactTile = kThreads * kCompactItems;          // 8192 rows per CTA

template <typename T>
__device__ __forceinline__ bool is_visible(T x);
template <>
__device__ __forceinline__ bool is_visible<uint8_t>(uint8_t x) { return x != 0; }
template <>
__device__ __forceinline__ bool is_visible<int32_t>(int32_t x) { return x > 0; }

// Load kLoadItems consecutive mask entries as a bitmask (bit j = row j visible).
template <typename T>
__device__ __forceinline__ uint32_t load_bits(const T* __restrict__ mask, int64_t row0,
                                              int64_t n, bool vec_ok);

template <>
__device__ __forceinline__ uint32_t load_bits<uint8_t>(const uint8_t* __restrict__ mask,
                                                       int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = 0;
  if (vec_ok && row0 + kLoadItems <= n) {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(mask + row0));
    uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) bits |= (((w[k] >> (8 * b)) & 0xffu) != 0u) << (4 * k + b);
  } else {
#pragma unroll
    for (int j = 0; j < kLoadItems; ++j)
      if (row0 + j < n) bits |= (uint32_t)(mask[row0 + j] != 0) << j;
  }
  return bits;
}

template <>
__device__ __forceinline__ uint32_t load_bits<int32_t>(const int32_t* __restrict__ mask,
                                                       int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = 0;
  if (vec_ok && row0 + kLoadItems <= n) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int4 q = __ldg(reinterpret_cast<const int4*>(mask + row0) + k);
      bits |= (uint32_t)(q.x > 0) << (4 * k) | (uint32_t)(q.y > 0) << (4 * k + 1) |
              (uint32_t)(q.z > 0) << (4 * k + 2) | (uint32_t)(q.w > 0) << (4 * k + 3);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kLoadItems; ++j)
      if (row0 + j < n) bits |= (uint32_t)(mask[row0 + j] > 0) << j;
  }
  return bits;
}

// Selection bits of the thread's rows: the mask bits, or their complement
// (invisible rows), restricted to alive rows when an alive mask is given.
template <typename T>
__device__ __forceinline__ uint32_t select_bits16(const T* __restrict__ mask,
                                                  const uint8_t* __restrict__ alive, bool invert,
                                                  int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = load_bits<T>(mask, row0, n, vec_ok);
  if (invert || alive) {
    const int64_t left = n - row0;
    const uint32_t in_range =
        left >= kLoadItems ? 0xffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
    if (invert) bits = ~bits & in_range;
    if (alive) bits &= load_bits<uint8_t>(alive, row0, n, vec_ok);
  }
  return bits;
}

// The thread's kCompactItems (32) rows: two 16-row loads, both in flight.
template <typename T>
__device__ __forceinline__ uint32_t select_bits(const T* __restrict__ mask,
                                                const uint8_t* __restrict__ alive, bool invert,
                                                int64_t row0, int64_t n, bool vec_ok) {
  const uint32_t lo = select_bits16<T>(mask, alive, invert, row0, n, vec_ok);
  const uint32_t hi = select_bits16<T>(mask, alive, invert, row0 + kLoadItems, n, vec_ok);
  return lo | (hi << 16);
}

__device__ __forceinline__ int block_exclusive_scan(int cnt, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < kThreads / 32 ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kThreads / 32) s_warp[lane] = wi - w;
    if (lane == kThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  return s_warp[warp] + incl - cnt;
}

// Pass 1: popcount of each tile (persistent CTAs, grid-stride over tiles),
// plus the selection bitmap.  The last CTA to finish (last_block_arrive, the
// counter wraps back to 0) turns the tile counts into exclusive offsets in
// place, 16 per thread per round, and writes the total.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    compact_count_kernel(const T* __restrict__ mask, const uint8_t* __restrict__ alive,
                         bool invert, int64_t n, int tiles, int32_t* __restrict__ counts,
                         unsigned int* __restrict__ counter, int32_t* __restrict__ count_out,
                         uint32_t* __restrict__ bitmap, bool vec_ok) {
  __shared__ int s_sum[2][kThreads / 32];
  __shared__ int s_total;
  int par = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, par ^= 1) {
    const int64_t row0 = (int64_t)tile * kCompactTile + (int64_t)threadIdx.x * kCompactItems;
    const uint32_t bits = select_bits<T>(mask, alive, invert, row0, n, vec_ok);
    bitmap[(int64_t)tile * kThreads + threadIdx.x] = bits;  // 1 bit per row for pass 2
    int c = __popc(bits);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s_sum[par][threadIdx.x >> 5] = c;
    __syncthreads();  // double-buffered partials: one barrier per tile
    if (threadIdx.x == 0) {
      int t = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) t += s_sum[par][w];
      counts[tile] = t;
    }
  }
  if (!last_block_arrive(counter)) return;
  int carry = 0;
  for (int base = 0; base < tiles; base += kThreads * 16) {
    const int i0 = base + (int)threadIdx.x * 16;
    int v[16];
    int sum = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = i0 + j < tiles ? __ldcg(counts + i0 + j) : 0;
      sum += v[j];
    }
    int run = carry + block_exclusive_scan(sum, s_sum[0], &s_total);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (i0 + j < tiles) counts[i0 + j] = run;
      run += v[j];
    }
    carry += s_total;
    __syncthreads();  // s_sum / s_total are reused by the next round
  }
  if (threadIdx.x == 0) *count_out = carry;
}

// Pass 2: each CTA reads its tile's selection bitmap (n/8 bytes in all,
// L2-resident; the mask itself is not read again), block-scans, stages its
// ascending indices in shared memory and writes them coalesced at the tile's
// offset.
__global__ void __launch_bounds__(kThreads)
    compact_write_kernel(const uint32_t* __restrict__ bitmap,
                         const int32_t* __restrict__ offsets, int32_t* __restrict__ idx_out) {
  __shared__ int32_t s_out[kCompactTile];
  __shared__ int s_warp[kThreads / 32];
  __shared__ int s_total;
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t excl = __ldg(offsets + tile);
  const int64_t row0 = tile * kCompactTile + (int64_t)tid * kCompactItems;
  const uint32_t bits = __ldg(bitmap + tile * kThreads + tid);
  const int local_off = block_exclusive_scan(__popc(bits), s_warp, &s_total);
  const int total = s_total;
  {
    uint32_t b = bits;
    int o = local_off;
    while (b) {
      const int j = __ffs(b) - 1;
      b &= b - 1;
      s_out[o++] = (int32_t)(row0 + j);
    }
  }
  __syncthreads();
  for (int i = tid; i < total; i += kThreads) idx_out[excl + i] = s_out[i];
}

template <typename T>
int compact_launch(const T* mask, int64_t n, int32_t* idx_out, int32_t* count_out, void* ws,
                   size_t ws_bytes, void* stream, const uint8_t* alive = nullptr,
                   bool invert = false, bool write_pass = true) {
  if (n < 0 || (n > 0 && (!mask || (write_pass && !idx_out))) || !count_out ||
      n >= (int64_t)INT32_MAX) {
    gs_set_error("gs_compact: invalid arguments (n=%lld)", (long long)n);
    return GS_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (cudaMemsetAsync(count_out, 0, sizeof(int32_t), s) != cudaSuccess)
      return gs_check_launch("gs_compact memset");
    return GS_OK;
  }
  if (ws_bytes < gs_compact_workspace_bytes(n) || !ws) {
    gs_set_error("gs_compact: workspace too small (%zu < %zu)", ws_bytes,
                 gs_compact_workspace_bytes(n));
    return GS_ERR_WORKSPACE;
  }
  const int64_t tiles = (n + kCompactTile - 1) / kCompactTile;
  auto* counts = reinterpret_cast<int32_t*>(ws);
  auto* counter = reinterpret_cast<unsigned int*>(counts + tiles);
  auto* bitmap = reinterpret_cast<uint32_t*>(counts + tiles + 1);
  const bool vec_ok = (reinterpret_cast<uintptr_t>(mask) & 15u) == 0 &&
                      (reinterpret_cast<uintptr_t>(alive) & 15u) == 0;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)gs_sm_count() * 8);
  compact_count_kernel<T><<<grid, kThreads, 0, s>>>(mask, alive, invert, n, (int)tiles, counts,
                                                    counter, count_out, bitmap, vec_ok);
  if (write_pass) compact_write_kernel<<<(unsigned)tiles, kThreads, 0, s>>>(bitmap, counts, idx_out);
  return gs_check_launch("gs_compact");
}

}  // namespace gs

extern "C" size_t gs_compact_workspace_bytes(int64_t n) {
  int64_t tiles = (n + gs::kCompactTile - 1) / gs::kCompactTile;
  if (tiles < 1) tiles = 1;
  // per-tile offsets + the arrival counter + one selection bit per row
  return (size_t)(tiles + 1 + tiles * gs::kThreads) * sizeof(int32_t);
}

extern "C" int gs_compact_u8(const uint8_t* mask, int64_t n, int32_t* idx_out,
                             int32_t* count_out, void* ws, size_t ws_bytes, void* stream) {
  return gs::compact_launch<uint8_t>(mask, n, idx_out, count_out, ws, ws_bytes, stream);
}

extern "C" int gs_compact_i32(const int32_t* radii, int64_t n, int32_t* idx_out,
                              int32_t* count_out, void* ws, size_t ws_bytes, void* stream) {
  return gs::compact_launch<int32_t>(radii, n, idx_out, count_out, ws, ws_bytes, stream);
}

extern "C" int gs_compact_select_u8(const uint8_t* mask, const uint8_t* alive, int32_t invert,
                                    int64_t n, int32_t* idx_out, int32_t* count_out, void* ws,
                                    size_t ws_bytes, void* stream) {
  return gs::compact_launch<uint8_t>(mask, n, idx_out, count_out, ws, ws_bytes, stream, alive,
                                     invert != 0);
}

extern "C" int gs_count_visible(const uint8_t* mask, const int32_t* radii, int64_t n,
                                int32_t* count_out, void* ws, size_t ws_bytes, void* stream) {
  if ((mask != nullptr) == (radii != nullptr)) {
    gs_set_error("gs_count_visible: exactly one of mask / radii");
    return GS_ERR_ARG;
  }
  if (radii)
    return gs::compact_launch<int32_t>(radii, n, nullptr, count_out, ws, ws_bytes, stream,
                                       nullptr, false, false);
  return gs::compact_launch<uint8_t>(mask, n, nullptr, count_out, ws, ws_bytes, stream, nullptr,
                                     false, false);
}
