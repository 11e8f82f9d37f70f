// K1 — visibility compaction (replaces np.flatnonzero(vis), optimizer.py:235,249).
//
// Reduce-then-scan over tiles of 4096 rows (16 per thread):
//   count   each CTA popcounts its tile and writes one int (no inter-CTA
//           waiting at all);
//   write   each CTA sums the counts of all preceding tiles with a block-wide
//           reduction (<= a few thousand L2-resident ints), re-reads its mask
//           tile (L2-resident after the count pass), block-scans, stages its
//           ascending indices in shared memory and writes them coalesced.
// The result is bit-identical to np.flatnonzero.  A decoupled look-back
// single pass was measured first: with ~1200 co-resident tiles its prefix
// chain advanced one look-back window per L2 round trip and the CTAs spent
// their time at the barrier (~40 us at 6M rows), while the two passes here
// have no dependency chain.  Workspace: one int per tile, fully overwritten
// by every call (graph-safe, no memset).
#include <stdio.h>

#include "gs_common.cuh"

namespace gs {

constexpr int kCompactItems = 16;                              // rows per thread
constexpr int kCompactTile = kThreads * kCompactItems;         // 4096 rows per CTA

template <typename T>
__device__ __forceinline__ bool is_visible(T x);
template <>
__device__ __forceinline__ bool is_visible<uint8_t>(uint8_t x) { return x != 0; }
template <>
__device__ __forceinline__ bool is_visible<int32_t>(int32_t x) { return x > 0; }

// Load the thread's kCompactItems mask entries as a bitmask (bit j = row j visible).
template <typename T>
__device__ __forceinline__ uint32_t load_bits(const T* __restrict__ mask, int64_t row0,
                                              int64_t n, bool vec_ok);

template <>
__device__ __forceinline__ uint32_t load_bits<uint8_t>(const uint8_t* __restrict__ mask,
                                                       int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = 0;
  if (vec_ok && row0 + kCompactItems <= n) {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(mask + row0));
    uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) bits |= (((w[k] >> (8 * b)) & 0xffu) != 0u) << (4 * k + b);
  } else {
#pragma unroll
    for (int j = 0; j < kCompactItems; ++j)
      if (row0 + j < n) bits |= (uint32_t)(mask[row0 + j] != 0) << j;
  }
  return bits;
}

template <>
__device__ __forceinline__ uint32_t load_bits<int32_t>(const int32_t* __restrict__ mask,
                                                       int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = 0;
  if (vec_ok && row0 + kCompactItems <= n) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int4 q = __ldg(reinterpret_cast<const int4*>(mask + row0) + k);
      bits |= (uint32_t)(q.x > 0) << (4 * k) | (uint32_t)(q.y > 0) << (4 * k + 1) |
              (uint32_t)(q.z > 0) << (4 * k + 2) | (uint32_t)(q.w > 0) << (4 * k + 3);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kCompactItems; ++j)
      if (row0 + j < n) bits |= (uint32_t)(mask[row0 + j] > 0) << j;
  }
  return bits;
}

// Selection bits of the thread's rows: the mask bits, or their complement
// (invisible rows), restricted to alive rows when an alive mask is given.
template <typename T>
__device__ __forceinline__ uint32_t select_bits(const T* __restrict__ mask,
                                                const uint8_t* __restrict__ alive, bool invert,
                                                int64_t row0, int64_t n, bool vec_ok) {
  uint32_t bits = load_bits<T>(mask, row0, n, vec_ok);
  if (invert || alive) {
    const int64_t left = n - row0;
    const uint32_t in_range =
        left >= kCompactItems ? 0xffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
    if (invert) bits = ~bits & in_range;
    if (alive) bits &= load_bits<uint8_t>(alive, row0, n, vec_ok);
  }
  return bits;
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

template <typename T>
__global__ void __launch_bounds__(kThreads)
    compact_count_kernel(const T* __restrict__ mask, const uint8_t* __restrict__ alive,
                         bool invert, int64_t n, int32_t* __restrict__ counts, bool vec_ok) {
  __shared__ int s_sum[kThreads / 32];
  const int64_t row0 = (int64_t)blockIdx.x * kCompactTile + (int64_t)threadIdx.x * kCompactItems;
  int c = __popc(select_bits<T>(mask, alive, invert, row0, n, vec_ok));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += s_sum[w];
    counts[blockIdx.x] = t;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    compact_write_kernel(const T* __restrict__ mask, const uint8_t* __restrict__ alive,
                         bool invert, int64_t n,
                         const int32_t* __restrict__ counts, int32_t* __restrict__ idx_out,
                         int32_t* __restrict__ count_out, bool vec_ok) {
  __shared__ int32_t s_out[kCompactTile];
  __shared__ int s_warp[kThreads / 32];
  __shared__ int s_total;
  __shared__ long long s_red[kThreads / 32];
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  // global offset: sum of the counts of all preceding tiles
  long long pre = 0;
  for (int64_t j = tid; j < tile; j += kThreads) pre += __ldg(counts + j);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if ((tid & 31) == 0) s_red[tid >> 5] = pre;
  const int64_t row0 = tile * kCompactTile + (int64_t)tid * kCompactItems;
  const uint32_t bits = select_bits<T>(mask, alive, invert, row0, n, vec_ok);
  const int local_off = block_exclusive_scan(__popc(bits), s_warp, &s_total);
  long long excl = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) excl += s_red[w];
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
  if (tile == gridDim.x - 1 && tid == 0) *count_out = (int32_t)(excl + total);
}

template <typename T>
int compact_launch(const T* mask, int64_t n, int32_t* idx_out, int32_t* count_out, void* ws,
                   size_t ws_bytes, void* stream, const uint8_t* alive = nullptr,
                   bool invert = false) {
  if (n < 0 || (n > 0 && (!mask || !idx_out)) || !count_out || n >= (int64_t)INT32_MAX) {
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
  const bool vec_ok = (reinterpret_cast<uintptr_t>(mask) & 15u) == 0 &&
                      (reinterpret_cast<uintptr_t>(alive) & 15u) == 0;
  compact_count_kernel<T><<<(unsigned)tiles, kThreads, 0, s>>>(mask, alive, invert, n, counts,
                                                               vec_ok);
  compact_write_kernel<T><<<(unsigned)tiles, kThreads, 0, s>>>(mask, alive, invert, n, counts,
                                                               idx_out, count_out, vec_ok);
  return gs_check_launch("gs_compact");
}

}  // namespace gs

extern "C" size_t gs_compact_workspace_bytes(int64_t n) {
  int64_t tiles = (n + gs::kCompactTile - 1) / gs::kCompactTile;
  if (tiles < 1) tiles = 1;
  return (size_t)tiles * sizeof(int32_t);
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
