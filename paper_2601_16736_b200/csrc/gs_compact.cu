// K1 — visibility compaction (replaces np.flatnonzero(vis), optimizer.py:235,249).
//
// Single pass over the mask: each CTA owns a tile of kItems rows, counts its
// visible rows with a block scan, obtains its global offset with a
// warp-parallel decoupled look-back over epoch-tagged tile descriptors, and
// writes its ascending indices through shared memory so the global stores are
// coalesced.  The result is bit-identical to np.flatnonzero.
//
// Tile status word (64 bit):  [63:34] epoch (30 bit) | [33:32] flag | [31:0] value
//   flag 1 = tile aggregate published, flag 2 = inclusive prefix published.
// The epoch lives in the workspace header and is bumped by the last CTA of
// every launch, so no per-call memset is needed and CUDA-graph replays stay
// correct.
#include <stdio.h>

#include "gs_common.cuh"

namespace gs {

constexpr int kCompactItems = 16;                              // rows per thread
constexpr int kCompactTile = kThreads * kCompactItems;         // 4096 rows per CTA
constexpr uint64_t kFlagAgg = 1ull, kFlagPre = 2ull;
constexpr int kLookPerLane = 8;  // look-back window 32*8 tiles

struct CompactHeader {
  unsigned int epoch;
  unsigned int done;
  unsigned int pad[14];  // 64-byte header
};

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

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

template <typename T>
__global__ void __launch_bounds__(kThreads)
    compact_kernel(const T* __restrict__ mask, int64_t n, int32_t* __restrict__ idx_out,
                   int32_t* __restrict__ count_out, CompactHeader* hdr,
                   uint64_t* __restrict__ status, bool vec_ok) {
  __shared__ int32_t s_out[kCompactTile];
  __shared__ int s_warp[kThreads / 32];
  __shared__ uint32_t s_excl, s_total;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t tile_row0 = tile * kCompactTile;
  const uint32_t epoch = ((*(volatile unsigned int*)&hdr->epoch) + 1u) & 0x3fffffffu;
  const uint32_t ep = epoch == 0 ? 1u : epoch;

  const int64_t row0 = tile_row0 + (int64_t)tid * kCompactItems;
  const uint32_t bits = load_bits<T>(mask, row0, n, vec_ok);
  const int cnt = __popc(bits);

  // block exclusive scan of cnt
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kThreads / 32 ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kThreads / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == kThreads / 32 - 1) s_total = (uint32_t)wi;  // tile total
  }
  __syncthreads();
  const int local_off = s_warp[warp] + incl - cnt;
  const uint32_t total = s_total;

  // stage this thread's indices in shared memory (ascending)
  {
    uint32_t b = bits;
    int o = local_off;
    while (b) {
      int j = __ffs(b) - 1;
      b &= b - 1;
      s_out[o++] = (int32_t)(row0 + j);
    }
  }

  // decoupled look-back for the tile's global offset
  if (warp == 0) {
    const uint64_t tag = (uint64_t)ep << 34;
    if (tile == 0) {
      if (lane == 0) st_status(&status[0], tag | (kFlagPre << 32) | total);
      if (lane == 0) s_excl = 0;
    } else {
      if (lane == 0) st_status(&status[tile], tag | (kFlagAgg << 32) | total);
      // warp-wide look-back, kLookback predecessors per round (8 per lane,
      // lane 0 nearest): one L2 round trip covers 256 tiles, so the chain of
      // dependent rounds is ~tile/256 instead of ~tile/32
      uint32_t excl = 0;
      int64_t end = tile - 1;
      while (true) {
        uint32_t sum_all = 0, sum_upto = 0;
        int first_pre = kLookPerLane;
#pragma unroll
        for (int k = 0; k < kLookPerLane; ++k) {
          const int64_t j = end - (int64_t)lane * kLookPerLane - k;
          uint64_t sv;
          if (j < 0) {
            sv = kFlagPre << 32;  // virtual inclusive prefix 0 before tile 0
          } else {
            do {
              sv = ld_status(&status[j]);
            } while (!(((sv >> 34) == ep) && (((sv >> 32) & 3ull) != 0ull)));
          }
          const uint32_t val = (uint32_t)(sv & 0xffffffffull);
          const bool pre = ((sv >> 32) & 3ull) == kFlagPre;
          sum_all += val;
          if (first_pre == kLookPerLane) {
            sum_upto += val;
            if (pre) first_pre = k;
          }
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, first_pre < kLookPerLane);
        uint32_t contrib;
        if (pmask) {
          const int fl = __ffs(pmask) - 1;
          contrib = lane < fl ? sum_all : (lane == fl ? sum_upto : 0u);
        } else {
          contrib = sum_all;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        excl += contrib;
        if (pmask) break;
        end -= 32 * kLookPerLane;
      }
      if (lane == 0) {
        st_status(&status[tile], tag | (kFlagPre << 32) | (excl + total));
        s_excl = excl;
      }
    }
  }
  __syncthreads();
  const uint32_t excl = s_excl;
  for (uint32_t i = tid; i < total; i += kThreads) idx_out[excl + i] = s_out[i];
  if (tile == gridDim.x - 1 && tid == 0) *count_out = (int32_t)(excl + total);

  // last CTA out bumps the epoch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    unsigned int prev = atomicInc(&hdr->done, gridDim.x - 1);
    if (prev == gridDim.x - 1) hdr->epoch = ep;
  }
}

template <typename T>
int compact_launch(const T* mask, int64_t n, int32_t* idx_out, int32_t* count_out, void* ws,
                   size_t ws_bytes, void* stream) {
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
  auto* hdr = reinterpret_cast<CompactHeader*>(ws);
  auto* status = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(ws) + sizeof(CompactHeader));
  const bool vec_ok = (reinterpret_cast<uintptr_t>(mask) & 15u) == 0;
  compact_kernel<T><<<(unsigned)tiles, kThreads, 0, s>>>(mask, n, idx_out, count_out, hdr,
                                                         status, vec_ok);
  return gs_check_launch("gs_compact");
}

}  // namespace gs

extern "C" size_t gs_compact_workspace_bytes(int64_t n) {
  int64_t tiles = (n + gs::kCompactTile - 1) / gs::kCompactTile;
  if (tiles < 1) tiles = 1;
  return sizeof(gs::CompactHeader) + (size_t)tiles * sizeof(uint64_t);
}

extern "C" int gs_compact_u8(const uint8_t* mask, int64_t n, int32_t* idx_out,
                             int32_t* count_out, void* ws, size_t ws_bytes, void* stream) {
  return gs::compact_launch<uint8_t>(mask, n, idx_out, count_out, ws, ws_bytes, stream);
}

extern "C" int gs_compact_i32(const int32_t* radii, int64_t n, int32_t* idx_out,
                              int32_t* count_out, void* ws, size_t ws_bytes, void* stream) {
  return gs::compact_launch<int32_t>(radii, n, idx_out, count_out, ws, ws_bytes, stream);
}
