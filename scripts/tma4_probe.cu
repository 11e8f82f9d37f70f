// Probe: can Blackwell's 2-D TMA row gathers (tile::gather4) and scatters
// (tile::scatter4) move the K2 traffic faster than 16-byte cp.async gathers?
//
// Per visible row (ascending index list, i.i.d. Bernoulli(p) or all rows):
// gather the 480-B moment record row (of a 512-B row), the 240-B parameter
// row and the 240-B gradient row (of 256-B rows) into a shared-memory ring,
// add 1 to every parameter and moment value in place, scatter the parameter
// row and the moment record row back.  Roles: warp 0 issues the gathers
// (lanes 0..7, 3 ops each per 32-row chunk), warp 1 issues the scatters,
// the remaining warps "update".  Validates the values afterwards.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma4 scripts/tma4_probe.cu
// /tmp/tma4 [N=6000000] [p=0.3] [box_rows=1] [stages=3] [ncw=8] [minb=2]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int R = 32;
constexpr int REC_W = 120;  // floats of the moment record moved per row
constexpr int ROW_W = 64;   // floats of the parameter / gradient row moved (4 rows = 1 KB: 128-B aligned boxes)
constexpr int REC_STRIDE = 128, ROW_STRIDE = 64;
constexpr int STAGE_BYTES = R * (REC_W + 2 * ROW_W) * 4;

__device__ __forceinline__ unsigned sm(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          sm(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                        int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sm(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sm(bar))
      : "memory");
}
__device__ __forceinline__ void scatter4(const CUtensorMap* map, const void* src, int col, int r0, int r1,
                                         int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group"
      " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map),
      "r"(sm(src)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

struct Maps {
  CUtensorMap rec, prm, grd;
};

template <int S, int NCW>
__global__ void __launch_bounds__((NCW + 2) * 32, 1) tma4_kernel(const __grid_constant__ Maps M,
                                                                 const int* __restrict__ rows, int n_vis,
                                                                 int n_rows) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S], done[S], empty[S];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NC = NCW * 32;
  const int n_chunks = (n_vis + R - 1) / R;
  const int G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], NC);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto stage = [&](int s) { return smem + s * STAGE_BYTES; };
  if (warp == 0) {  // loads
    int s = 0;
    unsigned ph = 0;
    for (int c = blockIdx.x, k = 0; c < n_chunks; c += G, ++k) {
      const int i = c * R + lane;
      const int id = i < n_vis ? __ldg(rows + i) : n_rows;  // past the end: OOB, zero-filled
      if (k >= S) mbar_wait(&empty[s], ph ^ 1u);
      unsigned char* sb = stage(s);
      if (lane == 0) mbar_expect(&full[s], STAGE_BYTES);
      __syncwarp();
      const int r0 = __shfl_sync(~0u, id, (4 * lane) & 31), r1 = __shfl_sync(~0u, id, (4 * lane + 1) & 31);
      const int r2 = __shfl_sync(~0u, id, (4 * lane + 2) & 31), r3 = __shfl_sync(~0u, id, (4 * lane + 3) & 31);
      if (lane < 8) {
        gather4(sb + lane * 4 * REC_W * 4, &M.rec, 0, r0, r1, r2, r3, &full[s]);
        gather4(sb + R * REC_W * 4 + lane * 4 * ROW_W * 4, &M.prm, 0, r0, r1, r2, r3, &full[s]);
        gather4(sb + R * (REC_W + ROW_W) * 4 + lane * 4 * ROW_W * 4, &M.grd, 0, r0, r1, r2, r3, &full[s]);
      }
      if (++s == S) s = 0, ph ^= 1u;
    }
  } else if (warp == 1) {  // stores
    int s = 0;
    unsigned ph = 0;
    for (int c = blockIdx.x; c < n_chunks; c += G) {
      const int i = c * R + lane;
      const int id = i < n_vis ? __ldg(rows + i) : n_rows;  // OOB rows are not written
      mbar_wait(&done[s], ph);
      unsigned char* sb = stage(s);
      const int r0 = __shfl_sync(~0u, id, (4 * lane) & 31), r1 = __shfl_sync(~0u, id, (4 * lane + 1) & 31);
      const int r2 = __shfl_sync(~0u, id, (4 * lane + 2) & 31), r3 = __shfl_sync(~0u, id, (4 * lane + 3) & 31);
      if (lane < 8) {
        scatter4(&M.rec, sb + lane * 4 * REC_W * 4, 0, r0, r1, r2, r3);
        scatter4(&M.prm, sb + R * REC_W * 4 + lane * 4 * ROW_W * 4, 0, r0, r1, r2, r3);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) s = 0, ph ^= 1u;
    }
    if (lane < 8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {  // "update": +1 on every parameter and moment value of the chunk
    const int t = tid - 64;
    int s = 0;
    unsigned ph = 0;
    for (int c = blockIdx.x; c < n_chunks; c += G) {
      mbar_wait(&full[s], ph);
      float* f = reinterpret_cast<float*>(stage(s));
      float* g = f + R * (REC_W + ROW_W);
      for (int e = t; e < R * ROW_W; e += NC) {
        const int r = e / ROW_W, col = e - r * ROW_W;
        float* th = f + R * REC_W + e;
        float2* mv = reinterpret_cast<float2*>(f) + r * (REC_W / 2) + col;
        const float gr = g[e];
        *th = *th + 1.0f + 0.0f * gr;
        if (col < REC_W / 2) {
          float2 x = *mv;
          x.x += 1.0f;
          x.y += 1.0f;
          *mv = x;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&done[s]);
      if (++s == S) s = 0, ph ^= 1u;
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(EncodeFn enc, CUtensorMap* m, float* base, int64_t n, int stride, int w, int box_rows,
                     CUtensorMapL2promotion l2) {
  cuuint64_t dim[2] = {(cuuint64_t)stride, (cuuint64_t)n};
  cuuint64_t str[1] = {(cuuint64_t)stride * 4};
  cuuint32_t box[2] = {(cuuint32_t)w, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed: %d (box %d x %d)\n", (int)r, w, box_rows);
    exit(1);
  }
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int S, int NCW>
float run(const Maps& M, const int* rows, int nv, int n, int grid) {
  const int smem = S * STAGE_BYTES;
  CK(cudaFuncSetAttribute(tma4_kernel<S, NCW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma4_kernel<S, NCW><<<grid, (NCW + 2) * 32, smem>>>(M, rows, nv, n);
  CK(cudaDeviceSynchronize());
  const int reps = 10;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) tma4_kernel<S, NCW><<<grid, (NCW + 2) * 32, smem>>>(M, rows, nv, n);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 6000000;
  const double p = argc > 2 ? atof(argv[2]) : 0.3;
  const int box_rows = argc > 3 ? atoi(argv[3]) : 1;
  const int l2p = argc > 4 ? atoi(argv[4]) : 3;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  std::vector<int> idx;
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0, 1);
  for (int64_t i = 0; i < n; ++i)
    if (p >= 1.0 || U(rng) < p) idx.push_back((int)i);
  const int nv = (int)idx.size();
  float *rec, *prm, *grd;
  int* rows;
  CK(cudaMalloc(&rec, n * REC_STRIDE * 4));
  CK(cudaMalloc(&prm, n * ROW_STRIDE * 4));
  CK(cudaMalloc(&grd, n * ROW_STRIDE * 4));
  CK(cudaMalloc(&rows, (size_t)nv * 4 + 4));
  CK(cudaMemset(rec, 0, n * REC_STRIDE * 4));
  CK(cudaMemset(prm, 0, n * ROW_STRIDE * 4));
  CK(cudaMemset(grd, 0, n * ROW_STRIDE * 4));
  CK(cudaMemcpy(rows, idx.data(), (size_t)nv * 4, cudaMemcpyHostToDevice));
  Maps M;
  const CUtensorMapL2promotion l2 = (CUtensorMapL2promotion)l2p;
  make_map(enc, &M.rec, rec, n, REC_STRIDE, REC_W, box_rows, l2);
  make_map(enc, &M.prm, prm, n, ROW_STRIDE, ROW_W, box_rows, l2);
  make_map(enc, &M.grd, grd, n, ROW_STRIDE, ROW_W, box_rows, l2);

  // correctness: one launch, every visible row +1 (pad columns untouched)
  CK(cudaFuncSetAttribute(tma4_kernel<3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * STAGE_BYTES));
  tma4_kernel<3, 8><<<sms * 2, 320, 3 * STAGE_BYTES>>>(M, rows, nv, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  {
    std::vector<float> h(n * ROW_STRIDE), hr(n * REC_STRIDE);
    CK(cudaMemcpy(h.data(), prm, h.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), rec, hr.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<char> vis(n, 0);
    for (int i : idx) vis[i] = 1;
    long bad = 0;
    for (int64_t r = 0; r < n; ++r) {
      for (int c = 0; c < ROW_STRIDE; ++c) {
        const float want = (vis[r] && c < ROW_W) ? 1.0f : 0.0f;
        bad += h[r * ROW_STRIDE + c] != want;
      }
      for (int c = 0; c < REC_STRIDE; ++c) {
        const float want = (vis[r] && c < REC_W) ? 1.0f : 0.0f;
        bad += hr[r * REC_STRIDE + c] != want;
      }
    }
    printf("validate: %ld bad values (n=%lld nv=%d box_rows=%d)\n", bad, (long long)n, nv, box_rows);
  }
  const double alg = (double)nv * 1664.0;  // the K2 algorithmic bytes per visible row
  const double moved = (double)nv * (480 + 240 + 240 + 480 + 240);
  auto report = [&](const char* name, float ms) {
    printf("%-28s %8.4f ms  alg %.0f GB/s (frac %.3f of 6550)  moved %.0f GB/s\n", name, ms, alg / ms / 1e6,
           alg / ms / 1e6 / 6550.0, moved / ms / 1e6);
  };
  report("S3 NCW8 grid 2/SM", run<3, 8>(M, rows, nv, (int)n, 2 * sms));
  report("S2 NCW8 grid 2/SM", run<2, 8>(M, rows, nv, (int)n, 2 * sms));
  report("S4 NCW8 grid 1/SM", run<4, 8>(M, rows, nv, (int)n, sms));
  report("S3 NCW4 grid 2/SM", run<3, 4>(M, rows, nv, (int)n, 2 * sms));
  report("S3 NCW4 grid 3/SM", run<3, 4>(M, rows, nv, (int)n, 3 * sms));
  report("S2 NCW4 grid 3/SM", run<2, 4>(M, rows, nv, (int)n, 3 * sms));
  report("S6 NCW8 grid 1/SM", run<6, 8>(M, rows, nv, (int)n, sms));
  // streaming copy of the same byte count, for reference
  {
    const size_t bytes = (size_t)(alg / 2) / 16 * 16;
    float4 *a, *b;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    copy_kernel<<<sms * 8, 512>>>(a, b, bytes / 16);
    cudaEvent_t x, y;
    cudaEventCreate(&x);
    cudaEventCreate(&y);
    cudaEventRecord(x);
    for (int i = 0; i < 10; ++i) copy_kernel<<<sms * 8, 512>>>(a, b, bytes / 16);
    cudaEventRecord(y);
    CK(cudaEventSynchronize(y));
    float ms;
    cudaEventElapsedTime(&ms, x, y);
    report("stream copy (same bytes)", ms / 10);
  }
  return 0;
}
