// Bandwidth probe: what does B200 HBM deliver for the AdamW-GS access
// pattern with no arithmetic in the way?
//
//   copy      streaming read+write of the same byte count (reference)
//   touch     per visible row: read theta+grad of the 6 SH-3 groups (SoA)
//             and the 480-byte state record, write theta and the record back
//             (the K2 traffic, trivial math), element-flattened, batches of 8
//   reads     the same gathers, no writes
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
// ./bw_probe [N=6000000] [p=0.3] [coherent=0]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int G = 6;
__constant__ int cW[G] = {3, 3, 45, 1, 3, 4};
__constant__ int cOFF[G] = {0, 3, 6, 51, 52, 55};

struct Arrays {
  float* p[G];
  const float* g[G];
  float* rec;  // [N, 120]
};

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// element e of the visible-row stream of group GI: row idx[e / W], col e % W
// (compile-time W, 32-bit index math; 8 independent elements per batch)
template <bool WRITE, int W, int OFF>
__device__ __forceinline__ void touch_group(float* __restrict__ P, const float* __restrict__ Gr,
                                            float* __restrict__ rec, const int* __restrict__ idx,
                                            int nv) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nth = gridDim.x * blockDim.x;
  const unsigned total = (unsigned)nv * W;
  for (unsigned base = tid; base < total; base += nth * 8) {
    float th[8], gr[8];
    float2 mv[8];
    unsigned off[8];
    float2* rp[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned e = base + b * nth;
      if (e < total) {
        const unsigned r = e / W;
        const unsigned c = e - r * W;
        const unsigned row = (unsigned)__ldg(idx + r);
        off[b] = row * W + c;
        rp[b] = reinterpret_cast<float2*>(rec + (size_t)row * 120) + OFF + c;
        th[b] = P[off[b]];
        gr[b] = __ldg(Gr + off[b]);
        mv[b] = *rp[b];
      }
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned e = base + b * nth;
      if (e < total) {
        const float x = th[b] + 1e-30f * gr[b] + 1e-30f * mv[b].x;
        if (WRITE) {
          P[off[b]] = x;
          *rp[b] = make_float2(mv[b].x + 1e-30f, mv[b].y);
        } else if (x == 12345.0f) {
          P[off[b]] = 0.f;
        }
      }
    }
  }
}

template <bool WRITE>
__global__ void __launch_bounds__(256) touch_kernel(Arrays A, const int* __restrict__ idx,
                                                    int nv) {
  touch_group<WRITE, 3, 0>(A.p[0], A.g[0], A.rec, idx, nv);
  touch_group<WRITE, 3, 3>(A.p[1], A.g[1], A.rec, idx, nv);
  touch_group<WRITE, 45, 6>(A.p[2], A.g[2], A.rec, idx, nv);
  touch_group<WRITE, 1, 51>(A.p[3], A.g[3], A.rec, idx, nv);
  touch_group<WRITE, 3, 52>(A.p[4], A.g[4], A.rec, idx, nv);
  touch_group<WRITE, 4, 55>(A.p[5], A.g[5], A.rec, idx, nv);
}

// pure streaming over the same arrays (all rows), for the p=1 reference
__global__ void stream_kernel(Arrays A, long n) {
  const long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long nth = (long)gridDim.x * blockDim.x;
  for (int g = 0; g < G; ++g) {
    const long tot = n * cW[g] / 4;
    float4* p = reinterpret_cast<float4*>(A.p[g]);
    const float4* q = reinterpret_cast<const float4*>(A.g[g]);
    for (long i = tid; i < tot; i += nth) {
      float4 a = p[i], b = q[i];
      a.x += 1e-30f * b.x;
      p[i] = a;
    }
  }
  const long tr = n * 30;
  float4* r = reinterpret_cast<float4*>(A.rec);
  for (long i = tid; i < tr; i += nth) {
    float4 a = r[i];
    a.x += 1e-30f;
    r[i] = a;
  }
}

int main(int argc, char** argv) {
  const long N = argc > 1 ? atol(argv[1]) : 6000000;
  const double p = argc > 2 ? atof(argv[2]) : 0.3;
  const int coherent = argc > 3 ? atoi(argv[3]) : 0;
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0, 1);
  std::vector<int> idx;
  if (coherent) {
    for (long b = 0; b < N; b += 64)
      if (U(rng) < p)
        for (long r = b; r < std::min(N, b + 64); ++r) idx.push_back((int)r);
  } else {
    for (long r = 0; r < N; ++r)
      if (U(rng) < p) idx.push_back((int)r);
  }
  const int nv = (int)idx.size();
  const int Wh[G] = {3, 3, 45, 1, 3, 4};
  Arrays A;
  for (int g = 0; g < G; ++g) {
    CK(cudaMalloc(&A.p[g], N * Wh[g] * 4));
    float* gg;
    CK(cudaMalloc(&gg, N * Wh[g] * 4));
    CK(cudaMemset(A.p[g], 0, N * Wh[g] * 4));
    CK(cudaMemset(gg, 0, N * Wh[g] * 4));
    A.g[g] = gg;
  }
  CK(cudaMalloc(&A.rec, N * 480));
  CK(cudaMemset(A.rec, 0, N * 480));
  int* didx;
  CK(cudaMalloc(&didx, nv * 4));
  CK(cudaMemcpy(didx, idx.data(), nv * 4, cudaMemcpyHostToDevice));
  const double alg = (double)nv * 1664;
  const size_t copy_bytes = (size_t)alg / 2 / 16 * 16;
  float4 *ca, *cb;
  CK(cudaMalloc(&ca, copy_bytes));
  CK(cudaMalloc(&cb, copy_bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, auto fn, double bytes) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0);
    const int K = 10;
    for (int i = 0; i < K; ++i) fn();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= K;
    printf("%-28s %8.3f ms  %8.1f GB/s (of %.3g bytes)\n", name, ms, bytes / ms / 1e6, bytes);
  };
  printf("N=%ld p=%.3f coherent=%d visible=%d\n", N, p, coherent, nv);
  timeit("copy (read+write)", [&] { copy_kernel<<<sms * 8, 256>>>(ca, cb, copy_bytes / 16); },
         2.0 * copy_bytes);
  for (int bpsm : {4, 8, 16}) {
    char name[64];
    snprintf(name, 64, "touch r+w (grid %dx)", bpsm);
    timeit(name, [&] { touch_kernel<true><<<sms * bpsm, 256>>>(A, didx, nv); }, alg);
    snprintf(name, 64, "gather reads (grid %dx)", bpsm);
    timeit(name, [&] { touch_kernel<false><<<sms * bpsm, 256>>>(A, didx, nv); },
           (double)nv * (16 * 59 + 4 + 4));
  }
  timeit("stream all rows r+w", [&] { stream_kernel<<<sms * 8, 256>>>(A, N); },
         (double)N * 1652);
  CK(cudaGetLastError());
  return 0;
}
