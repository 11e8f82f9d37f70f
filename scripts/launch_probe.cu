// Per-launch cost floor on B200: back-to-back launches of near-empty kernels
// shaped like K2 (296 CTAs x 320 threads, 95 KB dynamic shared memory each),
// captured in one CUDA graph and timed with events.  Separates the launch /
// drain cost from the kernel's dependent-latency chain (tail reduction,
// dependent global loads) and measures what programmatic dependent launch
// (PDL) recovers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe scripts/launch_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ unsigned int g_counter;
__device__ unsigned int g_counters[64 * 32];  // one 128-byte line per group counter
__device__ double g_partials[4096];
__device__ double g_out;

template <int MODE>
__global__ void __launch_bounds__(320, 2) probe(const int* __restrict__ chain, int depth, int pdl) {
  extern __shared__ unsigned char smem[];
  if (pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  double acc = threadIdx.x;
  if (MODE >= 1) {  // dependent global loads (a pointer chase of `depth` hops)
    if (threadIdx.x == 0) {
      int i = blockIdx.x;
      for (int d = 0; d < depth; ++d) i = __ldcg(chain + i);
      acc += i;
    }
  }
  if (MODE == 3 || MODE == 4) {  // acq_rel atomic, no fences; 11 doubles field-major
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x < 11) g_partials[threadIdx.x * 512 + blockIdx.x] = acc + threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev;
      if (MODE == 3) {
        __threadfence();
        prev = atomicInc(&g_counter, gridDim.x - 1);
      } else {
        asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(prev)
                     : "l"(&g_counter), "r"(gridDim.x - 1) : "memory");
      }
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      if (MODE == 3) __threadfence();
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      if (w < 11) {  // warp w reduces field w
        double s = 0;
        for (int b = l; b < gridDim.x; b += 32) s += __ldcg(g_partials + w * 512 + b);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (l == 0) (&g_out)[0] = s;
      }
    }
  }
  if (MODE == 5) {  // the bare atomic (no partials, no fence)
    if (threadIdx.x == 0) {
      unsigned prev = atomicInc(&g_counter, gridDim.x - 1);
      if (prev == 12345678) g_out = 1;
    }
  }
  if (MODE == 6) {  // two levels: groups of 16 CTAs, then the group leaders
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x < 11) g_partials[threadIdx.x * 512 + blockIdx.x] = acc + threadIdx.x;
    __syncthreads();
    const int grp = blockIdx.x >> 4, ng = (gridDim.x + 15) >> 4;
    const int gsz = min(16, (int)gridDim.x - grp * 16);
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(prev)
                   : "l"(&g_counters[grp * 32]), "r"(gsz - 1) : "memory");
      s_last = prev == gsz - 1;
    }
    __syncthreads();
    if (s_last) {
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      if (w < 11) {  // warp w: field w of the group
        double v = l < gsz ? __ldcg(g_partials + w * 512 + grp * 16 + l) : 0.0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) g_partials[w * 512 + 4096 / 8 * 0 + 300 + grp] = v;  // group partial
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(prev)
                     : "l"(&g_counters[63 * 32]), "r"(ng - 1) : "memory");
        s_last = prev == ng - 1;
      }
      __syncthreads();
      if (s_last && w < 11) {
        double v = l < ng ? __ldcg(g_partials + w * 512 + 300 + l) : 0.0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) (&g_out)[0] = v;
      }
    }
  }
  if (MODE == 2) {  // last-block-done reduction of one double per CTA
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      g_partials[blockIdx.x] = acc;
      __threadfence();
      const unsigned prev = atomicInc(&g_counter, gridDim.x - 1);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      double s = 0;
      for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(g_partials + b);
      if (threadIdx.x == 0) g_out = s;
    }
  }
  if (pdl) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (acc < 0) smem[0] = (unsigned char)acc;  // never taken (keeps acc live); smem may be 0 B
}

template <int MODE>
static float run(int grid, int smem, int depth, bool pdl, int* chain) {
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  const int reps = 200;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < reps; ++i)
    CK(cudaLaunchKernelEx(&cfg, probe<MODE>, (const int*)chain, depth, (int)pdl));
  CK(cudaStreamEndCapture(s, &g));
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
    printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return -1;
  }
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return best * 1000.f / reps;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int n_sm;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const int n = 1 << 24;
  int* chain;
  CK(cudaMalloc(&chain, n * sizeof(int)));
  {  // a random permutation cycle far apart (L2-missing hops)
    int* h = new int[n];
    for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 2654435761LL + 99991) % n);
    cudaMemcpy(chain, h, n * sizeof(int), cudaMemcpyHostToDevice);
    delete[] h;
  }
  printf("SMs %d\n", n_sm);
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("-- pdl %d (us per launch, graph of 200)\n", pdl);
    printf("empty     grid %4d smem 0      : %6.2f\n", 2 * n_sm, run<0>(2 * n_sm, 0, 0, pdl, chain));
    printf("empty     grid %4d smem 95360  : %6.2f\n", 2 * n_sm, run<0>(2 * n_sm, 95360, 0, pdl, chain));
    printf("empty     grid %4d smem 95360  : %6.2f\n", n_sm, run<0>(n_sm, 95360, 0, pdl, chain));
    printf("reduce    grid %4d smem 95360  : %6.2f\n", 2 * n_sm, run<2>(2 * n_sm, 95360, 0, pdl, chain));
    for (int d : {1, 2, 4, 8})
      printf("chain %d   grid %4d smem 95360  : %6.2f\n", d, 2 * n_sm, run<1>(2 * n_sm, 95360, d, pdl, chain));
    printf("chain4+red grid %4d smem 95360 : %6.2f\n", 2 * n_sm, run<2>(2 * n_sm, 95360, 4, pdl, chain));
    printf("red fm+fence grid %4d          : %6.2f\n", 2 * n_sm, run<3>(2 * n_sm, 95360, 0, pdl, chain));
    printf("red fm acq_rel grid %4d        : %6.2f\n", 2 * n_sm, run<4>(2 * n_sm, 95360, 0, pdl, chain));
    printf("bare atomic grid %4d           : %6.2f\n", 2 * n_sm, run<5>(2 * n_sm, 95360, 0, pdl, chain));
    printf("two-level 16 grid %4d          : %6.2f\n", 2 * n_sm, run<6>(2 * n_sm, 95360, 0, pdl, chain));
  }
  return 0;
}
