// Shared device helpers for the AdamW-GS kernels (sm_100a).
//
// Arithmetic contract: every fp32 operation of the step is an explicit
// round-to-nearest intrinsic (no FMA contraction) and every float64 term is
// evaluated with the reference's association, so that the CPU restatement in
// oracle/adamw_gs_oracle.py::step_fp32 reproduces the kernel bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "../../include/adamw_gs.h"

namespace gs {

constexpr int kThreads = 256;  // rows per chunk == threads per CTA

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

// Deterministic fp32 exp: Cody-Waite reduction x = n*ln2 + r, degree-7
// Taylor polynomial in Horner form, exact power-of-two scaling.  Every step is
// one correctly rounded fp32 operation, so oracle/adamw_gs_oracle.py::gs_expf
// reproduces it bit for bit (max error ~2 ulp).  Inputs below -86 return 0
// (the result would be subnormal; the penalty term is then negligible).
__device__ __forceinline__ float gs_expf(float x) {
  if (x < -86.0f) return 0.0f;
  const float n = rintf(__fmul_rn(x, 1.442695f));
  float r = __fsub_rn(x, __fmul_rn(n, 0.693145751953125f));
  r = __fsub_rn(r, __fmul_rn(n, 1.4286068e-06f));
  float p = 1.984127e-04f;                      // 1/5040
  p = __fadd_rn(__fmul_rn(p, r), 1.3888889e-03f);  // 1/720
  p = __fadd_rn(__fmul_rn(p, r), 8.333334e-03f);  // 1/120
  p = __fadd_rn(__fmul_rn(p, r), 4.1666668e-02f);  // 1/24
  p = __fadd_rn(__fmul_rn(p, r), 1.6666667e-01f);  // 1/6
  p = __fadd_rn(__fmul_rn(p, r), 0.5f);
  p = __fadd_rn(__fmul_rn(p, r), 1.0f);
  p = __fadd_rn(__fmul_rn(p, r), 1.0f);
  return __fmul_rn(p, __int_as_float(((int)n + 127) << 23));
}

// R'(theta) of the L1 penalty on the activated attribute (primitives.py:62-84):
// sigma'(tau) = e / (1 + e)^2 with e = exp(-|tau|) (both branches of the
// stable sigmoid give this form), and exp(kappa) for the scale.
__device__ __forceinline__ float reg_deriv(int role, float theta) {
  if (role == GS_ROLE_OPACITY) {
    const float e = gs_expf(-fabsf(theta));
    const float d = __fadd_rn(1.0f, e);
    return __fdiv_rn(e, __fmul_rn(d, d));
  }
  return gs_expf(theta);
}

// Step constants shared by the per-group and row-record kernels.
struct StepConsts {
  float a1, a2, eps;
  float lam_op, lam_sc;    // penalty lambdas (0 = none)
  float cap_op, cap_sc;    // C_t / clip
  float inv_ni, inv_nv;    // 1/N_I' (adamw-gs), 1/N_v (coupled)
};

// The per-element update, identical for every kernel and mirrored by
// oracle/adamw_gs_oracle.py::step_fp32.  MODE is a GS_MODE_*.  Returns the
// new theta / m / v; ex is the penalty term added to the step (0 if none).
template <int MODE>
__device__ __forceinline__ void update_element(int role, float lr, float th, float g, float mm,
                                               float vv, float2 bc, const StepConsts& K,
                                               float& th_out, float& m_out, float& v_out,
                                               float& ex, bool& clipped) {
  constexpr bool kCoupled = MODE == GS_MODE_COUPLED_ADAM || MODE == GS_MODE_SPARSE_ADAM;
  const float lam = role == GS_ROLE_OPACITY ? K.lam_op : role == GS_ROLE_SCALE ? K.lam_sc : 0.0f;
  ex = 0.0f;
  clipped = false;
  if (kCoupled && lam != 0.0f) {
    // loss.py:177-198 folded in: g += lambda * R'(theta) / N_v
    g = __fadd_rn(g, __fmul_rn(__fmul_rn(lam, reg_deriv(role, th)), K.inv_nv));
  }
  const float d = __fsub_rn(g, mm);
  const float mn = __fadd_rn(mm, __fmul_rn(K.a1, d));
  const float g2 = __fmul_rn(g, g);
  const float ee = __fsub_rn(g2, vv);
  const float vn = __fadd_rn(vv, __fmul_rn(K.a2, ee));
  const float mh = __fmul_rn(mn, bc.x);
  const float vh = __fmul_rn(vn, bc.y);
  const float den = __fadd_rn(__fsqrt_rn(vh), K.eps);
  float step = __fdiv_rn(mh, den);
  if (!kCoupled && lam != 0.0f) {
    const float deriv = reg_deriv(role, th);
    const float cap = role == GS_ROLE_OPACITY ? K.cap_op : K.cap_sc;
    if (MODE == GS_MODE_ADAMW_GS) {
      // optimizer.py:285-295: min(lambda * (R' / N_I') / (sqrt(v^) + eps), C_t)
      const float x = __fdiv_rn(__fmul_rn(__fmul_rn(lam, deriv), K.inv_ni), den);
      clipped = x >= cap;
      ex = clipped ? cap : x;
    } else if (MODE == GS_MODE_ADAMW_CONST_CLIP) {
      const float x = __fmul_rn(lam, deriv);          // optimizer.py:314-315
      clipped = x >= cap;
      ex = clipped ? cap : x;
    } else {
      ex = __fmul_rn(lam, deriv);
    }
    step = __fadd_rn(step, ex);
  }
  th_out = __fsub_rn(th, __fmul_rn(lr, step));
  m_out = mn;
  v_out = vn;
}

// Domain of the activation (primitives.py:44-48,78-84).
__device__ __forceinline__ bool domain_bad(int role, float theta) {
  if (!isfinite(theta)) return true;
  return role == GS_ROLE_SCALE && (double)theta > 80.0;
}

// Bias-correction factors for clock t (t >= 1).  The host builds the LUT
// until both factors round to exactly 1.0f, so clamping t is exact.
__device__ __forceinline__ float2 bias_factors(const float* lut, int lut_len, int t, double,
                                               double) {
  const int i = t < lut_len ? t : lut_len - 1;
  return __ldg(reinterpret_cast<const float2*>(lut) + i);
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Deterministic block reduction of NV doubles held per thread (sum or max per
// field, selected by is_max[f]); result valid in thread 0.  Uses scratch of
// NV * (kThreads/32) doubles.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], const bool (&is_max)[NV],
                                             double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kThreads / 32;
#pragma unroll
  for (int f = 0; f < NV; ++f) v[f] = is_max[f] ? warp_max(v[f]) : warp_sum(v[f]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) scratch[f * NW + warp] = v[f];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) {
      double acc = scratch[f * NW];
      for (int w = 1; w < NW; ++w)
        acc = is_max[f] ? fmax(acc, scratch[f * NW + w]) : acc + scratch[f * NW + w];
      v[f] = acc;
    }
  }
}

// Same as block_reduce for a block of NW warps (any block size).
template <int NV, int NW>
__device__ __forceinline__ void block_reduce_n(double (&v)[NV], const bool (&is_max)[NV],
                                               double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < NV; ++f) v[f] = is_max[f] ? warp_max(v[f]) : warp_sum(v[f]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) scratch[f * NW + warp] = v[f];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) {
      double acc = scratch[f * NW];
      for (int w = 1; w < NW; ++w)
        acc = is_max[f] ? fmax(acc, scratch[f * NW + w]) : acc + scratch[f * NW + w];
      v[f] = acc;
    }
  }
}

// Last-block-done finalisation: every CTA writes its partials, the last one
// to arrive reduces them in CTA order (deterministic) and re-arms the counter.
// Returns true in every thread of the last CTA.  Thread 0's increment is
// acquire-release at GPU scope: it releases the CTA's writes (ordered before
// it by the barrier) and, in the last CTA, acquires every other CTA's; the
// second barrier extends that to the CTA's other threads.  (Two
// __threadfence()s around a relaxed atomicInc cost ~0.4 us more per launch,
// scripts/launch_probe.cu.)
__device__ __forceinline__ bool last_block_arrive(unsigned int* counter) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev;  // wraps to 0 on the last arrival
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;\n"
                 : "=r"(prev)
                 : "l"(counter), "r"(gridDim.x - 1)
                 : "memory");
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  return s_last;
}

// Grid-wide barrier for kernels whose CTAs are all resident (the two-phase
// step kernel, launched with at most one wave of CTAs): bar[0] counts
// arrivals, bar[1] is the generation.  Thread 0 reads the generation, then
// arrives (acquire-release); the last arrival re-arms the count and releases
// the next generation, the others spin on it.  Both words start at any
// generation with bar[0] == 0 (zeroed workspace) and stay re-armed between
// launches.  A barrier that never opens (a CTA that cannot become resident)
// traps after ~seconds instead of hanging the device.
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen, old;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(gen) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n"
                 : "=r"(old)
                 : "l"(bar)
                 : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;\n" ::"l"(bar) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(bar + 1), "r"(gen + 1u)
                   : "memory");
    } else {
      unsigned int cur;
      long long spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (++spins > (1ll << 26)) __trap();
        if (spins > 64) __nanosleep(64);
      } while (cur == gen);
    }
  }
  __syncthreads();
}

// Densification statistics of one row from its position-group gradient
// (pipeline.py:77-82): accum += sqrt(sum_c g_c^2) * scale, count += 1, in a
// fixed fp32 order (oracle: densify_observe_fp32).
struct DensifyArgs {
  float* accum;
  int32_t* count;
  float scale;
  int group;  // < 0: off
};

__device__ __forceinline__ void densify_row(const DensifyArgs& D, uint32_t row, const float* g,
                                            int w, int stride) {
  float s2 = 0.0f;
  for (int c = 0; c < w; ++c) s2 = __fadd_rn(s2, __fmul_rn(g[c * stride], g[c * stride]));
  const float v = __fmul_rn(__fsqrt_rn(s2), D.scale);
  D.accum[row] = __fadd_rn(D.accum[row], v);
  D.count[row] += 1;
}

// Host: fp32 constants of a step from the C-ABI configuration (every value
// rounded once from float64, as the oracle does).
inline StepConsts make_consts(const gs_step_cfg* cfg) {
  StepConsts K;
  K.a1 = cfg->one_minus_beta1;
  K.a2 = cfg->one_minus_beta2;
  K.eps = cfg->eps;
  K.lam_op = (float)cfg->lambda_opacity;
  K.lam_sc = (float)cfg->lambda_scale;
  K.cap_op = (float)cfg->clip_opacity;
  K.cap_sc = (float)cfg->clip_scale;
  K.inv_ni = cfg->n_pixels_rounded > 0.0 ? (float)(1.0 / cfg->n_pixels_rounded) : 0.0f;
  K.inv_nv = 0.0f;  // coupled modes: set on the device from N_v
  return K;
}

// Final pass of the deterministic cross-CTA reduction, run by the last CTA:
// out[f] = sum (or max) over b of partials[b * stride + f].  Each thread folds
// a fixed strided subset of the CTAs, then a fixed-shape block tree combines
// the threads, so the result depends only on the grid size.
template <int NV>
__device__ __forceinline__ void final_reduce(const double* partials, int nblocks, int stride,
                                             double* out, const bool (&is_max)[NV],
                                             double* scratch) {
  double v[NV];
#pragma unroll
  for (int f = 0; f < NV; ++f) v[f] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
#pragma unroll
    for (int f = 0; f < NV; ++f) {
      const double x = partials[(size_t)b * stride + f];
      v[f] = is_max[f] ? fmax(v[f], x) : v[f] + x;
    }
  }
  block_reduce<NV>(v, is_max, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) out[f] = v[f];
  }
}

template <int NV, int NW>
__device__ __forceinline__ void final_reduce_n(const double* partials, int nblocks, int stride,
                                               double* out, const bool (&is_max)[NV],
                                               double* scratch) {
  double v[NV];
#pragma unroll
  for (int f = 0; f < NV; ++f) v[f] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
#pragma unroll
    for (int f = 0; f < NV; ++f) {
      const double x = partials[(size_t)b * stride + f];
      v[f] = is_max[f] ? fmax(v[f], x) : v[f] + x;
    }
  }
  block_reduce_n<NV, NW>(v, is_max, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < NV; ++f) out[f] = v[f];
  }
}

}  // namespace gs

// host-side error plumbing (gs_abi.cu)
void gs_set_error(const char* fmt, ...);
void gs_fail_launch();  // the next gs_check_launch reports GS_ERR_LAUNCH
int gs_check_launch(const char* what);
int gs_sm_count();

namespace gs {
// Measurement builds only (-DGS_TRACE=1): a device buffer of per-CTA
// globaltimer stamps the step kernel writes (gs_debug_set_trace); the
// product build passes nullptr and compiles no stamps.
inline unsigned long long*& trace_buf() {
  static unsigned long long* p = nullptr;
  return p;
}
#ifdef GS_TRACE
#define GS_STAMP(buf, slot)                                                   \
  do {                                                                        \
    if (buf) {                                                                \
      unsigned long long t_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      (buf)[(size_t)blockIdx.x * 16 + (slot)] = t_;                           \
    }                                                                         \
  } while (0)
#define GS_TRACE_VAL(buf, slot, v) \
  do {                             \
    if (buf) (buf)[(size_t)blockIdx.x * 16 + (slot)] = (v); \
  } while (0)
#else
#define GS_STAMP(buf, slot) \
  do {                      \
  } while (0)
#define GS_TRACE_VAL(buf, slot, v) \
  do {                             \
  } while (0)
#endif

// Opt KERNEL into `bytes` of dynamic shared memory on the current device.
// cudaFuncSetAttribute is per device, so the opt-in is cached per kernel in
// a bitmask of devices (thread-safe); a failure is reported and retried on
// the next launch (which then fails with the CUDA error).
template <auto KERNEL>
inline void smem_opt_in(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  const uint64_t bit = dev < 64 ? (uint64_t{1} << dev) : 0;
  if (bit != 0 && (done.load(std::memory_order_acquire) & bit)) return;
  const cudaError_t e =
      cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    gs_set_error("cudaFuncSetAttribute(%d bytes of shared memory): %s", bytes,
                 cudaGetErrorString(e));
    return;
  }
  done.fetch_or(bit, std::memory_order_acq_rel);
}
}  // namespace gs
