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

#include "../../include/adamw_gs.h"

namespace gs {

constexpr int kThreads = 256;  // rows per chunk == threads per CTA

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

// Stable float64 sigmoid derivative, primitives.py:51-66.
__device__ __forceinline__ double sigmoid_deriv_f64(double t) {
  double o;
  if (t >= 0.0) {
    o = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-t)));
  } else {
    double e = exp(t);
    o = __ddiv_rn(e, __dadd_rn(1.0, e));
  }
  return __dmul_rn(o, __dsub_rn(1.0, o));
}

// R'(theta) of the L1 penalty on the activated attribute (primitives.py:62-84).
__device__ __forceinline__ double reg_deriv_f64(int role, float theta) {
  double t = (double)theta;
  return role == GS_ROLE_OPACITY ? sigmoid_deriv_f64(t) : exp(t);
}

// Domain of the activation (primitives.py:44-48,78-84).
__device__ __forceinline__ bool domain_bad(int role, float theta) {
  if (!isfinite(theta)) return true;
  return role == GS_ROLE_SCALE && (double)theta > 80.0;
}

// Bias-correction factors for clock t (t >= 1).
__device__ __forceinline__ float2 bias_factors(const float* lut, int lut_len, int t,
                                               double beta1, double beta2) {
  if (t < lut_len) {
    return reinterpret_cast<const float2*>(lut)[t];
  }
  double td = (double)t;
  float c1 = __double2float_rn(__ddiv_rn(1.0, __dsub_rn(1.0, pow(beta1, td))));
  float c2 = __double2float_rn(__ddiv_rn(1.0, __dsub_rn(1.0, pow(beta2, td))));
  return make_float2(c1, c2);
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

// Last-block-done finalisation: every CTA writes its partials, the last one
// to arrive reduces them in CTA order (deterministic) and re-arms the counter.
// Returns true in thread 0 of the last CTA.
__device__ __forceinline__ bool last_block_arrive(unsigned int* counter) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicInc(counter, gridDim.x - 1);  // wraps to 0 on the last
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

}  // namespace gs

// host-side error plumbing (gs_abi.cu)
void gs_set_error(const char* fmt, ...);
int gs_check_launch(const char* what);
int gs_sm_count();
