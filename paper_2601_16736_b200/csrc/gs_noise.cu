// Opacity-gated position noise (optimizer.py:453-486; applied to every
// alive row after the step, pipeline.py:334-336):
//
//     delta = -eta_ratio * lr_position * gate(o) * Sigma @ gamma,
//     gate(o) = sigmoid(-lambda_mu * (o - lambda_t)),  o = sigmoid(tau),
//     Sigma = R diag(exp(2 kappa)) R^T,  gamma ~ N(0, I),  dead rows: 0.
//
// 2-D form (the reference testbed): R = rotation by the angle rot.  3-D form
// (3DGS): R from the normalised quaternion (w, x, y, z) as in 3DGS
// build_rotation, kappa = the 3 log-scales.  gamma comes from a counter-based
// Philox4x32-10 stream keyed by the seed and counted by (row, iteration), so
// the draws are reproducible and independent of the launch shape; the
// reference's own host Generator draws are not reproduced (statistical parity
// only).  One thread per row, all rows, HBM-bound:
// 2-D 37 B/row, 3-D 57 B/row.
#include "gs_common.cuh"

namespace gs {

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}

// two standard normals from two uniforms (Box-Muller)
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float u1 = ((float)(a >> 8) + 0.5f) * (1.0f / 16777216.0f);  // (0, 1)
  const float u2 = (float)(b >> 8) * (1.0f / 16777216.0f);           // [0, 1)
  const float r = sqrtf(-2.0f * logf(u1));
  float s, c;
  sincospif(2.0f * u2, &s, &c);
  return make_float2(r * c, r * s);
}

__device__ __forceinline__ float sigmoidf_stable(float x) {
  if (x >= 0.f) return 1.0f / (1.0f + expf(-x));
  const float e = expf(x);
  return e / (1.0f + e);
}

struct RowStrides {
  int64_t x, y, z, w;  // position, log_scale, rotation, opacity_logit
};

// 3DGS rows of the SH-3 parameter record (records.py): position at column
// 0, opacity 51, log-scales 52..54, quaternion 55..58 of one 16-byte-aligned
// row (stride a multiple of 4).  Four 16-byte loads bring a row's inputs
// (columns 0..3 and 48..59), one 16-byte store writes the position back
// (column 3, f_dc[0], is rewritten unchanged).
constexpr int kRecOpac = 51, kRecScale = 52, kRecRot = 55;

template <int D>
__global__ void __launch_bounds__(256)
    noise_kernel(float* __restrict__ pos, const float* __restrict__ kappa,
                 const float* __restrict__ rot, const float* __restrict__ tau,
                 const uint8_t* __restrict__ alive, int64_t n, float coef, float lambda_mu,
                 float lambda_t, uint2 key, uint32_t iteration, float* __restrict__ delta_out,
                 int add, RowStrides rs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float d[D];
#pragma unroll
    for (int k = 0; k < D; ++k) d[k] = 0.f;
    if (alive == nullptr || alive[i]) {
      const uint4 rnd = philox4x32_10(
          make_uint4((uint32_t)i, (uint32_t)(i >> 32), iteration, 0x6e6f6973u /* "nois" */), key);
      const float2 g01 = box_muller(rnd.x, rnd.y);
      const float2 g23 = box_muller(rnd.z, rnd.w);
      const float o = sigmoidf_stable(tau[i * rs.w]);
      const float gate = sigmoidf_stable(-lambda_mu * (o - lambda_t));
      const float a = -coef * gate;
      if (D == 2) {
        const float e0 = expf(2.0f * kappa[i * rs.y]), e1 = expf(2.0f * kappa[i * rs.y + 1]);
        float s, c;
        sincosf(rot[i * rs.z], &s, &c);
        const float sxx = c * c * e0 + s * s * e1;
        const float syy = s * s * e0 + c * c * e1;
        const float sxy = c * s * (e0 - e1);
        d[0] = a * (sxx * g01.x + sxy * g01.y);
        d[1] = a * (sxy * g01.x + syy * g01.y);
      } else {
        const float* qp = rot + i * rs.z;
        const float4 q4 = make_float4(qp[0], qp[1], qp[2], qp[3]);
        const float qn = rsqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
        const float w = q4.x * qn, x = q4.y * qn, y = q4.z * qn, z = q4.w * qn;
        const float Rm[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y)},
                                {2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x)},
                                {2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)}};
        const float g[3] = {g01.x, g01.y, g23.x};
        float u[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)  // u = S^2 R^T gamma
          u[r] = expf(2.0f * kappa[i * rs.y + r]) * (Rm[0][r] * g[0] + Rm[1][r] * g[1] + Rm[2][r] * g[2]);
#pragma unroll
        for (int r = 0; r < 3; ++r) d[r] = a * (Rm[r][0] * u[0] + Rm[r][1] * u[1] + Rm[r][2] * u[2]);
      }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (delta_out) delta_out[D * i + k] = d[k];
      if (add) pos[i * rs.x + k] += d[k];
    }
  }
}

__device__ __forceinline__ float3 noise_delta3(const float4 q4, const float3 ks, float tau,
                                               uint32_t row_lo, uint32_t row_hi, uint32_t it,
                                               uint2 key, float coef, float lambda_mu,
                                               float lambda_t) {
  const uint4 rnd = philox4x32_10(make_uint4(row_lo, row_hi, it, 0x6e6f6973u), key);
  const float2 g01 = box_muller(rnd.x, rnd.y);
  const float2 g23 = box_muller(rnd.z, rnd.w);
  const float o = sigmoidf_stable(tau);
  const float gate = sigmoidf_stable(-lambda_mu * (o - lambda_t));
  const float a = -coef * gate;
  const float qn = rsqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
  const float w = q4.x * qn, x = q4.y * qn, y = q4.z * qn, z = q4.w * qn;
  const float Rm[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y)},
                          {2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x)},
                          {2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)}};
  const float g[3] = {g01.x, g01.y, g23.x};
  const float e[3] = {expf(2.0f * ks.x), expf(2.0f * ks.y), expf(2.0f * ks.z)};
  float u[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)  // u = S^2 R^T gamma
    u[r] = e[r] * (Rm[0][r] * g[0] + Rm[1][r] * g[1] + Rm[2][r] * g[2]);
  return make_float3(a * (Rm[0][0] * u[0] + Rm[0][1] * u[1] + Rm[0][2] * u[2]),
                     a * (Rm[1][0] * u[0] + Rm[1][1] * u[1] + Rm[1][2] * u[2]),
                     a * (Rm[2][0] * u[0] + Rm[2][1] * u[1] + Rm[2][2] * u[2]));
}

// 16-byte load with a 64-byte L2 fetch: a record row's inputs sit in two
// 64-byte granules (columns 0..3 and 48..59 of 64); the default 128-byte
// fetch would pull the whole 256-byte row
__device__ __forceinline__ float4 ld_l2_64(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L2::64B.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// The same noise as noise_kernel<3> (identical draws and arithmetic) on SH-3
// parameter records, 16-byte accesses.
__global__ void __launch_bounds__(256)
    noise_rec_kernel(float* __restrict__ rec, int64_t stride, const uint8_t* __restrict__ alive,
                     int64_t n, float coef, float lambda_mu, float lambda_t, uint2 key,
                     uint32_t iteration, float* __restrict__ delta_out, int add) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float* row = rec + i * stride;
    const bool live = alive == nullptr || alive[i];
    float3 d = make_float3(0.f, 0.f, 0.f);
    float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      p4 = ld_l2_64(row);
      const float4 c48 = ld_l2_64(row + 48);  // .w = opacity (51)
      const float4 c52 = ld_l2_64(row + 52);  // log-scales, q.w
      const float4 c56 = ld_l2_64(row + 56);  // q.x, q.y, q.z, pad
      d = noise_delta3(make_float4(c52.w, c56.x, c56.y, c56.z), make_float3(c52.x, c52.y, c52.z),
                       c48.w, (uint32_t)i, (uint32_t)(i >> 32), iteration, key, coef, lambda_mu,
                       lambda_t);
    }
    if (delta_out) {
      delta_out[3 * i] = d.x;
      delta_out[3 * i + 1] = d.y;
      delta_out[3 * i + 2] = d.z;
    }
    if (add && live) {
      p4.x += d.x;
      p4.y += d.y;
      p4.z += d.z;
      *reinterpret_cast<float4*>(row) = p4;
    }
  }
}

}  // namespace gs

extern "C" int gs_noise_perturb(float* position, const float* log_scale, const float* rotation,
                                const float* opacity_logit, const uint8_t* alive, int64_t n,
                                int32_t dims, float lr_position, float eta_ratio,
                                float lambda_mu, float lambda_t, uint64_t seed,
                                uint32_t iteration, float* delta_out, int32_t add_in_place,
                                const int64_t* row_strides, void* stream) {
  using namespace gs;
  if (n < 0 || !position || !log_scale || !rotation || !opacity_logit ||
      (dims != 2 && dims != 3) || (!delta_out && !add_in_place)) {
    gs_set_error("gs_noise_perturb: invalid arguments");
    return GS_ERR_ARG;
  }
  const int64_t dense[4] = {dims, dims, dims == 2 ? 1 : 4, 1};
  RowStrides rs;
  int64_t* rp = &rs.x;
  for (int j = 0; j < 4; ++j) {
    rp[j] = (row_strides && row_strides[j] != 0) ? row_strides[j] : dense[j];
    if (rp[j] < dense[j]) {
      gs_set_error("gs_noise_perturb: row stride %d (%lld) below the row width", j,
                   (long long)rp[j]);
      return GS_ERR_ARG;
    }
  }
  if (n == 0) return GS_OK;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const float coef = eta_ratio * lr_position;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)gs_sm_count() * 32);
  cudaStream_t s = (cudaStream_t)stream;
  const bool rec = dims == 3 && rs.x == rs.y && rs.x == rs.z && rs.x == rs.w && rs.x % 4 == 0 &&
                   rs.x >= 60 && (reinterpret_cast<uintptr_t>(position) & 15u) == 0 &&
                   opacity_logit == position + kRecOpac && log_scale == position + kRecScale &&
                   rotation == position + kRecRot;
  if (rec) {
    noise_rec_kernel<<<grid, 256, 0, s>>>(position, rs.x, alive, n, coef, lambda_mu, lambda_t,
                                          key, iteration, delta_out, add_in_place);
  } else if (dims == 2)
    noise_kernel<2><<<grid, 256, 0, s>>>(position, log_scale, rotation, opacity_logit, alive, n,
                                         coef, lambda_mu, lambda_t, key, iteration, delta_out,
                                         add_in_place, rs);
  else
    noise_kernel<3><<<grid, 256, 0, s>>>(position, log_scale, rotation, opacity_logit, alive, n,
                                         coef, lambda_mu, lambda_t, key, iteration, delta_out,
                                         add_in_place, rs);
  return gs_check_launch("gs_noise_perturb");
}
