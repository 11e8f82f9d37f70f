// The reference's host Bernoulli draw on the GPU: NumPy's Philox4x64-10 bit
// generator (the rng.stream of rng.py:17-30; numpy/random/src/philox/
// philox.h) and Generator.random's next_double, restated bit for bit, so
// aiu_apply's picks ``rng.random(n_invisible) < prob`` (optimizer.py:
// 437-440) are drawn where the invisible list lives instead of on the host.
// Pinned by oracle.philox_uniforms (itself checked against numpy).
#include "gs_common.cuh"

namespace gs {

struct U256 {
  uint64_t v[4];
};

__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// out[i] = u(first + i) < prob for i < n, u(j) = (philox(ctr + 1 + j/4)[j%4]
// >> 11) * 2^-53: draw j of a generator whose buffer is empty
// (buffer_pos = 4) at counter ctr.  A thread per Philox block.
__global__ void __launch_bounds__(kThreads)
    philox_bernoulli_kernel(U256 ctr, uint64_t k0, uint64_t k1, int64_t first, int64_t n,
                            double prob, uint8_t* __restrict__ out) {
  const int64_t b0 = first >> 2, b1 = (first + n - 1) >> 2;
  for (int64_t b = b0 + blockIdx.x * (int64_t)kThreads + threadIdx.x; b <= b1;
       b += (int64_t)gridDim.x * kThreads) {
    // counter + 1 + b, 256-bit
    uint64_t c[4];
    const uint64_t add = (uint64_t)b + 1u;
    c[0] = ctr.v[0] + add;
    uint64_t carry = c[0] < add ? 1u : 0u;
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      c[w] = ctr.v[w] + carry;
      carry = (carry && c[w] == 0) ? 1u : 0u;
    }
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int64_t j = 4 * b + l;
      if (j >= first && j < first + n) {
        const double u = (double)(c[l] >> 11) * (1.0 / 9007199254740992.0);
        out[j - first] = u < prob ? 1 : 0;
      }
    }
  }
}

}  // namespace gs

extern "C" int gs_philox_bernoulli(const uint64_t* counter, const uint64_t* key, int64_t first,
                                   int64_t n, double prob, uint8_t* out, void* stream) {
  using namespace gs;
  if (!counter || !key || first < 0 || n < 0 || (n > 0 && !out)) {
    gs_set_error("gs_philox_bernoulli: invalid arguments");
    return GS_ERR_ARG;
  }
  if (n == 0) return GS_OK;
  U256 c{{counter[0], counter[1], counter[2], counter[3]}};
  const int64_t blocks = ((first + n - 1) >> 2) - (first >> 2) + 1;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((blocks + kThreads - 1) / kThreads, (int64_t)gs_sm_count() * 8));
  philox_bernoulli_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(c, key[0], key[1], first,
                                                                        n, prob, out);
  return gs_check_launch("gs_philox_bernoulli");
}
