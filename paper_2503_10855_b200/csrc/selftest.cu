// selftest.cu -- device self-checks of the branch-free fast paths in
// common.cuh against the compiler's IEEE __fdiv_rn / __fsqrt_rn, on random
// operands drawn uniformly in exponent and mantissa over a guarded range.
// Used by tests/test_fastmath_gpu.py; not on any benchmark path.
#include "common.cuh"

namespace jb {
namespace selftest {

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
// random float with exponent in [lo, hi], random mantissa and sign (if sgn)
__device__ __forceinline__ float rnd(uint64_t h, int lo, int hi, bool sgn) {
  const unsigned m = (unsigned)h & 0x7fffffu;
  const int e = lo + (int)((h >> 23) % (uint64_t)(hi - lo + 1));
  unsigned b = ((unsigned)(e + 127) << 23) | m;
  if (sgn && ((h >> 40) & 1)) b |= 0x80000000u;
  return __uint_as_float(b);
}

__global__ void fastmath_kernel(uint64_t n, uint64_t seed, int lo, int hi, unsigned long long *bad) {
  unsigned long long nd = 0, nr = 0, ns = 0, nb = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed * 0x9e3779b97f4a7c15ull + 2 * i), h2 = mix(h1 + 0x632be59bd9b4e019ull);
    const float a = rnd(h1, lo, hi, true), b = rnd(h2, lo, hi, true);
    // quotient outside the guarded range is not covered by the contract
    const float qe = __fdiv_rn(a, b);
    const float aq = fabsf(qe);
    if (aq >= 0x1p-96f && aq <= 0x1p96f) {
      nd += __float_as_uint(div_fast(a, b)) != __float_as_uint(qe);
      nb += __float_as_uint(div_by(a, b, recip_refined(b))) != __float_as_uint(qe);
    }
    nr += __float_as_uint(rcp_fast(b)) != __float_as_uint(__fdiv_rn(1.0f, b));
    const float x = fabsf(a);
    if (sqrt_fast_ok(x)) ns += __float_as_uint(sqrt_fast(x)) != __float_as_uint(__fsqrt_rn(x));
  }
  atomicAdd(bad + 0, nd);
  atomicAdd(bad + 1, nr);
  atomicAdd(bad + 2, ns);
  atomicAdd(bad + 3, nb);
}

}  // namespace selftest
}  // namespace jb

extern "C" jb_status jb_selftest_fastmath(uint64_t n, uint64_t seed, int exp_lo, int exp_hi,
                                         unsigned long long *mismatches, void *stream) {
  JB_REQUIRE(mismatches && exp_lo <= exp_hi && exp_lo >= -126 && exp_hi <= 127, "selftest: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  JB_CHECK_CUDA(cudaMemsetAsync(mismatches, 0, 4 * sizeof(unsigned long long), s));
  jb::selftest::fastmath_kernel<<<jb::sm_count() * 8, 256, 0, s>>>(n, seed, exp_lo, exp_hi, mismatches);
  JB_LAUNCHED("selftest_fastmath");
  return JB_OK;
}
