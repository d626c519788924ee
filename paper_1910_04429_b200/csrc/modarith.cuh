// Word-size modular arithmetic for the multi-prime NTT (sm_100a integer pipe).
//
// The reference multiplies in the Fermat ring Z/(2^N'+1) with shift twiddles
// (pkg/src/modpa/ntt.py:123-160).  On B200 the product is instead formed as
// an exact cyclic convolution of 64-bit (or 32-bit) coefficients over five
// (or three) primes p_i < 2^30
// (CRT-recombined in the carry kernel), so every operation here is on u32
// registers: Shoup multiplication for known twiddles, Montgomery reduction
// for products of two data values, and Harvey-style lazy butterflies that
// keep values in [0, 2p) or [0, 4p) instead of fully reducing.
#pragma once
#include <cstdint>

namespace pab {

typedef uint32_t u32;
typedef uint64_t u64;

// Two convolution modes (the "coefficient width" cw of a job):
//   cw = 2: 64-bit coefficients (two words each) over all five primes; product
//           ~2^148.85, so K' * (2^64-1)^2 < P for K' <= 1,895,236 coefficients;
//           lengths m * 2^lg with lg <= kMaxLg5 (n <= 121,295,104 bits).
//   cw = 1: 32-bit coefficients over the first three primes (2-adicity >= 22),
//           product ~2^89.02, lengths up to 5 * 2^22 (n <= 335,544,320 bits).
// Every p_i < 2^30 (so 4p < 2^32) with 3 * 5 | p_i - 1 (radix-3/5 lengths).
// kGen: a primitive root of each prime.
constexpr int kNumPrimes = 5;
constexpr u32 kPrimes[kNumPrimes] = {943718401u, 880803841u, 754974721u, 1053818881u,
                                     975175681u};
constexpr u32 kGen[kNumPrimes] = {7u, 26u, 11u, 7u, 17u};
constexpr int kMaxLg = 22;        // 2-adicity common to primes 0..2 (cw = 1)
constexpr int kMaxLg5 = 20;       // 2-adicity common to all five (cw = 2)
constexpr int kTwN = 4096;        // largest in-CTA sub-transform
constexpr int kTwLg = 12;

#ifdef __CUDACC__
// Shoup multiplication a*w mod p with precomputed wp = floor(w*2^32/p).
// Any a < 2^32; result in [0, 2p).
__device__ __forceinline__ u32 shoup(u32 a, u32 w, u32 wp, u32 p) {
  u32 q = __umulhi(a, wp);
  return a * w - q * p;
}
__device__ __forceinline__ u32 shoup(u32 a, uint2 w, u32 p) { return shoup(a, w.x, w.y, p); }

// [0, 2m) -> [0, m) (unsigned wrap makes the min pick the right branch).
__device__ __forceinline__ u32 red(u32 a, u32 m) { return min(a, a - m); }

// Montgomery product a*b*2^-32 mod p; a*b < 4p^2 gives a result in [0, 2p).
__device__ __forceinline__ u32 montmul(u32 a, u32 b, u32 p, u32 p_mont) {
  u64 t = (u64)a * b;
  u32 lo = (u32)t, hi = (u32)(t >> 32);
  u32 m = lo * p_mont;
  u32 mh = __umulhi(m, p);
  return hi + mh + (lo != 0u ? 1u : 0u);
}

#endif

}  // namespace pab
