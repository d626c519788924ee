// On-GPU seed expansion: SHAKE-256 of the reference's per-block seed material.
//
// Reference (pkg/src/modpa/pa.py):
//   _expand(material, label, n)      pa.py:138-153
//       shake_256(le16(len(label)) || label || le32(len(material)) || material)
//           .digest(ceil(n/8)), read little-endian, masked to n bits
//   gen_seed(n, material)            pa.py:156-167  c = _expand(.., b"multiplier", n) | 1,
//                                                   d = _expand(.., b"offset", n)
//   derive_block_seed(master, i)     pa.py:170-172  _expand(master, b"block-%d" % i, 256)
//                                                   .to_bytes(32, "little")
// run_pa hashes block i with gen_seed(n, derive_block_seed(rng_seed, i))
// (pkg/src/modpa/bench.py:256-262).  Here one thread owns one XOF stream
// (block i's c or d): it derives the 32-byte block seed (one Keccak-f), absorbs
// the c/d message (one block) and squeezes ceil(n/8) bytes straight into the
// operand row in the layout pab_hash_batch reads.  The squeeze is a chain of
// dependent permutations, so the kernel is latency-bound per stream; it uses a
// small slice of the GPU and is meant to run on its own stream beside the
// convolution of the previous batch.
//
// Keccak-f[1600] (FIPS 202 §3): 24 rounds of theta, rho, pi, chi, iota on 25
// 64-bit lanes A[x + 5y]; SHAKE-256 rate 136 bytes, domain/pad bytes 0x1F ... 0x80.
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "pa_kernels.cuh"

namespace pab {
namespace {

__constant__ uint64_t kRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

// rho offsets r[x][y] at index x + 5y
constexpr int kRho[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                          25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

constexpr int kRate = 136;     // SHAKE-256 rate in bytes
constexpr int kRateW = 17;     // ... in 64-bit lanes

template <int R>
__device__ __forceinline__ uint64_t rotl(uint64_t v) {
  if constexpr (R == 0) {
    return v;
  } else {
    // two funnel shifts (SHF.L.W) on the 32-bit halves
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    uint32_t nlo, nhi;
    if constexpr (R < 32) {
      nhi = __funnelshift_l(lo, hi, R);
      nlo = __funnelshift_l(hi, lo, R);
    } else if constexpr (R == 32) {
      nhi = lo;
      nlo = hi;
    } else {
      nhi = __funnelshift_l(hi, lo, R - 32);
      nlo = __funnelshift_l(lo, hi, R - 32);
    }
    return ((uint64_t)nhi << 32) | nlo;
  }
}

template <int I>
struct IC {
  static constexpr int value = I;
};
template <int N, typename F, int... Is>
__device__ __forceinline__ void unroll_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(IC<Is>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void unroll(F&& f) {
  unroll_impl<N>(f, std::make_integer_sequence<int, N>{});
}

// Keccak-f[1600] in registers (every index compile-time).
__device__ __forceinline__ void keccak_f(uint64_t (&A)[25]) {
#pragma unroll 1
  for (int round = 0; round < 24; ++round) {
    uint64_t C[5], D[5], B[25];
#pragma unroll
    for (int x = 0; x < 5; ++x) C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];
#pragma unroll
    for (int x = 0; x < 5; ++x) D[x] = C[(x + 4) % 5] ^ rotl<1>(C[(x + 1) % 5]);
    // theta, rho and pi: B[y + 5 ((2x + 3y) mod 5)] = rotl(A[x + 5y] ^ D[x], r[x][y])
    unroll<25>([&](auto i) {
      constexpr int x = decltype(i)::value % 5, y = decltype(i)::value / 5;
      B[y + 5 * ((2 * x + 3 * y) % 5)] = rotl<kRho[x + 5 * y]>(A[x + 5 * y] ^ D[x]);
    });
    // chi
#pragma unroll
    for (int y = 0; y < 5; ++y)
#pragma unroll
      for (int x = 0; x < 5; ++x)
        A[x + 5 * y] = B[x + 5 * y] ^ (~B[(x + 1) % 5 + 5 * y] & B[(x + 2) % 5 + 5 * y]);
    // iota
    A[0] ^= kRC[round];
  }
}

// Absorb one message of `len` bytes given by byte(k) and pad it (SHAKE domain
// 0x1F, final 0x80): state A (zeroed by the caller) ends permuted, ready to squeeze.
template <typename ByteFn>
__device__ __forceinline__ void absorb(uint64_t (&A)[25], int len, ByteFn byte) {
  uint64_t blk[kRateW];  // local memory: dynamic byte indexing
  for (int base = 0;; base += kRate) {
    const int rem = len - base;  // bytes of the message left (may be <= 0)
    for (int w = 0; w < kRateW; ++w) {
      uint64_t v = 0;
      for (int q = 0; q < 8; ++q) {
        const int k = 8 * w + q;
        uint64_t b = k < rem ? (uint64_t)byte(base + k) : 0u;
        if (k == rem) b ^= 0x1Fu;
        if (k == kRate - 1 && rem < kRate) b ^= 0x80u;
        v |= b << (8 * q);
      }
      blk[w] = v;
    }
#pragma unroll
    for (int w = 0; w < kRateW; ++w) A[w] ^= blk[w];
    keccak_f(A);
    if (rem < kRate) break;
  }
}

__device__ __forceinline__ int dec_len(unsigned long long v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// Thread t: block j = t / 2 (index first + j), stream t % 2 (0: c, 1: d).
__global__ void __launch_bounds__(32) k_seed_expand(const SeedMaster master, int mlen,
                                                     unsigned long long first, int batch,
                                                     long long n_bits, int msf, int word_io,
                                                     uint8_t* __restrict__ c,
                                                     uint8_t* __restrict__ d, long long stride) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * batch) return;
  const int j = t >> 1, which = t & 1;
  const unsigned long long idx = first + (unsigned long long)j;
  uint64_t A[25];
  // derive_block_seed(master, idx): label b"block-%d" % idx
  const int dl = dec_len(idx);
  const int llen = 6 + dl;  // "block-" + digits
  {
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] = 0;
    const int len = 2 + llen + 4 + mlen;
    absorb(A, len, [&](int k) -> uint8_t {
      if (k < 2) return (uint8_t)(llen >> (8 * k));
      k -= 2;
      if (k < llen) {
        if (k < 6) return (uint8_t)"block-"[k];
        unsigned long long v = idx;
        for (int e = dl - 1 - (k - 6); e > 0; --e) v /= 10;
        return (uint8_t)('0' + v % 10);
      }
      k -= llen;
      if (k < 4) return (uint8_t)((unsigned)mlen >> (8 * k));
      return master.b[k - 4];
    });
  }
  uint64_t S[4];  // 32-byte block seed = first four lanes
#pragma unroll
  for (int i = 0; i < 4; ++i) S[i] = A[i];
  // gen_seed(n, S): label b"multiplier" (c) or b"offset" (d), material S (32 bytes)
  {
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] = 0;
    const int ll = which ? 6 : 10;
    const int len = 2 + ll + 4 + 32;
    absorb(A, len, [&](int k) -> uint8_t {
      if (k < 2) return (uint8_t)(ll >> (8 * k));
      k -= 2;
      if (k < ll) return (uint8_t)(which ? "offset"[k] : "multiplier"[k]);
      k -= ll;
      if (k < 4) return (uint8_t)(32u >> (8 * k));
      k -= 4;
      return (uint8_t)(S[k >> 3] >> (8 * (k & 7)));
    });
  }
  // squeeze ceil(n/8) bytes, masked to n bits; c |= 1
  const long long nb = (n_bits + 7) >> 3;
  const int top = (int)(n_bits & 7);
  const uint8_t topmask = top ? (uint8_t)((1u << top) - 1u) : (uint8_t)0xFF;
  uint8_t* row = (which ? d : c) + (long long)j * stride;
  for (long long base = 0; base < nb; base += kRate) {
    if (base) keccak_f(A);
    const long long rem = nb - base;
    if (word_io && rem >= kRate) {  // LSF, 8-byte aligned row: whole lanes
      uint64_t* o = reinterpret_cast<uint64_t*>(row + base);
#pragma unroll
      for (int w = 0; w < kRateW; ++w) o[w] = A[w];
    } else {
#pragma unroll
      for (int w = 0; w < kRateW; ++w) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const long long k = base + 8 * w + q;
          if (k < nb) {
            uint8_t b = (uint8_t)(A[w] >> (8 * q));
            if (k == nb - 1) b &= topmask;
            if (k == 0 && !which) b |= 1u;
            row[msf ? nb - 1 - k : k] = b;
          }
        }
      }
    }
  }
  if (word_io && nb >= kRate) {  // fix the first / last byte written as whole lanes
    if (!which) row[0] |= 1u;
    if (nb % kRate == 0) row[nb - 1] &= topmask;
  }
}

}  // namespace

// (pa_kernels.cu's launch_seed_expand wraps this with the profiling scope)
void seed_expand_raw(const SeedMaster& master, int mlen, unsigned long long first, int batch,
                     long long n_bits, int msf, int word_io, uint8_t* c, uint8_t* d,
                     long long stride, cudaStream_t st) {
  const int threads = 2 * batch;
  const int per = 32;  // one warp per CTA: the few streams spread over the SMs
  const dim3 grid((threads + per - 1) / per);
  k_seed_expand<<<grid, per, 0, st>>>(master, mlen, first, batch, n_bits, msf, word_io, c, d,
                                      stride);
}

}  // namespace pab
