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
// (pkg/src/modpa/bench.py:256-262).  Here each XOF stream (block i's c or d)
// is owned by a lane pair holding the two bit-interleaved
// halves of the Keccak state: it derives the 32-byte block seed (one
// Keccak-f), absorbs the c/d message (one block) and squeezes ceil(n/8) bytes
// straight into the operand row in the layout pab_hash_batch reads.  The
// squeeze is a chain of dependent permutations, so the kernel is latency-bound
// per stream (measured 3.2 us per Keccak-f = 260 cycles per round of 119
// instructions, 90 of them on the half-rate alu pipe: ~0.7 of one SMSP's alu
// issue bound); it uses a small slice of the GPU and runs on its own stream
// beside the hashing of the previous batch.
//
// Keccak-f[1600] (FIPS 202 §3): 24 rounds of theta, rho, pi, chi, iota on 25
// 64-bit lanes A[x + 5y]; SHAKE-256 rate 136 bytes, domain/pad bytes 0x1F ... 0x80.
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "pa_kernels.cuh"

namespace pab {
namespace {

// rho offsets r[x][y] at index x + 5y
constexpr int kRho[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                          25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

constexpr int kRate = 136;     // SHAKE-256 rate in bytes
constexpr int kRateW = 17;     // ... in 64-bit lanes
constexpr unsigned kFull = 0xFFFFFFFFu;

// Bit interleaving (the standard 32-bit Keccak representation): a 64-bit lane v
// is held as e = its even bits and o = its odd bits.  XOR/AND/NOT act on each
// half alone, and rotl64(v, 2k) = (rotl32(e, k), rotl32(o, k)),
// rotl64(v, 2k+1) = (rotl32(o, k+1), rotl32(e, k)).  So a pair of lanes of a
// warp can share one permutation: lane 2s holds the e halves of all 25 Keccak
// lanes and lane 2s+1 the o halves; odd rotations trade halves with one
// shuffle.  This halves the instructions on each thread's dependent chain
// (the squeeze is a chain of permutations, so its latency is the cost).
__host__ __device__ constexpr uint32_t even_bits(uint64_t v) {
  uint32_t r = 0;
  for (int i = 0; i < 32; ++i) r |= (uint32_t)((v >> (2 * i)) & 1u) << i;
  return r;
}
struct RC2 {
  uint32_t h[48];  // [round][half]: even / odd bits of the round constant
};
constexpr uint64_t kRC64[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};
constexpr RC2 make_rc2() {
  RC2 r{};
  for (int i = 0; i < 24; ++i) {
    r.h[2 * i] = even_bits(kRC64[i]);
    r.h[2 * i + 1] = even_bits(kRC64[i] >> 1);
  }
  return r;
}
__constant__ RC2 kRC2 = make_rc2();

// 16 bits -> the even bit positions of a 32-bit word, and back
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}
__device__ __forceinline__ uint32_t compact16(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}
// this thread's half (par 0: even bits, 1: odd bits) of a 64-bit lane
__device__ __forceinline__ uint32_t half_of(uint64_t v, uint32_t par) {
  const uint32_t lo = (uint32_t)v >> par, hi = (uint32_t)(v >> 32) >> par;
  return compact16(lo) | (compact16(hi) << 16);
}
__device__ __forceinline__ uint64_t zip(uint32_t e, uint32_t o) {
  const uint32_t lo = spread16(e) | (spread16(o) << 1);
  const uint32_t hi = spread16(e >> 16) | (spread16(o >> 16) << 1);
  return ((uint64_t)hi << 32) | lo;
}

// rotl32 with SHF.L.W (alu pipe).  Moving rotations to the fma pipe as an
// IMAD.HI + IMAD pair (disjoint bits: the add is the OR) was measured slower:
// the round is latency-bound on one warp per SMSP, and the pair doubles the
// rotation's latency (1e6: 3.94 / 4.90 ms for constant / all rotations vs 3.75).
template <int K>
__device__ __forceinline__ uint32_t rotc(uint32_t v) {  // compile-time rotl32
  if constexpr (K % 32 == 0) {
    return v;
  } else {
    return __funnelshift_l(v, v, K);
  }
}
__device__ __forceinline__ uint32_t rotv(uint32_t v, uint32_t k) {  // rotl32 by k mod 32
  return __funnelshift_l(v, v, k);
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

// Keccak-f[1600] on a lane pair: A holds this thread's halves (every index
// compile-time); par = lane & 1.  All 32 lanes of the warp must call it.
__device__ __forceinline__ void keccak_f2(uint32_t (&A)[25], uint32_t par) {
  const uint32_t a1 = 1u - par;  // extra rotation of an odd-offset lane's e half
  // 8 rounds per loop iteration: the scheduler overlaps one round's chi with the
  // next round's theta (1e6: 3.75 -> 2.92 ms per launch; 2 / 4 / 6 / 12 rounds:
  // 3.31 / 3.10 / 2.98 / 2.94 ms; all 24: 4.32 ms, i-cache)
#pragma unroll 8
  for (int round = 0; round < 24; ++round) {
    uint32_t C[5], R[5], B[25];
#pragma unroll
    for (int x = 0; x < 5; ++x) C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];
    // theta: D[x] = C[x-1] ^ rotl64(C[x+1], 1)
#pragma unroll
    for (int x = 0; x < 5; ++x) R[x] = rotv(__shfl_xor_sync(kFull, C[(x + 1) % 5], 1), a1);
    // theta, rho and pi: B[y + 5 ((2x + 3y) mod 5)] = rotl64(A[x + 5y] ^ D[x], r[x][y])
    unroll<25>([&](auto i) {
      constexpr int x = decltype(i)::value % 5, y = decltype(i)::value / 5;
      constexpr int r = kRho[x + 5 * y];
      const uint32_t v = A[x + 5 * y] ^ C[(x + 4) % 5] ^ R[x];
      uint32_t o;
      if constexpr (r % 2 == 0) {
        o = rotc<r / 2>(v);
      } else {
        o = rotv(__shfl_xor_sync(kFull, v, 1), (uint32_t)(r / 2) + a1);
      }
      B[y + 5 * ((2 * x + 3 * y) % 5)] = o;
    });
    // chi
#pragma unroll
    for (int y = 0; y < 5; ++y)
#pragma unroll
      for (int x = 0; x < 5; ++x)
        A[x + 5 * y] = B[x + 5 * y] ^ (~B[(x + 1) % 5 + 5 * y] & B[(x + 2) % 5 + 5 * y]);
    // iota
    A[0] ^= kRC2.h[2 * round + par];
  }
}

// Absorb one message of `len` bytes given by byte(k) and pad it (SHAKE domain
// 0x1F, final 0x80): state A (zeroed by the caller) ends permuted, ready to squeeze.
template <typename ByteFn>
__device__ __forceinline__ void absorb(uint32_t (&A)[25], uint32_t par, int len, ByteFn byte) {
  uint32_t blk[kRateW];  // local memory: dynamic byte indexing
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
      blk[w] = half_of(v, par);
    }
#pragma unroll
    for (int w = 0; w < kRateW; ++w) A[w] ^= blk[w];
    keccak_f2(A, par);
    if (rem < kRate) break;
  }
}

// the 64-bit Keccak lane w from both halves of a pair (a warp-wide shuffle)
__device__ __forceinline__ uint64_t lane64(uint32_t mine, uint32_t par) {
  const uint32_t other = __shfl_xor_sync(kFull, mine, 1);
  return par ? zip(other, mine) : zip(mine, other);
}

__device__ __forceinline__ int dec_len(unsigned long long v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// Lane pair s = t / 2 of the grid owns XOF stream s: block j = s / 2 (index
// first + j), stream s % 2 (0: c, 1: d); lane parity = which half it holds.
// fixed_index < 0 (run_pa, pkg/src/modpa/bench.py:258): block j's seed is
//   gen_seed(n, derive_block_seed(master, first + j));
// fixed_index >= 0 (the reference's bench protocol, bench.py:156): block j's
// seed material is the integer s = first + j itself and the label index is fixed,
//   gen_seed(n, derive_block_seed(s, fixed_index))   (fixed_index = n there).
__global__ void __launch_bounds__(64) k_seed_expand(const SeedMaster master, int mlen,
                                                     unsigned long long first, int batch,
                                                     long long n_bits, int msf, int word_io,
                                                     uint8_t* __restrict__ c,
                                                     uint8_t* __restrict__ d, long long stride,
                                                     long long fixed_index) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t par = t & 1;
  const int s_raw = t >> 1;
  const bool active = s_raw < 2 * batch;  // idle pairs still shuffle with the warp
  const int s = active ? s_raw : 2 * batch - 1;
  const int j = s >> 1, which = s & 1;
  const unsigned long long blk = first + (unsigned long long)j;
  const bool bench = fixed_index >= 0;
  // derive_block_seed(material, idx): label b"block-%d" % idx
  const unsigned long long idx = bench ? (unsigned long long)fixed_index : blk;
  // an int seed s is s.to_bytes(max(1, ceil(bitlen / 8)), "little") (pa.py:141-146)
  const int ml = bench ? (blk ? (64 - __clzll((long long)blk) + 7) / 8 : 1) : mlen;
  uint32_t A[25];
  const int dl = dec_len(idx);
  const int llen = 6 + dl;  // "block-" + digits
  {
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] = 0;
    const int len = 2 + llen + 4 + ml;
    absorb(A, par, len, [&](int k) -> uint8_t {
      if (k < 2) return (uint8_t)(llen >> (8 * k));
      k -= 2;
      if (k < llen) {
        if (k < 6) return (uint8_t)"block-"[k];
        unsigned long long v = idx;
        for (int e = dl - 1 - (k - 6); e > 0; --e) v /= 10;
        return (uint8_t)('0' + v % 10);
      }
      k -= llen;
      if (k < 4) return (uint8_t)((unsigned)ml >> (8 * k));
      return bench ? (uint8_t)(blk >> (8 * (k - 4))) : master.b[k - 4];
    });
  }
  uint64_t S[4];  // 32-byte block seed = first four lanes
#pragma unroll
  for (int i = 0; i < 4; ++i) S[i] = lane64(A[i], par);
  // gen_seed(n, S): label b"multiplier" (c) or b"offset" (d), material S (32 bytes)
  {
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] = 0;
    const int ll = which ? 6 : 10;
    const int len = 2 + ll + 4 + 32;
    absorb(A, par, len, [&](int k) -> uint8_t {
      if (k < 2) return (uint8_t)(ll >> (8 * k));
      k -= 2;
      if (k < ll) return (uint8_t)(which ? "offset"[k] : "multiplier"[k]);
      k -= ll;
      if (k < 4) return (uint8_t)(32u >> (8 * k));
      k -= 4;
      return (uint8_t)(S[k >> 3] >> (8 * (k & 7)));
    });
  }
  // squeeze ceil(n/8) bytes, masked to n bits; c |= 1.  Of each lane pair
  // (2q, 2q+1) of the output block, the e thread writes lane 2q, the o thread 2q+1.
  const long long nb = (n_bits + 7) >> 3;
  const int top = (int)(n_bits & 7);
  const uint8_t topmask = top ? (uint8_t)((1u << top) - 1u) : (uint8_t)0xFF;
  uint8_t* row = (which ? d : c) + (long long)j * stride;
  for (long long base = 0; base < nb; base += kRate) {
    if (base) keccak_f2(A, par);
    const long long rem = nb - base;
    uint64_t W[9];  // lanes 2q + par, q < 9 (lane 17 does not exist)
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const uint32_t mine = par ? (2 * q + 1 < kRateW ? A[2 * q + 1] : 0u) : A[2 * q];
      const uint32_t give = par ? A[2 * q] : (2 * q + 1 < kRateW ? A[2 * q + 1] : 0u);
      const uint32_t got = __shfl_xor_sync(kFull, give, 1);
      W[q] = par ? zip(got, mine) : zip(mine, got);
    }
    if (!active) continue;
    if (word_io && rem >= kRate) {  // LSF, 8-byte aligned row: whole lanes
      uint64_t* o = reinterpret_cast<uint64_t*>(row + base);
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (2 * q + (int)par < kRateW) o[2 * q + par] = W[q];
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int w = 2 * q + (int)par;
#pragma unroll
        for (int b8 = 0; b8 < 8; ++b8) {
          const long long k = base + 8 * w + b8;
          if (w < kRateW && k < nb) {
            uint8_t b = (uint8_t)(W[q] >> (8 * b8));
            if (k == nb - 1) b &= topmask;
            if (k == 0 && !which) b |= 1u;
            row[msf ? nb - 1 - k : k] = b;
          }
        }
      }
    }
  }
  if (active && word_io && nb >= kRate) {  // first / last byte written as whole lanes
    if (!which && par == 0) row[0] |= 1u;                  // lane 0: the e thread
    if (nb % kRate == 0 && par == 0) row[nb - 1] &= topmask;  // lane 16: the e thread
  }
}

}  // namespace

// (pa_kernels.cu's launch_seed_expand wraps this with the profiling scope)
void seed_expand_raw(const SeedMaster& master, int mlen, unsigned long long first, int batch,
                     long long n_bits, int msf, int word_io, uint8_t* c, uint8_t* d,
                     long long stride, cudaStream_t st, long long fixed_index) {
  const int threads = 4 * batch;  // a lane pair per XOF stream, two streams per block
  const int per = 64;  // two warps per CTA: the few streams spread over the SMs
  const dim3 grid((threads + per - 1) / per);
  k_seed_expand<<<grid, per, 0, st>>>(master, mlen, first, batch, n_bits, msf, word_io, c, d,
                                      stride, fixed_index);
}

}  // namespace pab
