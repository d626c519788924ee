// CUDA kernels for the modular-hash PA pipeline on sm_100a.
//
// Pipeline per block (reference path: compress -> fused_mul_add -> mul ->
// ssa_multiply -> mod_pow2 -> shift_right, pkg/src/modpa/pa.py:175-190,
// pkg/src/modpa/bignum.py:161-238, pkg/src/modpa/ntt.py:270-284):
//   k_col_fwd  column DIF pass of the four-step NTT, reading the operands'
//              32-bit words straight from the serialized blocks (import_block /
//              split, pa.py:111-125, ntt.py:111-120; forward_ntt ntt.py:209-212)
//   k_row      row pass: four-step twiddle, DIF of c and x, pointwise product,
//              DIT, inverse twiddle (pointwise_mul, ntt.py:225-243)
//   k_col_inv  column DIT pass + 1/L scale -> residues mod p_i (inverse_ntt, ntt.py:215-222)
//   k_carry    CRT + overlap-add + "+d" + carry-lookahead scan + mod 2^n + >> (n-r),
//              writing the key bytes (combine_and_carry ntt.py:246-267, fused_mul_add
//              bignum.py:238, mod_pow2 bignum.py:161-165, shift_right bignum.py:168-172,
//              export_block pa.py:128-132)
//   k_pack / k_unpack  only for MSF or unaligned layouts.
// For L <= 4096 a single k_row CTA per (block, prime) does the whole transform.
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "conv_kernels.cuh"

namespace pab {

// ---------------------------------------------------------------------------
// Optional per-kernel event timing (pab_profile_*): events are recorded on the
// launching stream around every kernel while enabled.
namespace prof {
struct Rec {
  const char* name;
  cudaEvent_t a, b;
};
static std::mutex mu;
static bool on = false;
static std::vector<Rec> recs;
static std::vector<cudaEvent_t> pool;
static cudaEvent_t get_ev() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct Scope {
  bool active;
  Rec r;
  cudaStream_t st;
  Scope(const char* name, cudaStream_t s) : active(false), st(s) {
    std::lock_guard<std::mutex> lk(mu);
    if (!on) return;
    active = true;
    r.name = name;
    r.a = get_ev();
    r.b = get_ev();
    cudaEventRecord(r.a, st);
  }
  ~Scope() {
    if (!active) return;
    cudaEventRecord(r.b, st);
    std::lock_guard<std::mutex> lk(mu);
    recs.push_back(r);
  }
};
}  // namespace prof

void profile_enable(bool enable) {
  std::lock_guard<std::mutex> lk(prof::mu);
  prof::on = enable;
}
// Aggregates by kernel name: returns number of distinct names written.
int profile_collect(const char** names, int* counts, double* ms, int cap) {
  std::lock_guard<std::mutex> lk(prof::mu);
  int nn = 0;
  for (auto& r : prof::recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    int i = 0;
    while (i < nn && std::string(names[i]) != r.name) ++i;
    if (i == nn) {
      if (nn == cap) continue;
      names[nn] = r.name;
      counts[nn] = 0;
      ms[nn] = 0.0;
      ++nn;
    }
    counts[i] += 1;
    ms[i] += t;
    prof::pool.push_back(r.a);
    prof::pool.push_back(r.b);
  }
  prof::recs.clear();
  return nn;
}

void launch_seed_expand(const SeedMaster& master, int mlen, unsigned long long first, int batch,
                        long long n_bits, int msf, int word_io, uint8_t* c, uint8_t* d,
                        long long stride, cudaStream_t st, long long fixed_index) {
  prof::Scope ps_("k_seed_expand", st);
  seed_expand_raw(master, mlen, first, batch, n_bits, msf, word_io, c, d, stride, st,
                  fixed_index);
}

// ---------------------------------------------------------------------------
// pack / unpack (MSF byte order or unaligned blocks only)

__global__ void k_pack(const uint8_t* __restrict__ in, long long in_stride, long long n_bits,
                       int msf, u32* __restrict__ words, long long word_stride, long long kw) {
  const int b = blockIdx.y;
  const uint8_t* src = in + (long long)b * in_stride;
  u32* dst = words + (long long)b * word_stride;
  const long long nbytes = (n_bits + 7) >> 3;
  const long long kn = (n_bits + 31) >> 5;
  // whole 4-byte words in place (LSF) or byte-reversed (MSF) when the row allows
  const bool a4 = ((reinterpret_cast<uintptr_t>(src) & 3) == 0) && (msf ? (nbytes & 3) == 0 : true);
  const long long kfull = nbytes >> 2;  // words made only of input bytes
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < kw;
       j += (long long)gridDim.x * blockDim.x) {
    u32 w = 0;
    if (a4 && j < kfull) {
      const u32* s32 = reinterpret_cast<const u32*>(src);
      w = msf ? __byte_perm(__ldg(s32 + (kfull - 1 - j)), 0u, 0x0123) : __ldg(s32 + j);
      if (j == kn - 1 && (n_bits & 31)) w &= (1u << (n_bits & 31)) - 1u;
    } else if (j < kn) {
      const long long q0 = 4 * j;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long bi = q0 + q;
        if (bi < nbytes) {
          const u32 byte = msf ? src[nbytes - 1 - bi] : src[bi];
          w |= byte << (8 * q);
        }
      }
      if (j == kn - 1 && (n_bits & 31)) w &= (1u << (n_bits & 31)) - 1u;
    }
    dst[j] = w;
  }
}

__global__ void k_unpack(const u32* __restrict__ words, long long word_stride, long long m_bits,
                         int msf, uint8_t* __restrict__ out, long long out_stride) {
  const int b = blockIdx.y;
  const u32* src = words + (long long)b * word_stride;
  uint8_t* dst = out + (long long)b * out_stride;
  const long long mb = (m_bits + 7) >> 3;
  if (!msf && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {  // whole words where possible
    const long long mw4 = mb >> 2;
    u32* d32 = reinterpret_cast<u32*>(dst);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mw4;
         q += (long long)gridDim.x * blockDim.x)
      d32[q] = src[q];
    for (long long q = 4 * mw4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mb;
         q += (long long)gridDim.x * blockDim.x)
      dst[q] = (uint8_t)(src[q >> 2] >> (8 * (q & 3)));
    return;
  }
  if (!msf && (reinterpret_cast<uintptr_t>(dst) & 1) == 0) {  // 2-byte aligned rows: halves
    const long long mh = mb >> 1;
    uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mh;
         q += (long long)gridDim.x * blockDim.x)
      d16[q] = (uint16_t)(src[q >> 1] >> (16 * (q & 1)));
    if ((mb & 1) && blockIdx.x == 0 && threadIdx.x == 0)
      dst[mb - 1] = (uint8_t)(src[(mb - 1) >> 2] >> (8 * ((mb - 1) & 3)));
    return;
  }
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mb;
       q += (long long)gridDim.x * blockDim.x) {
    const uint8_t byte = (uint8_t)(src[q >> 2] >> (8 * (q & 3)));
    dst[msf ? (mb - 1 - q) : q] = byte;
  }
}

// ---------------------------------------------------------------------------
// CPython integer digits <-> words (the drop-in's Python-int boundary)
//
// A CPython int holds its magnitude as 30-bit digits in 32-bit slots, least
// significant first (sys.int_info: bits_per_digit 30).  The drop-in hands the
// digit arrays of BitBlock.value / HashSeed.c / HashSeed.d straight to the GPU
// and receives the key as digits, instead of int.to_bytes / int.from_bytes on
// the host (pkg/src/modpa/pa.py:175-190 converts nothing: its ints are the data).

// word j of operand y = bits [32j, 32j + 32): digits i0 = 32j / 30 and i0 + 1
__global__ void k_digits_pack(DigitOperands ops, long long n_bits, u32* __restrict__ words,
                              long long word_stride, long long kw) {
  const int y = blockIdx.y;
  const u32* __restrict__ dig = ops.d[y];
  const long long nd = ops.nd[y];
  u32* dst = words + (long long)y * word_stride;
  const long long kn = (n_bits + 31) >> 5;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < kw;
       j += (long long)gridDim.x * blockDim.x) {
    u32 w = 0;
    if (j < kn) {
      const long long b0 = 32 * j;
      const long long i0 = b0 / 30;
      const int o = (int)(b0 - 30 * i0);  // even, 0 .. 28
      const u32 lo = i0 < nd ? __ldg(dig + i0) : 0u;
      const u32 hi = i0 + 1 < nd ? __ldg(dig + i0 + 1) : 0u;
      w = (lo >> o) | (hi << (30 - o));
      if (j == kn - 1 && (n_bits & 31)) w &= (1u << (n_bits & 31)) - 1u;
    }
    dst[j] = w;
  }
}

// digit i of an m-bit LSF key = bits [30i, 30i + 30) of its words (bits >= m cleared)
__global__ void k_digits_unpack(const u32* __restrict__ words, long long m_bits,
                                u32* __restrict__ dig, long long nd) {
  const long long mw = (m_bits + 31) >> 5;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nd;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b0 = 30 * i;
    const long long w0 = b0 >> 5;
    const int off = (int)(b0 & 31);
    u32 v = w0 < mw ? __ldg(words + w0) >> off : 0u;
    if (off > 2 && w0 + 1 < mw) v |= __ldg(words + w0 + 1) << (32 - off);
    v &= 0x3FFFFFFFu;
    const long long left = m_bits - b0;
    if (left < 30) v = left <= 0 ? 0u : (v & ((1u << left) - 1u));
    dig[i] = v;
  }
}

void launch_digits_pack(const DigitOperands& ops, int nops, long long n_bits, u32* words,
                        long long word_stride, long long kw, cudaStream_t st) {
  const int threads = 256;
  long long gx = (kw + threads - 1) / threads;
  if (gx > 4096) gx = 4096;
  if (gx < 1) gx = 1;
  prof::Scope ps_("k_digits_pack", st);
  k_digits_pack<<<dim3((unsigned)gx, nops), threads, 0, st>>>(ops, n_bits, words, word_stride, kw);
}

void launch_digits_unpack(const u32* words, long long m_bits, u32* dig, long long nd,
                          cudaStream_t st) {
  const int threads = 256;
  long long gx = (nd + threads - 1) / threads;
  if (gx > 4096) gx = 4096;
  if (gx < 1) gx = 1;
  prof::Scope ps_("k_digits_unpack", st);
  k_digits_unpack<<<(unsigned)gx, threads, 0, st>>>(words, m_bits, dig, nd);
}

void launch_pack(const uint8_t* in, long long in_stride_bytes, long long n_bits, int msf,
                 int batch, u32* words, long long word_stride, long long kw, cudaStream_t st) {
  const int threads = 256;
  long long gx = (kw + threads - 1) / threads;
  if (gx > 4096) gx = 4096;
  if (gx < 1) gx = 1;
  prof::Scope ps_("k_pack", st);
  k_pack<<<dim3((unsigned)gx, batch), threads, 0, st>>>(in, in_stride_bytes, n_bits, msf, words,
                                                        word_stride, kw);
}

void launch_unpack(const u32* words, long long word_stride, long long m_bits, int msf, int batch,
                   uint8_t* out, long long out_stride_bytes, cudaStream_t st) {
  const int threads = 256;
  const long long mb = (m_bits + 7) >> 3;
  long long gx = (mb + threads - 1) / threads;
  if (gx > 4096) gx = 4096;
  if (gx < 1) gx = 1;
  prof::Scope ps_("k_unpack", st);
  k_unpack<<<dim3((unsigned)gx, batch), threads, 0, st>>>(words, word_stride, m_bits, msf, out,
                                                          out_stride_bytes);
}

// ---------------------------------------------------------------------------
// Carry: CRT of the residues, overlap-add of the 160-bit (cw = 2) or 96-bit
// (cw = 1) coefficients at 64/32-bit stride, + D, carry-lookahead scan (decoupled look-back across tiles),
// mask to n_mod_bits, shift right, write the key.

struct CarryFn {  // c -> q + (c >= t); id marks the identity
  u32 q, t;
  bool id;
};
constexpr u32 kInf = 0xFFFFFFFFu;

__device__ __forceinline__ CarryFn cf_compose(CarryFn outer, CarryFn inner) {
  if (outer.id) return inner;
  if (inner.id) return outer;
  CarryFn r;
  r.id = false;
  r.q = outer.q + (inner.q >= outer.t ? 1u : 0u);
  r.t = (inner.q + 1u == outer.t) ? inner.t : kInf;
  return r;
}
__device__ __forceinline__ u32 cf_apply(CarryFn f, u32 c) {
  return f.id ? c : f.q + (c >= f.t ? 1u : 0u);
}

// CRT by Garner's mixed radix, all constants compile-time (SASS immediates):
// v_0 = r_0, v_i = (...((r_i - v_0) p_0^-1 - v_1) p_1^-1 ... - v_{i-1}) p_{i-1}^-1 mod p_i,
// x = v_0 + p_0 (v_1 + p_1 (v_2 + ...)).  Lazy values stay in [0, 2 p_i).
template <int I, int J>
struct Garner {  // p_J^-1 mod p_I with its Shoup companion
  static constexpr u32 w = cpow(kPrimes[J] % kPrimes[I], kPrimes[I] - 2, kPrimes[I]);
  static constexpr u32 wp = cshoup(w, kPrimes[I]);
};

template <int NP>
__device__ __forceinline__ void garner(const u32 (&r)[NP], u32 (&v)[NP]) {
  v[0] = r[0];
  sfor<NP - 1>([&](auto im1) {
    constexpr int I = decltype(im1)::value + 1;
    constexpr u32 p = kPrimes[I];
    u32 t = r[I];
    sfor<I>([&](auto jc) {
      constexpr int J = decltype(jc)::value;
      t = shoup(t + 2u * p - v[J], Garner<I, J>::w, Garner<I, J>::wp, p);  // 2p > v_J
    });
    v[I] = red(t, p);
  });
}

// Mixed-radix reconstruction x = v0 + p0 (v1 + p1 (v2 + ...)) in 32-bit limbs:
// every step is limb * p + (addend) < 2^62, one IMAD.WIDE.U32 each.
// three primes (cw = 1): x < 2^90 -> 3 words
__device__ __forceinline__ void crt3(u32 r0, u32 r1, u32 r2, u32& w0, u32& w1, u32& w2) {
  const u32 r[3] = {r0, r1, r2};
  u32 v[3];
  garner<3>(r, v);
  constexpr u32 p0 = kPrimes[0], p1 = kPrimes[1];
  u64 t = (u64)v[2] * p1 + v[1];  // < 2^60
  const u32 a0 = (u32)t, a1 = (u32)(t >> 32);
  t = (u64)a0 * p0 + v[0];
  w0 = (u32)t;
  t = (u64)a1 * p0 + (t >> 32);
  w1 = (u32)t;
  w2 = (u32)(t >> 32);
}

// five primes (cw = 2): x < 2^149 -> 5 words
__device__ __forceinline__ void crt5(const u32 (&r)[5], u32 (&w)[5]) {
  u32 v[5];
  garner<5>(r, v);
  constexpr u32 p0 = kPrimes[0], p1 = kPrimes[1], p2 = kPrimes[2], p3 = kPrimes[3];
  u64 t = (u64)v[4] * p3 + v[3];  // a = v3 + p3 v4 < 2^60
  const u32 a0 = (u32)t, a1 = (u32)(t >> 32);
  t = (u64)a0 * p2 + v[2];  // b = v2 + p2 a < 2^90
  const u32 b0 = (u32)t;
  t = (u64)a1 * p2 + (t >> 32);
  const u32 b1 = (u32)t, b2 = (u32)(t >> 32);
  t = (u64)b0 * p1 + v[1];  // c = v1 + p1 b < 2^120
  const u32 c0 = (u32)t;
  t = (u64)b1 * p1 + (t >> 32);
  const u32 c1 = (u32)t;
  t = (u64)b2 * p1 + (t >> 32);
  const u32 c2 = (u32)t, c3 = (u32)(t >> 32);
  t = (u64)c0 * p0 + v[0];  // x = v0 + p0 c < 2^150
  w[0] = (u32)t;
  t = (u64)c1 * p0 + (t >> 32);
  w[1] = (u32)t;
  t = (u64)c2 * p0 + (t >> 32);
  w[2] = (u32)t;
  t = (u64)c3 * p0 + (t >> 32);
  w[3] = (u32)t;
  w[4] = (u32)(t >> 32);
}

__device__ __forceinline__ u32 fetch_word(const u32* __restrict__ src, long long gi, long long kv,
                                          u32 mask) {
  if (gi >= kv) return 0u;
  const u32 w = __ldg(src + gi);
  return gi == kv - 1 ? (w & mask) : w;
}

struct CarrySmem {
  u32 tile, cin;
  volatile u32 cin_ready;  // look-back mode: sm.cin valid (set by warp 0)
  u32 wq[kCarryWarps], wt[kCarryWarps];
  u32 first[kCarryWarps];  // each warp's first word, resolved with carry-in 0
  // cw = 2: high words of each warp's top two coefficients for the warp above
  // (w2, w3 of lane 31, w4 of lanes 30 and 31), double-buffered by tile parity
  u32 nb[2][kCarryWarps][4];
};

// Column sums of one warp's kCarryRows x 32 words starting at word wb:
// S[i] (lane j) = sum of the CRT'd coefficient words landing on word wb + 32 i + j.
// s_next (warp-uniform `last` only): the same sum for word wb + 32 kCarryRows.
//
// cw = 1: coefficient k (3 words) lands on words k, k+1, k+2.
__device__ __forceinline__ void sums_cw1(const u32* __restrict__ res, long long L, long long nres,
                                         long long wb, bool last, u64 (&S)[kCarryRows],
                                         u64& s_next) {
  constexpr int NR = kCarryRows;
  const int lane = threadIdx.x & 31;
  const u32* res0 = res;
  const u32* res1 = res + L;
  const u32* res2 = res + 2 * L;
  // issue every load first (memory-level parallelism), then CRT
  u32 V0[NR], V1[NR], V2[NR];
  const bool in_res = wb + NR * 32 <= nres;
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const long long k = wb + i * 32 + lane;
    const bool ok = in_res || k < nres;
    V0[i] = ok ? __ldg(res0 + k) : 0u;
    V1[i] = ok ? __ldg(res1 + k) : 0u;
    V2[i] = ok ? __ldg(res2 + k) : 0u;
  }
  // virtual row -1 (lanes 30, 31 hold coefficients wb-2, wb-1)
  u32 P1 = 0, P2 = 0;
  {
    const long long k = wb - 32 + lane;
    const bool ok = lane >= 30 && k >= 0 && k < nres;
    const u32 q0 = ok ? __ldg(res0 + k) : 0u, q1 = ok ? __ldg(res1 + k) : 0u,
              q2 = ok ? __ldg(res2 + k) : 0u;
    u32 x0;
    crt3(q0, q1, q2, x0, P1, P2);
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) crt3(V0[i], V1[i], V2[i], V0[i], V1[i], V2[i]);
  // S_k = V0[k] + V1[k-1] + V2[k-2]  (zero residues CRT to zero)
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const u32 p1row = i ? V1[i - 1] : P1, p2row = i ? V2[i - 1] : P2;
    const u32 a1 = __shfl_up_sync(0xFFFFFFFFu, V1[i], 1);
    const u32 b1 = __shfl_sync(0xFFFFFFFFu, p1row, 31);
    const u32 a2 = __shfl_up_sync(0xFFFFFFFFu, V2[i], 2);
    const u32 b2 = __shfl_sync(0xFFFFFFFFu, p2row, 30 + (lane & 1));
    S[i] = (u64)V0[i] + (lane ? a1 : b1) + (lane >= 2 ? a2 : b2);
  }
  if (last) {
    const long long k = wb + NR * 32;
    u32 n0 = 0, n1, n2;
    if (lane == 0 && k < nres) crt3(__ldg(res0 + k), __ldg(res1 + k), __ldg(res2 + k), n0, n1, n2);
    n0 = __shfl_sync(0xFFFFFFFFu, n0, 0);
    const u32 v1 = __shfl_sync(0xFFFFFFFFu, V1[NR - 1], 31);
    const u32 v2 = __shfl_sync(0xFFFFFFFFu, V2[NR - 1], 30);
    s_next = (u64)n0 + v1 + v2;
  }
}

// cw = 2: coefficient c (5 words) lands on words 2c .. 2c+4, so even word 2c
// sums w0(c) + w2(c-1) + w4(c-2) and odd word 2c+1 sums w1(c) + w3(c-1).
// A pair of rows (64 words) is 32 coefficients: lane j CRTs coefficient
// cb + 32 q + j, then shuffles route the words.  In the sequential mode the
// two coefficients below a warp come from the warp beneath through shared
// memory (the previous tile's top warp for warp 0; contains a __syncthreads);
// in the look-back mode each warp recomputes them.
template <bool LOOKBACK>
__device__ __forceinline__ void sums_cw2(const u32* __restrict__ res, long long L, long long nres,
                                         long long wb, int tile, CarrySmem& sm,
                                         u64 (&S)[kCarryRows], u64& s_next) {
  constexpr int NQ = kCarryRows / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool last = warp == kCarryWarps - 1;
  const long long cb = wb >> 1;
  u32 W[NQ][5];
  const bool in_res = cb + NQ * 32 <= nres;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const long long k = cb + q * 32 + lane;
    const bool ok = in_res || k < nres;
#pragma unroll
    for (int i = 0; i < 5; ++i) W[q][i] = ok ? __ldg(res + i * L + k) : 0u;
  }
  u32 nx[5] = {0u, 0u, 0u, 0u, 0u};  // top warp: the next tile's first coefficient (lane 0)
  const long long kn = cb + NQ * 32;
  if (last && lane == 0 && kn < nres) {
#pragma unroll
    for (int i = 0; i < 5; ++i) nx[i] = __ldg(res + i * L + kn);
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) crt5(W[q], W[q]);
  if (last && lane == 0 && kn < nres) crt5(nx, nx);
  // w2(c-1), w3(c-1) from lane 31 and w4(c-2) from lanes 30 / 31 of the pair below
  u32 pw2 = 0, pw3 = 0, pw4a = 0, pw4b = 0;
  if constexpr (LOOKBACK) {  // every warp recomputes them (no barrier: warps stay independent)
    const long long k = cb - 32 + lane;
    const bool ok = lane >= 30 && k >= 0 && k < nres;
    u32 Pv[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) Pv[i] = ok ? __ldg(res + i * L + k) : 0u;
    crt5(Pv, Pv);
    pw2 = __shfl_sync(0xFFFFFFFFu, Pv[2], 31);
    pw3 = __shfl_sync(0xFFFFFFFFu, Pv[3], 31);
    pw4a = __shfl_sync(0xFFFFFFFFu, Pv[4], 30);
    pw4b = __shfl_sync(0xFFFFFFFFu, Pv[4], 31);
  } else {  // from the warp beneath (the previous tile's top warp for warp 0)
    if (lane >= 30) {
      u32* nb = sm.nb[tile & 1][warp];
      if (lane == 31) {
        nb[0] = W[NQ - 1][2];
        nb[1] = W[NQ - 1][3];
        nb[3] = W[NQ - 1][4];
      } else {
        nb[2] = W[NQ - 1][4];
      }
    }
    __syncthreads();
    if (warp > 0 || tile > 0) {
      const u32* nb = warp ? sm.nb[tile & 1][warp - 1] : sm.nb[(tile - 1) & 1][kCarryWarps - 1];
      pw2 = nb[0];
      pw3 = nb[1];
      pw4a = nb[2];
      pw4b = nb[3];
    }
  }
  const bool odd = lane & 1;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sl = 16 * h + (lane >> 1);  // source lane of coefficient c
      const u32 x0 = __shfl_sync(0xFFFFFFFFu, W[q][0], sl);
      const u32 x1 = __shfl_sync(0xFFFFFFFFu, W[q][1], sl);
      u32 y2 = __shfl_sync(0xFFFFFFFFu, W[q][2], (sl - 1) & 31);
      u32 y3 = __shfl_sync(0xFFFFFFFFu, W[q][3], (sl - 1) & 31);
      u32 z4 = __shfl_sync(0xFFFFFFFFu, W[q][4], (sl - 2) & 31);
      if (h == 0) {  // c-1 / c-2 below this pair: lanes 31 / 30 + sl of the previous one
        u32 py2, py3, pz4;
        if (q == 0) {
          py2 = pw2;
          py3 = pw3;
          pz4 = sl == 0 ? pw4a : pw4b;
        } else {
          py2 = __shfl_sync(0xFFFFFFFFu, W[q - 1][2], 31);
          py3 = __shfl_sync(0xFFFFFFFFu, W[q - 1][3], 31);
          pz4 = __shfl_sync(0xFFFFFFFFu, W[q - 1][4], (30 + sl) & 31);
        }
        if (sl == 0) {
          y2 = py2;
          y3 = py3;
        }
        if (sl < 2) z4 = pz4;
      }
      S[2 * q + h] = odd ? (u64)x1 + y3 : (u64)x0 + y2 + z4;
    }
  }
  if (last) {  // word wb + 32 NR = 2 kn: w0(kn) + w2(kn - 1) + w4(kn - 2)
    const u32 n0 = __shfl_sync(0xFFFFFFFFu, nx[0], 0);
    const u32 v2 = __shfl_sync(0xFFFFFFFFu, W[NQ - 1][2], 31);
    const u32 v4 = __shfl_sync(0xFFFFFFFFu, W[NQ - 1][4], 30);
    s_next = (u64)n0 + v2 + v4;
  }
}

// Warp-striped carry: a CTA tile is kCarryWarps * kCarryRows rows of 32 words;
// lane j of warp w holds words tile_base + (w*kCarryRows + i)*32 + j, so every
// load/store of a row is one coalesced 128-byte access.  Within a row, the
// multi-bit carries (< 8) are folded one word up and the remaining 1-bit
// carries resolved with a ballot carry-lookahead: with G = ballot(overflow),
// P = ballot(word == ~0), the carries into all lanes are (A+B)^A^B for
// A = G|P, B = G.  Rows chain sequentially inside the warp; warps and tiles
// compose carry functions c -> q + (c >= t).

// Resolve one row: s = column sums (u64) of this lane's word, cin_row = carry
// into lane 0 (< 2^32).  Returns final word; updates cin_row to the row's
// carry-out (into the next row), computes all-ones ballot.
__device__ __forceinline__ u32 carry_row(u64 s, u32& cin_row, unsigned& ones_mask) {
  const int lane = threadIdx.x & 31;
  const u32 lo = (u32)s, hi = (u32)(s >> 32);
  const u32 hprev = __shfl_up_sync(0xFFFFFFFFu, hi, 1);
  const u32 hlast = __shfl_sync(0xFFFFFFFFu, hi, 31);
  const u32 add = lane ? hprev : cin_row;
  const u32 u = lo + add;
  const bool g = u < lo;
  const unsigned G = __ballot_sync(0xFFFFFFFFu, g);
  const unsigned Pm = __ballot_sync(0xFFFFFFFFu, u == 0xFFFFFFFFu);
  const unsigned A = G | Pm, B = G;
  const u64 sum = (u64)A + B;
  const unsigned carries = ((unsigned)sum ^ A ^ B);
  const u32 kout = (u32)(sum >> 32);
  const u32 t = u + ((carries >> lane) & 1u);
  ones_mask = __ballot_sync(0xFFFFFFFFu, t == 0xFFFFFFFFu);
  cin_row = hlast + kout;
  return t;
}

// One tile of block b; LOOKBACK: carry-in via decoupled look-back, else cin_seq.
// Returns the carry out of the tile.
template <bool LOOKBACK, int CW>
__device__ __forceinline__ u32 carry_tile(const ConvJob& job, CarrySmem& sm, int b, int tile,
                                          u32 cin_seq) {
  constexpr int NR = kCarryRows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long L = job.L;
  const u32* res = job.buf + (long long)b * 2 * job.np * L;  // prime i at res + i * L
  const u32* dw = job.srcD ? job.srcD + (long long)b * job.src_stride : nullptr;
  const long long tbase = (long long)tile * kCarryTile;
  const long long wb = tbase + (long long)warp * NR * 32;  // first word of this warp
  const bool last = warp == kCarryWarps - 1;

  u32 DV[NR];
  const long long kd = dw ? job.kD : 0;
  if (wb + NR * 32 < kd) {
#pragma unroll
    for (int i = 0; i < NR; ++i) DV[i] = __ldg(dw + wb + i * 32 + lane);
  } else {
#pragma unroll
    for (int i = 0; i < NR; ++i) DV[i] = fetch_word(dw, wb + i * 32 + lane, kd, job.maskD);
  }
  u64 S[NR];
  u64 s_next = 0;
  if constexpr (CW == 1) {
    sums_cw1(res, L, job.nRes, wb, last, S, s_next);
  } else {
    sums_cw2<LOOKBACK>(res, L, job.nRes, wb, tile, sm, S, s_next);
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) S[i] += DV[i];
  // resolve the warp's words with carry-in 0 and its carry function
  // c -> q + (c >= t): the extra carry needs word 0 + c to overflow and every
  // other word to be all-ones
  CarryFn f;
  u32 T[NR];
  unsigned ones[NR];
  {
    u32 c = 0;
    bool allones = true;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      T[i] = carry_row(S[i], c, ones[i]);
      allones &= ((i == 0 ? (ones[i] | 1u) : ones[i]) == 0xFFFFFFFFu);
    }
    const u32 first = __shfl_sync(0xFFFFFFFFu, T[0], 0);
    f.id = false;
    f.q = c;
    f.t = (allones && first != 0u) ? (0u - first) : kInf;
  }
  if (lane == 0) {
    sm.wq[warp] = f.q;
    sm.wt[warp] = f.t;
    sm.first[warp] = T[0];
    if (LOOKBACK && warp == 0) sm.cin_ready = 0u;
  }
  __syncthreads();
  CarryFn wpre{0, 0, true}, agg{0, 0, true};
#pragma unroll
  for (int w = 0; w < kCarryWarps; ++w) {
    const CarryFn fw{sm.wq[w], sm.wt[w], false};
    if (w < warp) wpre = cf_compose(fw, wpre);
    agg = cf_compose(fw, agg);
  }
  // carry into the tile.  Only warp 0, and a warp whose predecessors in the tile
  // let a carry through (wpre.t != kInf: all-ones runs, rare), depend on it; the
  // others go on without waiting for the look-back (ncu: 26% barrier stalls).
  u32 tile_cin = cin_seq;
  if (LOOKBACK) {
    if (warp == 0) {  // decoupled look-back: 32 predecessor tiles per probe
      volatile unsigned long long* st = job.tile_state + (long long)b * job.tiles;
      u32 cin = 0;
      if (tile > 0) {
        if (lane == 0) st[tile] = (1ull << 62) | ((unsigned long long)agg.q << 32) | agg.t;
        CarryFn F{0, 0, true};
        int base = tile - 1;
        while (true) {
          const int j = base - lane;
          const unsigned long long v = j >= 0 ? st[j] : (2ull << 62);
          const u32 flag = (u32)(v >> 62);
          const unsigned zero = __ballot_sync(0xFFFFFFFFu, flag == 0);
          const unsigned pre = __ballot_sync(0xFFFFFFFFu, flag == 2);
          const int first = pre ? __ffs(pre) - 1 : 32;
          const unsigned need = first == 32 ? 0xFFFFFFFFu : ((2u << first) - 1u);
          if (zero & need) continue;
          const u32 q = (u32)((v >> 32) & 0xFFu), t = (u32)v;
          for (int i = 0; i < first; ++i) {
            const CarryFn g{__shfl_sync(0xFFFFFFFFu, q, i), __shfl_sync(0xFFFFFFFFu, t, i), false};
            F = cf_compose(F, g);
          }
          if (first < 32) {
            cin = cf_apply(F, __shfl_sync(0xFFFFFFFFu, q, first));
            break;
          }
          base -= 32;
        }
      }
      if (lane == 0) {
        st[tile] = (2ull << 62) | ((unsigned long long)cf_apply(agg, cin) << 32);
        sm.cin = cin;
        __threadfence_block();
        sm.cin_ready = 1u;
      }
      tile_cin = cin;
    } else if (wpre.t != kInf) {
      while (sm.cin_ready == 0u) {
      }
      __threadfence_block();
      tile_cin = *((volatile u32*)&sm.cin);
    }
  }

  // add the real carry-in at word 0 and ripple it through all-ones words
  // (almost always it stops in word 0)
  const u32 cin_w = cf_apply(wpre, tile_cin);
  const u32 c = cf_apply(f, cin_w);  // carry out of the warp
  {
    u32 cr = cin_w;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      if (cr == 0u) break;
      const u32 t0 = __shfl_sync(0xFFFFFFFFu, T[i], 0);
      const bool ov = t0 + cr < cr;
      if (lane == 0) T[i] = t0 + cr;
      if (!ov) break;
      const unsigned stop = ~ones[i] & ~1u;  // lanes >= 1 that absorb the carry
      const int k = stop ? __ffs(stop) - 1 : 32;
      if (lane >= 1 && lane < k) T[i] = 0u;
      if (lane == k) T[i] += 1u;
      cr = k == 32 ? 1u : 0u;
    }
  }
  const long long nT = job.nT;
  const long long rbits = job.n_mod_bits - 32ll * (nT - 1);
  const u32 tmask = rbits >= 32 ? 0xFFFFFFFFu : ((1u << rbits) - 1u);
  if (wb + NR * 32 >= nT) {  // the warp reaches the top word: clear bits >= n_mod_bits
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const long long w = wb + i * 32 + lane;
      T[i] = w >= nT ? 0u : (w == nT - 1 ? (T[i] & tmask) : T[i]);
    }
  }
  // word after this warp's last word: the next warp's first word resolved with
  // carry-in 0, plus this warp's carry out; or (last warp) the next tile's first
  // word = S_next + carry
  u32 nextw;
  {
    const long long k = wb + NR * 32;  // first word after the warp
    if (last) {
      const u32 dv = fetch_word(dw, k, kd, job.maskD);
      nextw = (u32)(s_next + dv + c);
    } else {
      nextw = sm.first[warp + 1] + c;
    }
    nextw = k >= nT ? 0u : (k == nT - 1 ? (nextw & tmask) : nextw);
  }
  // output words y_o = (T >> shift), o = w - shift/32
  const long long ws = job.shift >> 5;
  const int sh = (int)(job.shift & 31);
  uint8_t* outb = job.out_words ? nullptr : job.out_bytes + (long long)b * job.out_stride;
  u32* outw = job.out_words ? job.out_words + (long long)b * job.mw : nullptr;
  const long long o0 = wb - ws;
  const bool out_full = o0 >= 0 && o0 + NR * 32 <= job.mw &&
                        (outw != nullptr || 4 * (o0 + NR * 32) <= job.rbytes);
  if (sh == 0 && out_full) {  // word-aligned shift, whole warp inside the key: plain stores
    u32* ow = outw ? outw : reinterpret_cast<u32*>(outb);
#pragma unroll
    for (int i = 0; i < NR; ++i) ow[o0 + i * 32 + lane] = T[i];
  } else {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const u32 up = __shfl_down_sync(0xFFFFFFFFu, T[i], 1);
      const u32 nx = i + 1 < NR ? T[i + 1] : nextw;
      const u32 wrap = __shfl_sync(0xFFFFFFFFu, nx, 0);
      const u32 hiw = lane < 31 ? up : (i + 1 < NR ? wrap : nextw);
      const long long oj = o0 + i * 32 + lane;
      if (oj >= 0 && oj < job.mw) {
        const u32 y = sh ? ((T[i] >> sh) | (hiw << (32 - sh))) : T[i];
        if (outw) {
          outw[oj] = y;
        } else if (4 * oj + 4 <= job.rbytes) {
          reinterpret_cast<u32*>(outb)[oj] = y;
        } else {
          for (int q = 0; q < 4 && 4 * oj + q < job.rbytes; ++q)
            outb[4 * oj + q] = (uint8_t)(y >> (8 * q));
        }
      }
    }
  }
  const u32 cout = cf_apply(agg, tile_cin);
  if (!LOOKBACK) __syncthreads();  // smem reuse by the next tile (look-back CTAs own one tile)
  return cout;
}

// Decoupled look-back across tiles: one CTA per tile (few, huge blocks).
// Grid (batch, tiles): blocks vary fastest, so the CTAs in flight spread over
// the batch and each look-back finds an inclusive predecessor within a probe or
// two (tile-major order kept ~600 tiles of one block in flight: ncu showed 54%
// barrier stalls behind warp 0's long look-back walks).
template <int CW>
__global__ void __launch_bounds__(kCarryThreads) k_carry_lb(ConvJob job) {
  pdl_enter();
  __shared__ CarrySmem sm;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) sm.tile = atomicAdd(&job.tile_ctr[b], 1u);
  __syncthreads();
  carry_tile<true, CW>(job, sm, b, (int)sm.tile, 0u);
}

// ---------------------------------------------------------------------------
// Wide carry (cw = 2): lane-contiguous coefficient ranges.  Lane l of a warp
// CRTs 8 consecutive coefficients and owns the words of coefficient positions
// cb + 2 .. cb + 9 (cb = its first CRT): their column sums need x_c, x_{c-1},
// x_{c-2}, all in the lane or its upper neighbour (6 shuffles), and its 16
// words resolve with a sequential carry chain in registers.  A warp owns 254
// positions (508 words; lane 31 owns 6) from 256 CRTs, so warps need no
// neighbour CRTs.  Carries cross lanes by a 5-step shuffle scan of carry
// functions c -> q + (c >= t), warps and tiles compose them as in carry_tile
// (decoupled look-back), and each warp stages its words in smem to write the
// shifted key coalesced.  Replaces the warp-striped layout's per-word routing
// shuffles and ballots (~325 -> ~150 instructions per coefficient).
#ifndef PAB_WIDE_CPT
#define PAB_WIDE_CPT 8
#endif
constexpr int kWCpt = PAB_WIDE_CPT;                    // CRTs (positions) per lane
constexpr int kWLw = 2 * kWCpt;                        // words per lane
constexpr int kWPos = 32 * kWCpt - 2;                  // positions a warp owns
constexpr int kWWords = 2 * kWPos;                     // 508 words per warp
#ifndef PAB_WIDE_WARPS
#define PAB_WIDE_WARPS 4
#endif
constexpr int kWWarps = PAB_WIDE_WARPS;                // warps per CTA (one tile)
constexpr int kWThreads = 32 * kWWarps;
constexpr int kWTileWords = kWWarps * kWWords;         // words per tile
constexpr int kWStage = (kWLw + 1) * 32;              // per-warp staging, padded lane stride
static_assert(kWTileWords >= kCarryTileMin, "look-back state is sized for kCarryTileMin tiles");
// (4 coefficients per lane: 64 registers and no spills, but 0.181 vs 0.172 ms at C2)

struct WideSmem {
  u32 tile, cin;
  volatile u32 cin_ready;
  u32 wq[kWWarps], wt[kWWarps];
  u32 first[kWWarps];  // each warp's first word, resolved with carry-in 0
  u32 stage[kWWarps][kWStage];
};

__device__ __forceinline__ u32 res_or0(const u32* __restrict__ res, long long L, int i,
                                       long long k, long long nres) {
  return (k >= 0 && k < nres) ? __ldg(res + i * L + k) : 0u;
}

#ifndef PAB_WIDE_MINB
#define PAB_WIDE_MINB 6
#endif
__global__ void __launch_bounds__(kWThreads, PAB_WIDE_MINB) k_carry_wide(ConvJob job) {
  pdl_enter();
  __shared__ WideSmem sm;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) sm.tile = atomicAdd(&job.tile_ctr[b], 1u);
  __syncthreads();
  const int tile = (int)sm.tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool last = warp == kWWarps - 1;
  const long long L = job.L, nres = job.nRes, nT = job.nT;
  const u32* res = job.buf + (long long)b * 2 * job.np * L;  // prime i at res + i * L
  const u32* dw = job.srcD ? job.srcD + (long long)b * job.src_stride : nullptr;
  const long long kd = dw ? job.kD : 0;
  const long long ps = (long long)tile * (kWWarps * kWPos) + (long long)warp * kWPos;
  const long long cb = ps - 2 + kWCpt * lane;  // first CRT coefficient of this lane
  const long long wb = 2 * ps;             // first word of this warp
  const long long lw = wb + kWLw * lane;     // first word of this lane
  const int nwl = lane == 31 ? kWLw - 4 : kWLw;    // words this lane owns

  // residues -> CRT of coefficients cb .. cb + 7
  u32 X[kWCpt][5];
  if (kWCpt % 4 == 0 && cb >= 0 && cb + kWCpt <= nres && (cb & 3) == 0 && (L & 3) == 0) {
    // 16-byte quads (cb mod 4 is warp-uniform: half the warps)
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint4* rp = reinterpret_cast<const uint4*>(res + i * L + cb);
#pragma unroll
      for (int j = 0; j < kWCpt / 4; ++j) {
        const uint4 v = __ldg(rp + j);
        X[4 * j][i] = v.x;
        X[4 * j + 1][i] = v.y;
        X[4 * j + 2][i] = v.z;
        X[4 * j + 3][i] = v.w;
      }
    }
  } else if (cb >= 0 && cb + kWCpt <= nres) {  // cb is even and L a multiple of 2: 8-byte pairs
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint2* rp = reinterpret_cast<const uint2*>(res + i * L + cb);
#pragma unroll
      for (int j = 0; j < kWCpt / 2; ++j) {
        const uint2 v = __ldg(rp + j);
        X[2 * j][i] = v.x;
        X[2 * j + 1][i] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int j = 0; j < kWCpt; ++j) X[j][i] = res_or0(res, L, i, cb + j, nres);
  }
  // the last warp also needs x_P, P = the next tile's first position (lane 31)
  u32 XP[5] = {0u, 0u, 0u, 0u, 0u};
  const long long P = ps + kWPos;
  if (last && lane == 31 && P < nres) {
#pragma unroll
    for (int i = 0; i < 5; ++i) XP[i] = __ldg(res + i * L + P);
  }
#pragma unroll
  for (int j = 0; j < kWCpt; ++j) crt5(X[j], X[j]);
  if (last && lane == 31 && P < nres) crt5(XP, XP);
  // D words of this lane (loaded after the CRT: fewer live registers)
  u32 DV[kWLw];
  if (lw + kWLw <= kd && (reinterpret_cast<uintptr_t>(dw + lw) & 7) == 0) {
    const uint2* dp = reinterpret_cast<const uint2*>(dw + lw);
#pragma unroll
    for (int w = 0; w < kWCpt; ++w) {
      const uint2 v = __ldg(dp + w);
      DV[2 * w] = v.x;
      DV[2 * w + 1] = v.y;
    }
  } else if (lw + kWLw < kd) {  // 4-byte aligned rows, whole words (the last one is masked)
#pragma unroll
    for (int w = 0; w < kWLw; ++w) DV[w] = __ldg(dw + lw + w);
  } else {
#pragma unroll
    for (int w = 0; w < kWLw; ++w) DV[w] = fetch_word(dw, lw + w, kd, job.maskD);
  }
  // x_{cb+8}[0..3] and x_{cb+9}[0..1] from lane + 1 (its first two coefficients)
  u32 N8[4], N9[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) N8[i] = __shfl_down_sync(0xFFFFFFFFu, X[0][i], 1);
#pragma unroll
  for (int i = 0; i < 2; ++i) N9[i] = __shfl_down_sync(0xFFFFFFFFu, X[1][i], 1);
  // column sums of positions c = cb + 2 + q (q < 8): words 2q, 2q + 1 of the lane
  u32 W[kWLw];
  u32 cq = 0;  // carry out of the lane with carry-in 0
  {
    u64 carry = 0;
#pragma unroll
    for (int q = 0; q < kWCpt; ++q) {
      const int j = q + 2;  // x_c = X[j] (j < 8), N8 (j = 8), N9 (j = 9)
      const u32 c0 = j < kWCpt ? X[j][0] : (j == kWCpt ? N8[0] : N9[0]);
      const u32 c1 = j < kWCpt ? X[j][1] : (j == kWCpt ? N8[1] : N9[1]);
      const u32 m2 = j - 1 < kWCpt ? X[j - 1][2] : N8[2];
      const u32 m3 = j - 1 < kWCpt ? X[j - 1][3] : N8[3];
      const u32 m4 = X[j - 2][4];
      const bool own = lane != 31 || q < kWCpt - 2;
      const u64 se = own ? (u64)c0 + m2 + m4 + DV[2 * q] + carry : 0ull;
      W[2 * q] = (u32)se;
      const u64 so = own ? (u64)c1 + m3 + DV[2 * q + 1] + (se >> 32) : 0ull;
      W[2 * q + 1] = (u32)so;
      carry = own ? (so >> 32) : carry;
    }
    cq = (u32)carry;
  }
  // lane carry function c -> cq + (c >= t): the extra carry needs word 0 + c to
  // overflow and every other owned word to be all-ones
  u32 tq;
  {
    bool ones = true;
#pragma unroll
    for (int w = 1; w < kWLw; ++w) ones &= (w >= nwl) || W[w] == 0xFFFFFFFFu;
    tq = (ones && W[0] != 0u) ? (0u - W[0]) : kInf;
  }
  // warp inclusive scan of the lane functions (lower lanes applied first)
  CarryFn inc{cq, tq, false};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const CarryFn g{__shfl_up_sync(0xFFFFFFFFu, inc.q, d), __shfl_up_sync(0xFFFFFFFFu, inc.t, d),
                    false};
    if (lane >= d) inc = cf_compose(inc, g);
  }
  CarryFn exl{__shfl_up_sync(0xFFFFFFFFu, inc.q, 1), __shfl_up_sync(0xFFFFFFFFu, inc.t, 1), lane == 0};
  const CarryFn f{__shfl_sync(0xFFFFFFFFu, inc.q, 31), __shfl_sync(0xFFFFFFFFu, inc.t, 31), false};
  if (lane == 0) {
    sm.wq[warp] = f.q;
    sm.wt[warp] = f.t;
    sm.first[warp] = W[0];
    if (warp == 0) sm.cin_ready = 0u;
  }
  __syncthreads();
  CarryFn wpre{0, 0, true}, agg{0, 0, true};
#pragma unroll
  for (int w = 0; w < kWWarps; ++w) {
    const CarryFn fw{sm.wq[w], sm.wt[w], false};
    if (w < warp) wpre = cf_compose(fw, wpre);
    agg = cf_compose(fw, agg);
  }
  // carry into the tile (decoupled look-back by warp 0; other warps wait only
  // if their predecessors in the tile let a carry through)
  u32 tile_cin = 0;
  if (warp == 0) {
    volatile unsigned long long* st = job.tile_state + (long long)b * job.tiles;
    u32 cin = 0;
    if (tile > 0) {
      if (lane == 0) st[tile] = (1ull << 62) | ((unsigned long long)agg.q << 32) | agg.t;
      CarryFn F{0, 0, true};
      int base = tile - 1;
      while (true) {
        const int j = base - lane;
        const unsigned long long v = j >= 0 ? st[j] : (2ull << 62);
        const u32 flag = (u32)(v >> 62);
        const unsigned zero = __ballot_sync(0xFFFFFFFFu, flag == 0);
        const unsigned pre = __ballot_sync(0xFFFFFFFFu, flag == 2);
        const int first = pre ? __ffs(pre) - 1 : 32;
        const unsigned need = first == 32 ? 0xFFFFFFFFu : ((2u << first) - 1u);
        if (zero & need) continue;
        const u32 q = (u32)((v >> 32) & 0xFFu), t = (u32)v;
        for (int i = 0; i < first; ++i) {
          const CarryFn g{__shfl_sync(0xFFFFFFFFu, q, i), __shfl_sync(0xFFFFFFFFu, t, i), false};
          F = cf_compose(F, g);
        }
        if (first < 32) {
          cin = cf_apply(F, __shfl_sync(0xFFFFFFFFu, q, first));
          break;
        }
        base -= 32;
      }
    }
    if (lane == 0) {
      st[tile] = (2ull << 62) | ((unsigned long long)cf_apply(agg, cin) << 32);
      sm.cin = cin;
      __threadfence_block();
      sm.cin_ready = 1u;
    }
    tile_cin = cin;
  } else if (wpre.t != kInf) {
    while (sm.cin_ready == 0u) {
    }
    __threadfence_block();
    tile_cin = *((volatile u32*)&sm.cin);
  }
  const u32 cin_w = cf_apply(wpre, tile_cin);
  const u32 cw_out = cf_apply(f, cin_w);    // carry out of the warp
  const u32 cl = cf_apply(exl, cin_w);      // carry into this lane
  // add it at word 0 and ripple through all-ones words (almost always stops at once)
  W[0] += cl;
  if (W[0] < cl) {
    u32 cr = 1u;
#pragma unroll
    for (int w = 1; w < kWLw; ++w) {
      if (w < nwl && cr) {
        W[w] += 1u;
        cr = W[w] == 0u ? 1u : 0u;
      }
    }
  }
  // clear words >= n_mod_bits
  const long long rbits = job.n_mod_bits - 32ll * (nT - 1);
  const u32 tmask = rbits >= 32 ? 0xFFFFFFFFu : ((1u << rbits) - 1u);
  if (wb + kWWords >= nT) {
#pragma unroll
    for (int w = 0; w < kWLw; ++w) {
      const long long g = lw + w;
      W[w] = g >= nT ? 0u : (g == nT - 1 ? (W[w] & tmask) : W[w]);
    }
  }
  // the word after the warp: the next warp's first word + this warp's carry out,
  // or (last warp) the next tile's first word
  u32 nextw;
  {
    const long long k = wb + kWWords;
    if (last) {
      const u32 x1 = __shfl_sync(0xFFFFFFFFu, X[kWCpt - 1][2], 31);  // x_{P-1}[2]
      const u32 x2 = __shfl_sync(0xFFFFFFFFu, X[kWCpt - 2][4], 31);  // x_{P-2}[4]
      const u32 x0 = __shfl_sync(0xFFFFFFFFu, XP[0], 31);
      nextw = x0 + x1 + x2 + fetch_word(dw, k, kd, job.maskD) + cw_out;
    } else {
      nextw = sm.first[warp + 1] + cw_out;
    }
    nextw = k >= nT ? 0u : (k == nT - 1 ? (nextw & tmask) : nextw);
  }
  // stage the warp's words, then write the shifted key coalesced
  u32* sg = sm.stage[warp];
#pragma unroll
  for (int w = 0; w < kWLw; ++w)
    if (w < nwl) sg[(kWLw + 1) * lane + w] = W[w];
  __syncwarp();
  const long long ws = job.shift >> 5;
  const int sh = (int)(job.shift & 31);
  uint8_t* outb = job.out_words ? nullptr : job.out_bytes + (long long)b * job.out_stride;
  u32* outw = job.out_words ? job.out_words + (long long)b * job.mw : nullptr;
  const long long o0 = wb - ws;  // output word of the warp's first word
  if (o0 >= 0 && o0 + kWWords <= job.mw && (outw || 4 * (o0 + kWWords) <= job.rbytes)) {
    // the whole warp inside the key: no bounds, whole words
    u32* ow = outw ? outw : reinterpret_cast<u32*>(outb);
    if (sh == 0) {
#pragma unroll 4
      for (int j = lane; j < kWWords; j += 32) ow[o0 + j] = sg[(kWLw + 1) * (j / kWLw) + (j % kWLw)];
    } else {
#pragma unroll 4
      for (int j = lane; j < kWWords; j += 32) {
        const u32 lo = sg[(kWLw + 1) * (j / kWLw) + (j % kWLw)];
        const u32 hi = j + 1 < kWWords ? sg[(kWLw + 1) * ((j + 1) / kWLw) + ((j + 1) % kWLw)] : nextw;
        ow[o0 + j] = (lo >> sh) | (hi << (32 - sh));
      }
    }
    return;
  }
#pragma unroll 4
  for (int j = lane; j < kWWords; j += 32) {
    const long long oj = o0 + j;
    if (oj < 0 || oj >= job.mw) continue;
    const u32 lo = sg[(kWLw + 1) * (j / kWLw) + (j % kWLw)];
    const u32 hi = j + 1 < kWWords ? sg[(kWLw + 1) * ((j + 1) / kWLw) + ((j + 1) % kWLw)] : nextw;
    const u32 y = sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
    if (outw) {
      outw[oj] = y;
    } else if (4 * oj + 4 <= job.rbytes) {
      reinterpret_cast<u32*>(outb)[oj] = y;
    } else {
      for (int q = 0; q < 4 && 4 * oj + q < job.rbytes; ++q) outb[4 * oj + q] = (uint8_t)(y >> (8 * q));
    }
  }
}

// One CTA per block walking its tiles in order (many blocks): no inter-CTA waits.
template <int CW>
__global__ void __launch_bounds__(kCarryThreads) k_carry_seq(ConvJob job) {
  pdl_enter();
  __shared__ CarrySmem sm;
  const int b = blockIdx.y;
  u32 c = 0;
  for (int tile = 0; tile < job.tiles; ++tile) c = carry_tile<false, CW>(job, sm, b, tile, c);
}


// ---------------------------------------------------------------------------
// Tiny blocks (n <= kTinyBits): one warp per block, low-half schoolbook product
// with 96-bit column sums, + d, sequential carry (<= 64 words), mask, shift,
// serialize.  Used by the host path with mapped pinned memory so a drop-in
// compress() call is one launch + one synchronize (the reference's desk-scale
// tests call compress ~1.6M times at alpha <= 10, pkg/tests/test_acceptance.py:96-128).
__global__ void __launch_bounds__(32) k_tiny(const uint8_t* __restrict__ x,
                                             const uint8_t* __restrict__ c,
                                             const uint8_t* __restrict__ d, long long stride,
                                             int n_bits, int r_bits, int msf,
                                             uint8_t* __restrict__ out, long long out_stride) {
  constexpr int KW = kTinyBits / 32;
  __shared__ u32 sx[KW], sc[KW], sd[KW], st[KW + 1];
  const int b = blockIdx.x, lane = threadIdx.x;
  const int nbytes = (n_bits + 7) >> 3, K = (n_bits + 31) >> 5;
  const uint8_t* px = x + (long long)b * stride;
  const uint8_t* pc = c + (long long)b * stride;
  const uint8_t* pd = d + (long long)b * stride;
  for (int j = lane; j < KW; j += 32) {
    u32 wx = 0, wc = 0, wd = 0;
    if (j < K) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int bi = 4 * j + q;
        if (bi < nbytes) {
          const int src = msf ? nbytes - 1 - bi : bi;
          wx |= (u32)px[src] << (8 * q);
          wc |= (u32)pc[src] << (8 * q);
          wd |= (u32)pd[src] << (8 * q);
        }
      }
      if (j == K - 1 && (n_bits & 31)) {
        const u32 m = (1u << (n_bits & 31)) - 1u;
        wx &= m;
        wc &= m;
        wd &= m;
      }
    }
    sx[j] = wx;
    sc[j] = wc;
    sd[j] = wd;
  }
  __syncwarp();
  // column sums S_k = sum_{i<=k} c_i x_{k-i} + d_k as (lo64, hi32)
  u64 slo[2];
  u32 shi[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = lane + 32 * h;
    u64 lo = 0;
    u32 hi = 0;
    if (k < K) {
      lo = sd[k];
      for (int i = 0; i <= k; ++i) {
        const u64 p = (u64)sc[i] * sx[k - i];
        lo += p;
        hi += (lo < p) ? 1u : 0u;
      }
    }
    slo[h] = lo;
    shi[h] = hi;
  }
  // sequential carry by lane 0 over K words (carry < 2^38)
  __shared__ u64 s_lo[KW];
  __shared__ u32 s_hi[KW];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = lane + 32 * h;
    if (k < KW) {
      s_lo[k] = slo[h];
      s_hi[k] = shi[h];
    }
  }
  __syncwarp();
  if (lane == 0) {
    u64 carry = 0;  // < 2^39
    for (int k = 0; k < K; ++k) {
      const u64 lo = s_lo[k];
      const u64 t = (lo & 0xFFFFFFFFull) + (carry & 0xFFFFFFFFull);
      st[k] = (u32)t;
      carry = (t >> 32) + (lo >> 32) + (carry >> 32) + ((u64)s_hi[k] << 32);
    }
    if (n_bits & 31) st[K - 1] &= (1u << (n_bits & 31)) - 1u;
    st[K] = 0u;
  }
  __syncwarp();
  // y = T >> (n - r): ceil(r/8) bytes
  const int rb = (r_bits + 7) >> 3, shift = n_bits - r_bits;
  uint8_t* po = out + (long long)b * out_stride;
  for (int q = lane; q < rb; q += 32) {
    const int bit = shift + 8 * q;
    const int w = bit >> 5, o = bit & 31;
    u32 v = st[w] >> o;
    if (o > 24 && w + 1 <= K) v |= st[w + 1] << (32 - o);
    u32 byte = v & 0xFFu;
    const int valid = r_bits - 8 * q;  // bits of y in this byte
    if (valid < 8) byte &= (1u << valid) - 1u;
    po[msf ? rb - 1 - q : q] = (uint8_t)byte;
  }
}

void launch_tiny(const uint8_t* x, const uint8_t* c, const uint8_t* d, long long stride, int n_bits,
                 int r_bits, int msf, int batch, uint8_t* out, long long out_stride,
                 cudaStream_t st) {
  prof::Scope ps_("k_tiny", st);
  k_tiny<<<batch, 32, 0, st>>>(x, c, d, stride, n_bits, r_bits, msf, out, out_stride);
}

// ---------------------------------------------------------------------------
// dispatch over compile-time transform sizes

#define PAB_DECL(L) ConvKernels conv_kernels_##L();
PAB_DECL(1) PAB_DECL(2) PAB_DECL(3) PAB_DECL(4) PAB_DECL(5) PAB_DECL(6)
PAB_DECL(7) PAB_DECL(8) PAB_DECL(9) PAB_DECL(10) PAB_DECL(11) PAB_DECL(12)
#undef PAB_DECL

static ConvKernels conv_for(int lg) {
  switch (lg) {
    case 1: return conv_kernels_1();
    case 2: return conv_kernels_2();
    case 3: return conv_kernels_3();
    case 4: return conv_kernels_4();
    case 5: return conv_kernels_5();
    case 6: return conv_kernels_6();
    case 7: return conv_kernels_7();
    case 8: return conv_kernels_8();
    case 9: return conv_kernels_9();
    case 10: return conv_kernels_10();
    case 11: return conv_kernels_11();
    case 12: return conv_kernels_12();
    default: {
      ConvKernels k{};
      return k;
    }
  }
}
static ConvKernel row_kernel(int lg, bool small) {
  const ConvKernels k = conv_for(lg);
  return small ? k.row_small : k.row;
}
static ConvKernel colm_kernel(int m, int lgR, int lgC, bool inv) {
  const int dc = lgC - lgR - 2;
  if (lgR < 3 || lgR > 10 || (m != 3 && m != 5) || dc < 0 || dc > 2 || lgC > 12) return nullptr;
  const ConvKernels k = conv_for(lgR);
  const int i = m == 3 ? 0 : 1;
  return inv ? k.colm_inv[i][dc] : k.colm_fwd[i][dc];
}
static ConvKernel colm_fwd_all_kernel(int m, int lgR, int lgC) {
  const int dc = lgC - lgR - 2;
  if (lgR < 3 || lgR > 10 || (m != 3 && m != 5) || dc < 0 || dc > 2 || lgC > 12) return nullptr;
  return conv_for(lgR).colm_fwd_all[m == 3 ? 0 : 1][dc];
}
static ConvKernel col_fwd_all_kernel(int lgR, int lgC) {
  if (lgR < 6) return nullptr;
  const ConvKernels k = conv_for(lgR);
  if (lgC == lgR) return k.col_fwd_all;
  if (lgC == lgR + 1) return k.col_fwd_all1;
  return nullptr;
}
static ConvKernel col_kernel(int lgR, int lgC, bool inv) {
  if (lgR < 6) return nullptr;
  const ConvKernels k = conv_for(lgR);
  if (lgC == lgR) return inv ? k.col_inv : k.col_fwd;
  if (lgC == lgR + 1) return inv ? k.col_inv1 : k.col_fwd1;
  return nullptr;
}

constexpr unsigned kSMs = 148;  // B200

// Launch a kernel whose predecessor in the stream is another kernel of the same
// hash, as its programmatic dependent when `small` (pdl_enter() in
// conv_kernels.cuh): its launch and prologue overlap the predecessor's tail.
// Only launches of a few blocks gain (one 1e6-bit block: 0.0405 -> 0.0368 ms per
// hash); at full batches the early-resident dependents cost 2-4% (C2 1.647 ->
// 1.676 ms, 16 x 1e8 3.42 -> 3.57 ms), so those launch the ordinary way.
// PAB_PDL=0 / 1 (development switch) forces it off / on for every launch.
template <class... KArgs, class... Args>
static void launch_dep(bool small, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  static const int force = [] {
    const char* e = getenv("PAB_PDL");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool pdl = force < 0 ? small : force != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}

void launch_conv(const ConvJob& job, const PlanTables& tab, cudaStream_t st) {
  const int threads = 256;
  if (job.m == 1 && job.lgR == 0) {
    const size_t sm = (size_t)sm_len(job.lgC) * 2 * 4;
    prof::Scope ps_("k_row_single", st);
    row_kernel(job.lgC, true)<<<dim3(1, job.batch, job.pn), threads, sm, st>>>(job, tab, 0);
    return;
  }
  const long long R = (long long)job.m << job.lgR;
  const int lct = job.m == 1 ? col_lct(job.lgR, job.lgC) : col_lct_rows(R, job.lgC);
  const size_t smc = (size_t)job.m * sm_len(job.lgR) * (1u << lct) * 4;
  ConvKernel cf = job.m == 1 ? col_kernel(job.lgR, job.lgC, false)
                             : colm_kernel(job.m, job.lgR, job.lgC, false);
  ConvKernel ci = job.m == 1 ? col_kernel(job.lgR, job.lgC, true)
                             : colm_kernel(job.m, job.lgR, job.lgC, true);
  // mixed-radix inverse: 512 threads for radix 3 (its 384-task first pass and
  // 512-task fused radix pass), 256 otherwise; the forward pass keeps 256
  // (measured with thread-count overrides in scripts/quick_perf.py runs).
  const int ct_threads = job.m == 3 ? 512 : threads;
  const int cf_threads = threads;
  // Forward column pass: all primes per CTA from one staged operand tile (loads
  // once, reused five times) where measured faster -- pow2 columns up to 2^8,
  // mixed radix up to 2^7 per sub-column; longer columns stage too many rows
  // per CTA (occupancy) and use the per-prime kernel with its L2-chunked grid.
  // Which one exists for a size is fixed at compile time (make_conv_kernels).
  const bool fwd_all = job.m == 1 ? col_fwd_all_kernel(job.lgR, job.lgC) != nullptr
                                  : colm_fwd_all_kernel(job.m, job.lgR, job.lgC) != nullptr;
  const long long kcmax = ((job.kA > job.kX ? job.kA : job.kX) + job.cw - 1) / job.cw;
  const unsigned ctas_all = (1u << (job.lgC - lct)) * 2u * (unsigned)job.batch;
  if (job.m == 1 && fwd_all) {
    const int rows = kcmax <= (job.L >> 1) ? (int)(R >> 1) : (int)R;
    const PassPlan pp = pass_plan(job.lgR);
    const size_t ntw = (size_t)job.np << (pp.slo[0] + pp.rs[0]);  // staged first-pass twiddles
    const size_t sma = smc + (size_t)rows * (1u << lct) * 8 + ntw * 8;
    prof::Scope ps_("k_col_fwd", st);
    // fewer CTAs than two waves' worth of SMs (a few blocks): one prime per CTA
    const unsigned gy = ctas_all < 2 * kSMs ? (unsigned)job.pn : 1u;
    col_fwd_all_kernel(job.lgR, job.lgC)<<<dim3(ctas_all, gy), threads, sma, st>>>(job, tab, lct);
  } else if (job.m > 1 && fwd_all) {
    const int dl = 1;  // half-width tiles: the staged rows fit with 4-5 CTAs per SM (measured)
    const int lcta = lct - dl < 2 ? 2 : lct - dl;
    long long rows = (kcmax + (1ll << job.lgC) - 1) >> job.lgC;
    if (rows > R) rows = R;
    const size_t sma = (size_t)job.m * sm_len(job.lgR) * (1u << lcta) * 4 + (size_t)rows * (1u << lcta) * 8;
    const unsigned ctas = (1u << (job.lgC - lcta)) * 2u * (unsigned)job.batch;
    prof::Scope ps_("k_col_fwd", st);
    const unsigned gy = ctas < 2 * kSMs ? (unsigned)job.pn : 1u;  // as above
    colm_fwd_all_kernel(job.m, job.lgR, job.lgC)<<<dim3(ctas, gy), cf_threads, sma, st>>>(job, tab,
                                                                                          lcta);
  } else {
    prof::Scope ps_("k_col_fwd", st);
    // ~32 MiB of operand words per chunk (L2-resident across the prime sweeps)
    ConvJob jf = job;
    const long long kmax = job.kA > job.kX ? job.kA : job.kX;
    long long chunk = (32ll << 20) / (8 * kmax);
    jf.fwd_chunk = (int)(chunk < 1 ? 1 : (chunk > job.batch ? job.batch : chunk));
    const unsigned ctas = (1u << (job.lgC - lct)) * 2u * (unsigned)job.pn * (unsigned)job.batch;
    cf<<<ctas, cf_threads, smc, st>>>(jf, tab, lct);
  }
  // rows: 4K words of rows (A+X: 8K words) per 128-thread CTA -- the same
  // resident warps as 256-thread CTAs of twice the rows (smem-bound), but
  // twice the independent CTAs per SM to overlap barriers (measured -4..6%)
  // rows of up to 256 points: 8 rows per 64-thread CTA (C2 k_row -1%); longer
  // rows: 4K words per 128-thread CTA (8 rows / 64 threads loses 1-2% at 2^9+)
  const bool narrow = job.lgC <= 8;
  int lnr = 12 - job.lgC - (narrow ? 1 : 0);
  if (lnr < 0) lnr = 0;
  if (lnr > job.lgR) lnr = job.lgR;
  const size_t smr = (size_t)sm_len(job.lgC) * (2u << lnr) * 4;
  {
    prof::Scope ps_("k_row", st);
    const ConvKernel rt = tab.tw4 ? conv_for(job.lgC).row_tw4 : nullptr;
    const ConvKernel rk = rt ? rt : row_kernel(job.lgC, false);
    // a few blocks (under two waves of CTAs): 256 threads per CTA, so each CTA's
    // passes finish in fewer task rounds (latency rather than throughput)
    const long long ctas = (long long)job.batch * (R >> lnr) * job.pn;
    const int rthreads = ctas < 2 * (long long)kSMs ? 256 : (narrow ? 64 : 128);
    launch_dep(ctas < 2 * (long long)kSMs, rk, dim3(job.batch, (unsigned)(R >> lnr), job.pn),
               dim3(rthreads), smr, st, job, tab, lnr);
  }
  {
    prof::Scope ps_("k_col_inv", st);
    // pow2 inverse: half-width tiles in 128-thread CTAs while >= 32 columns wide
    // (same resident warps, more independent CTAs; measured -1.5%)
    const int lci = job.m == 1 ? col_inv_lct(job.lgR, job.lgC) : lct;
    const int xi = lct - lci;
    const size_t smi = (size_t)job.m * sm_len(job.lgR) * (1u << lci) * 4;
    const long long ctas = ((long long)job.batch * job.pn) << (job.lgC - lci);
    launch_dep(ctas < 2 * (long long)kSMs, ci, dim3(1u << (job.lgC - lci), job.batch, job.pn),
               dim3(ct_threads >> xi), smi, st, job, tab, lci);
  }
}

bool conv_supported(int m, int lgR, int lgC) {
  if (m == 1 && lgR == 0) return row_kernel(lgC, true) != nullptr;
  const ConvKernel cf = m == 1 ? col_kernel(lgR, lgC, false) : colm_kernel(m, lgR, lgC, false);
  const ConvKernel ca = m == 1 ? col_fwd_all_kernel(lgR, lgC) : colm_fwd_all_kernel(m, lgR, lgC);
  const ConvKernel ci = m == 1 ? col_kernel(lgR, lgC, true) : colm_kernel(m, lgR, lgC, true);
  return (cf != nullptr || ca != nullptr) && ci != nullptr && row_kernel(lgC, false) != nullptr;
}

void launch_carry(const ConvJob& job, cudaStream_t st) {
  prof::Scope ps_("k_carry", st);
  static const int force = [] {  // development override: PAB_CARRY_MODE=seq|lb|wide
    const char* e = getenv("PAB_CARRY_MODE");
    return e ? (e[0] == 's' ? 1 : e[0] == 'l' ? 2 : 0) : 0;
  }();
  // (the workspace holds look-back states for tiles of kCarryTileMin words;
  // each kernel indexes them with its own tile count)
  if (job.cw == 2 && force != 1 && force != 2) {  // wide layout (PAB_CARRY_MODE=seq|lb: the old ones)
    ConvJob jw = job;
    jw.tiles = (int)((job.nT + kWTileWords - 1) / kWTileWords);
    launch_dep((long long)job.batch * jw.tiles < 2 * (long long)kSMs, k_carry_wide,
               dim3(job.batch, jw.tiles), dim3(kWThreads), 0, st, jw);
    return;
  }
  ConvJob jo = job;
  jo.tiles = (int)((job.nT + kCarryTile - 1) / kCarryTile);
  // look-back everywhere (batch-major grid, measured faster than one CTA per
  // block walking its tiles even at 1024 blocks); sequential for one-tile blocks
  const bool seq = jo.tiles == 1 || force == 1;
  const dim3 grid = seq ? dim3(1, jo.batch) : dim3(jo.batch, jo.tiles);
  if (jo.cw == 2) {
    if (seq) k_carry_seq<2><<<grid, kCarryThreads, 0, st>>>(jo);
    else k_carry_lb<2><<<grid, kCarryThreads, 0, st>>>(jo);
  } else {
    if (seq) k_carry_seq<1><<<grid, kCarryThreads, 0, st>>>(jo);
    else k_carry_lb<1><<<grid, kCarryThreads, 0, st>>>(jo);
  }
}

// Opt every dynamic-smem kernel into > 48 KB once per device.
void set_kernel_attrs() {
  for (int lg = 1; lg <= 12; ++lg) {
    for (int s = 0; s < 2; ++s) {
      ConvKernel k = row_kernel(lg, s != 0);
      if (k) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      for (int dc = 0; dc < 2; ++dc) {
        ConvKernel c = col_kernel(lg, lg + dc, s != 0);
        if (c) cudaFuncSetAttribute(c, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        ConvKernel a = s ? nullptr : col_fwd_all_kernel(lg, lg + dc);
        if (a) cudaFuncSetAttribute(a, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }
      for (int m = 3; m <= 5; m += 2)
        for (int dc = 2; dc <= 4; ++dc) {
          ConvKernel c = colm_kernel(m, lg, lg + dc, s != 0);
          if (c) cudaFuncSetAttribute(c, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
          ConvKernel a = s ? nullptr : colm_fwd_all_kernel(m, lg, lg + dc);
          if (a) cudaFuncSetAttribute(a, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        }
    }
  }
}

}  // namespace pab
