// CUDA kernels for the modular-hash PA pipeline on sm_100a.
//
// Pipeline per block (reference path: compress -> fused_mul_add -> mul ->
// ssa_multiply -> mod_pow2 -> shift_right, pkg/src/modpa/pa.py:175-190,
// pkg/src/modpa/bignum.py:161-238, pkg/src/modpa/ntt.py:270-284):
//   k_pack      bytes -> 32-bit words (import_block/split, pa.py:111-125, ntt.py:111-120)
//   k_col_fwd   column DIF pass of the four-step NTT (forward_ntt, ntt.py:209-212)
//   k_row       row twiddle + DIF, pointwise product, DIT + twiddle (pointwise_mul, ntt.py:225-243)
//   k_col_inv   column DIT pass + 1/L scale -> residues mod p_i (inverse_ntt, ntt.py:215-222)
//   k_carry     CRT + overlap-add + "+d" + carry-lookahead scan + mod 2^n + >> (n-r)
//               (combine_and_carry ntt.py:246-267, fused_mul_add bignum.py:238,
//                mod_pow2 bignum.py:161-165, shift_right bignum.py:168-172)
//   k_unpack    words -> ceil(r/8) bytes (export_block, pa.py:128-132)
#include "pa_kernels.cuh"
#include "ntt_panel.cuh"

#include <mutex>
#include <string>
#include <vector>

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

__constant__ PrimeInfo c_primes[kNumPrimes];
__constant__ CrtConst c_crt;

void upload_constants(const PrimeInfo* primes, const CrtConst& crt) {
  cudaMemcpyToSymbol(c_primes, primes, sizeof(PrimeInfo) * kNumPrimes);
  cudaMemcpyToSymbol(c_crt, &crt, sizeof(CrtConst));
}

__device__ __forceinline__ int brev(int x, int bits) {
  return bits == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - bits));
}

// ---------------------------------------------------------------------------
// pack / unpack

__global__ void k_pack(const uint8_t* __restrict__ in, long long in_stride, long long n_bits,
                       int msf, u32* __restrict__ words, long long word_stride, long long kw) {
  const int b = blockIdx.y;
  const uint8_t* src = in + (long long)b * in_stride;
  u32* dst = words + (long long)b * word_stride;
  const long long nbytes = (n_bits + 7) >> 3;
  const long long kn = (n_bits + 31) >> 5;
  const bool aligned = !msf && ((reinterpret_cast<uintptr_t>(src) & 3) == 0);
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < kw;
       j += (long long)gridDim.x * blockDim.x) {
    u32 w = 0;
    if (j < kn) {
      const long long q0 = 4 * j;
      if (aligned && q0 + 4 <= nbytes) {
        w = reinterpret_cast<const u32*>(src)[j];
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long bi = q0 + q;
          if (bi < nbytes) {
            const u32 byte = msf ? src[nbytes - 1 - bi] : src[bi];
            w |= byte << (8 * q);
          }
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
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mb;
       q += (long long)gridDim.x * blockDim.x) {
    const uint8_t byte = (uint8_t)(src[q >> 2] >> (8 * (q & 3)));
    dst[msf ? (mb - 1 - q) : q] = byte;
  }
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
// four-step twiddle w_L^(e) in Montgomery form, e < L.
__device__ __forceinline__ u32 fourstep_tw(const PlanTables& tab, int prime, int dir, u32 e,
                                           u32 p) {
  const int off = (prime * 2 + dir) * kTwN;
  const u32 lo = __ldg(&tab.tlo_m[off + (e & (kTwN - 1))]);
  const uint2 hi = __ldg(&tab.thi[off + (e >> kTwLg)]);
  return shoup(lo, hi, p);
}

// ---------------------------------------------------------------------------
// Column pass (forward): CT columns x R rows per CTA; DIF over rows.
// grid: x = C / CT, y = prime, z = b * 2 + op.
__global__ void k_col_fwd(ConvJob job, PlanTables tab, int lct) {
  extern __shared__ u32 smem[];
  const int prime = blockIdx.y;
  const int b = blockIdx.z >> 1, op = blockIdx.z & 1;
  const PrimeInfo pi = c_primes[prime];
  const int lgR = job.lgR, lgC = job.lgC;
  const int CT = 1 << lct;
  const long long L = 1ll << job.lg;
  const int c0 = blockIdx.x << lct;
  const u32* src = job.words + ((long long)b * 3 + op) * job.in_stride;
  const long long kvalid = op == 0 ? job.kA : job.kX;
  const int total = (1 << lgR) << lct;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx >> lct, t = idx & (CT - 1);
    const long long gi = ((long long)r << lgC) + c0 + t;
    const u32 raw = gi < kvalid ? __ldg(&src[gi]) : 0u;
    smem[pidx(r, t, lct)] = shoup(raw, 1u, pi.one_sh, pi.p);
  }
  __syncthreads();
  const uint2* tw = tab.stw + (prime * 2 + 0) * kTwN;
  panel_dif<false>(smem, lgR, lct, lct, 1, 0, tw, pi.p, pi.two_p);
  u32* dst = job.buf + (((long long)b * 2 + op) * 3 + prime) * L;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx >> lct, t = idx & (CT - 1);
    dst[((long long)r << lgC) + c0 + t] = smem[pidx(r, t, lct)];
  }
}

// Column pass (inverse): DIT over rows, scale, full reduction, residues -> slot A.
__global__ void k_col_inv(ConvJob job, PlanTables tab, int lct) {
  extern __shared__ u32 smem[];
  const int prime = blockIdx.y;
  const int b = blockIdx.z;
  const PrimeInfo pi = c_primes[prime];
  const int lgR = job.lgR, lgC = job.lgC;
  const int CT = 1 << lct;
  const long long L = 1ll << job.lg;
  const int c0 = blockIdx.x << lct;
  const u32* src = job.buf + (((long long)b * 2 + 1) * 3 + prime) * L;
  const int total = (1 << lgR) << lct;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx >> lct, t = idx & (CT - 1);
    smem[pidx(r, t, lct)] = src[((long long)r << lgC) + c0 + t];
  }
  __syncthreads();
  const uint2* tw = tab.stw + (prime * 2 + 1) * kTwN;
  panel_dit<false>(smem, lgR, lct, lct, 1, 0, tw, pi.p, pi.two_p);
  u32* dst = job.buf + (((long long)b * 2 + 0) * 3 + prime) * L;
  const u32 sc = tab.scale[prime], sc_sh = tab.scale_sh[prime];
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx >> lct, t = idx & (CT - 1);
    const long long gi = ((long long)r << lgC) + c0 + t;
    if (gi < job.nRes) dst[gi] = red(shoup(smem[pidx(r, t, lct)], sc, sc_sh, pi.p), pi.p);
  }
}

// Row pass: NR rows per CTA, A and X interleaved (t = 2*row + op).
// Forward four-step twiddle, DIF (A and X), pointwise Montgomery product,
// DIT (X), inverse twiddle; R == 1 is the whole transform (small blocks):
// inputs come straight from the packed words and residues are written out.
// grid: x = R / NR, y = prime, z = b.
__global__ void k_row(ConvJob job, PlanTables tab, int lnr) {
  extern __shared__ u32 smem[];
  const int prime = blockIdx.y;
  const int b = blockIdx.z;
  const PrimeInfo pi = c_primes[prime];
  const int lgR = job.lgR, lgC = job.lgC;
  const int C = 1 << lgC;
  const int NR = 1 << lnr;
  const int lnc = lnr + 1;
  const long long L = 1ll << job.lg;
  const int q0 = blockIdx.x << lnr;
  const bool single = (lgR == 0);
  const int total = (2 * NR) << lgC;

  // load
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int i = idx & (C - 1);
    const int t = idx >> lgC;
    const int row = t >> 1, op = t & 1;
    u32 v;
    if (single) {
      const u32* src = job.words + ((long long)b * 3 + op) * job.in_stride;
      const long long kvalid = op == 0 ? job.kA : job.kX;
      const u32 raw = i < kvalid ? __ldg(&src[i]) : 0u;
      v = shoup(raw, 1u, pi.one_sh, pi.p);
    } else {
      const u32* src = job.buf + (((long long)b * 2 + op) * 3 + prime) * L;
      v = src[((long long)(q0 + row) << lgC) + i];
      // forward four-step twiddle w_L^(i * k1), k1 = bitrev_R(q)
      const u32 k1 = (u32)brev(q0 + row, lgR);
      const u32 m = fourstep_tw(tab, prime, 0, (u32)i * k1, pi.p);
      v = montmul(v, m, pi.p, pi.p_mont);
    }
    smem[tidx(i, t, lgC)] = v;
  }
  __syncthreads();
  const uint2* twf = tab.stw + (prime * 2 + 0) * kTwN;
  const uint2* twi = tab.stw + (prime * 2 + 1) * kTwN;
  panel_dif<true>(smem, lgC, lnc, 0, 1, 0, twf, pi.p, pi.two_p);
  // pointwise product into the X slot (factor 2^-32 folded into the final scale)
  for (int idx = threadIdx.x; idx < (NR << lgC); idx += blockDim.x) {
    const int i = idx & (C - 1);
    const int row = idx >> lgC;
    const int ia = tidx(i, 2 * row, lgC), ix = tidx(i, 2 * row + 1, lgC);
    smem[ix] = montmul(smem[ia], smem[ix], pi.p, pi.p_mont);
  }
  __syncthreads();
  panel_dit<true>(smem, lgC, lnr, 0, 2, 1, twi, pi.p, pi.two_p);
  // store
  for (int idx = threadIdx.x; idx < (NR << lgC); idx += blockDim.x) {
    const int i = idx & (C - 1);
    const int row = idx >> lgC;
    u32 v = smem[tidx(i, 2 * row + 1, lgC)];
    if (single) {
      if (i < job.nRes) {
        u32* dst = job.buf + (((long long)b * 2 + 0) * 3 + prime) * L;
        dst[i] = red(shoup(v, tab.scale[prime], tab.scale_sh[prime], pi.p), pi.p);
      }
    } else {
      const u32 k1 = (u32)brev(q0 + row, lgR);
      const u32 m = fourstep_tw(tab, prime, 1, (u32)i * k1, pi.p);
      v = montmul(red(v, pi.two_p), m, pi.p, pi.p_mont);
      u32* dst = job.buf + (((long long)b * 2 + 1) * 3 + prime) * L;
      dst[((long long)(q0 + row) << lgC) + i] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Carry: CRT of the three residues, overlap-add of 96-bit coefficients at
// 32-bit stride, + D, carry-lookahead scan (decoupled look-back across tiles),
// mask to n_mod_bits, shift right, write output words.

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

__device__ __forceinline__ void crt3(u32 r0, u32 r1, u32 r2, u32& w0, u32& w1, u32& w2) {
  const CrtConst& k = c_crt;
  const u32 v0 = r0;
  u32 x1 = r1 + 2u * k.p1 - v0;
  u32 v1 = red(shoup(x1, k.inv01, k.inv01_sh, k.p1), k.p1);
  u32 u = v0 + shoup(v1, k.p0m2, k.p0m2_sh, k.p2);  // [0, 4 p2)
  u = red(u, 2u * k.p2);
  u32 x2 = r2 + 2u * k.p2 - u;
  u32 v2 = red(shoup(x2, k.inv012, k.inv012_sh, k.p2), k.p2);
  u64 lo = (u64)v0 + (u64)k.p0 * v1;        // < 2^61
  u64 prod_lo = k.p0p1 * (u64)v2;
  u64 prod_hi = __umul64hi(k.p0p1, (u64)v2);
  u64 s = lo + prod_lo;
  prod_hi += (s < lo) ? 1ull : 0ull;
  w0 = (u32)s;
  w1 = (u32)(s >> 32);
  w2 = (u32)prod_hi;
}

__global__ void __launch_bounds__(kCarryThreads) k_carry(ConvJob job) {
  __shared__ u32 s_tile;
  __shared__ u32 s_wq[kCarryThreads / 32], s_wt[kCarryThreads / 32];
  __shared__ u32 s_cin;
  const int b = blockIdx.y;
  if (threadIdx.x == 0) s_tile = atomicAdd(&job.tile_ctr[b], 1u);
  __syncthreads();
  const int tile = (int)s_tile;
  const long long L = 1ll << job.lg;
  const u32* res0 = job.buf + (((long long)b * 2 + 0) * 3 + 0) * L;
  const u32* res1 = res0 + L;
  const u32* res2 = res1 + L;
  const u32* dw = job.words + ((long long)b * 3 + 2) * job.in_stride;
  const long long w0 = (long long)tile * kCarryTile + (long long)threadIdx.x * kCarryItems;

  // column sums S[j] for words w0 .. w0+8
  u64 S[kCarryItems + 1];
  {
    u32 A0[kCarryItems + 3], A1[kCarryItems + 3], A2[kCarryItems + 3];
#pragma unroll
    for (int j = 0; j < kCarryItems + 3; ++j) {
      const long long k = w0 - 2 + j;
      if (k >= 0 && k < job.nRes) {
        crt3(__ldg(&res0[k]), __ldg(&res1[k]), __ldg(&res2[k]), A0[j], A1[j], A2[j]);
      } else {
        A0[j] = A1[j] = A2[j] = 0u;
      }
    }
#pragma unroll
    for (int j = 0; j <= kCarryItems; ++j) {
      const long long w = w0 + j;
      const u32 d = (w < job.kD) ? __ldg(&dw[w]) : 0u;
      S[j] = (u64)A0[j + 2] + A1[j + 1] + A2[j] + d;
    }
  }
  // local carry function
  CarryFn f;
  {
    u32 c = 0;
    u32 first = 0;
    bool allones = true;
#pragma unroll
    for (int j = 0; j < kCarryItems; ++j) {
      const u64 s = S[j] + c;
      const u32 t = (u32)s;
      c = (u32)(s >> 32);
      if (j == 0) first = t;
      else allones &= (t == 0xFFFFFFFFu);
    }
    f.id = false;
    f.q = c;
    f.t = (allones && first != 0u) ? (0u - first) : kInf;
  }
  // warp inclusive scan
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  CarryFn inc = f;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    CarryFn o;
    o.q = __shfl_up_sync(0xFFFFFFFFu, inc.q, d);
    o.t = __shfl_up_sync(0xFFFFFFFFu, inc.t, d);
    o.id = false;
    if (lane >= d) inc = cf_compose(inc, o);
  }
  CarryFn excl;
  excl.q = __shfl_up_sync(0xFFFFFFFFu, inc.q, 1);
  excl.t = __shfl_up_sync(0xFFFFFFFFu, inc.t, 1);
  excl.id = (lane == 0);
  if (lane == 31) {
    s_wq[warp] = inc.q;
    s_wt[warp] = inc.t;
  }
  __syncthreads();
  // prefix of earlier warps, and the tile aggregate
  CarryFn wpre{0, 0, true};
  CarryFn agg{0, 0, true};
#pragma unroll
  for (int w = 0; w < kCarryThreads / 32; ++w) {
    CarryFn fw{s_wq[w], s_wt[w], false};
    if (w < warp) wpre = cf_compose(fw, wpre);
    agg = cf_compose(fw, agg);
  }
  excl = cf_compose(excl, wpre);

  // decoupled look-back over the tiles of this block
  if (threadIdx.x == 0) {
    volatile unsigned long long* st = job.tile_state + (long long)b * job.tiles;
    u32 cin;
    if (tile == 0) {
      cin = 0;
    } else {
      st[tile] = (1ull << 62) | ((unsigned long long)agg.q << 32) | agg.t;
      CarryFn F{0, 0, true};
      int j = tile - 1;
      while (true) {
        const unsigned long long v = st[j];
        const u32 flag = (u32)(v >> 62);
        if (flag == 0) continue;
        if (flag == 2) {
          cin = cf_apply(F, (u32)((v >> 32) & 0xFFu));
          break;
        }
        CarryFn g{(u32)((v >> 32) & 0xFFu), (u32)v, false};
        F = cf_compose(F, g);
        --j;
      }
    }
    const u32 cout = cf_apply(agg, cin);
    st[tile] = (2ull << 62) | ((unsigned long long)cout << 32);
    s_cin = cin;
  }
  __syncthreads();
  u32 c = cf_apply(excl, s_cin);

  // final words, masked
  u32 T[kCarryItems + 1];
#pragma unroll
  for (int j = 0; j <= kCarryItems; ++j) {
    const u64 s = S[j] + c;
    T[j] = (u32)s;
    c = (u32)(s >> 32);
    const long long w = w0 + j;
    if (w >= job.nT) {
      T[j] = 0u;
    } else if (w == job.nT - 1) {
      const long long rb = job.n_mod_bits - 32ll * (job.nT - 1);
      if (rb < 32) T[j] &= (1u << rb) - 1u;
    }
  }
  // output words y_j = T >> shift
  const long long ws = job.shift >> 5;
  const int sh = (int)(job.shift & 31);
  u32* out = job.out_words + (long long)b * job.mw;
#pragma unroll
  for (int j = 0; j < kCarryItems; ++j) {
    const long long oj = w0 + j - ws;
    if (oj >= 0 && oj < job.mw) {
      out[oj] = sh ? ((T[j] >> sh) | (T[j + 1] << (32 - sh))) : T[j];
    }
  }
}

// ---------------------------------------------------------------------------

static int col_lct(int lgR, int lgC) {
  int lct = 14 - lgR;  // ~16K words per CTA
  if (lct > 5) lct = 5;
  if (lct < 3) lct = 3;
  if (lct > lgC) lct = lgC;
  return lct;
}

void launch_conv(const ConvJob& job, const PlanTables& tab, cudaStream_t st) {
  const int threads = 256;
  if (job.lgR == 0) {
    const int lnr = 0;
    const size_t sm = (size_t)tm_stride(job.lgC) * (2 << lnr) * 4;
    prof::Scope ps_("k_row_single", st);
    k_row<<<dim3(1, kNumPrimes, job.batch), threads, sm, st>>>(job, tab, lnr);
    return;
  }
  const int lct = col_lct(job.lgR, job.lgC);
  const size_t smc = (size_t)panel_words(job.lgR, lct) * 4;
  {
    prof::Scope ps_("k_col_fwd", st);
    k_col_fwd<<<dim3(1u << (job.lgC - lct), kNumPrimes, job.batch * 2), threads, smc, st>>>(
        job, tab, lct);
  }
  int lnr = 13 - job.lgC;  // ~8K words (A+X) per CTA
  if (lnr < 0) lnr = 0;
  if (lnr > job.lgR) lnr = job.lgR;
  const size_t smr = (size_t)tm_stride(job.lgC) * (2 << lnr) * 4;
  {
    prof::Scope ps_("k_row", st);
    k_row<<<dim3(1u << (job.lgR - lnr), kNumPrimes, job.batch), threads, smr, st>>>(job, tab, lnr);
  }
  {
    prof::Scope ps_("k_col_inv", st);
    k_col_inv<<<dim3(1u << (job.lgC - lct), kNumPrimes, job.batch), threads, smc, st>>>(job, tab,
                                                                                        lct);
  }
}

void launch_carry(const ConvJob& job, cudaStream_t st) {
  prof::Scope ps_("k_carry", st);
  k_carry<<<dim3(job.tiles, job.batch), kCarryThreads, 0, st>>>(job);
}

// Opt every dynamic-smem kernel into > 48 KB once.
void set_kernel_attrs() {
  cudaFuncSetAttribute(k_col_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_col_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace pab
