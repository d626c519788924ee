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
#include <mutex>
#include <string>
#include <vector>

#include "ntt_core.cuh"
#include "pa_kernels.cuh"

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
// pack / unpack (MSF byte order or unaligned blocks only)

__global__ void k_pack(const uint8_t* __restrict__ in, long long in_stride, long long n_bits,
                       int msf, u32* __restrict__ words, long long word_stride, long long kw) {
  const int b = blockIdx.y;
  const uint8_t* src = in + (long long)b * in_stride;
  u32* dst = words + (long long)b * word_stride;
  const long long nbytes = (n_bits + 7) >> 3;
  const long long kn = (n_bits + 31) >> 5;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < kw;
       j += (long long)gridDim.x * blockDim.x) {
    u32 w = 0;
    if (j < kn) {
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
// operand word fetch: zero beyond the valid words, mask the last one
__device__ __forceinline__ u32 fetch_word(const u32* __restrict__ src, long long gi, long long kv,
                                          u32 mask) {
  if (gi >= kv) return 0u;
  const u32 w = __ldg(src + gi);
  return gi == kv - 1 ? (w & mask) : w;
}

// four-step twiddle seed w_L^e * 2^32 (Montgomery form, lazy [0, 2p)), e < L
template <int P>
__device__ __forceinline__ u32 tw_seed(const PlanTables& tab, int dir, u32 e) {
  const int off = (P * 2 + dir) * kTwN;
  const u32 lo = __ldg(&tab.tlo_m[off + (e & (kTwN - 1))]);
  const uint2 hi = __ldg(&tab.thi[off + (e >> kTwLg)]);
  return shoup(lo, hi, PK<P>::p);
}

// ---------------------------------------------------------------------------
// Row pass.  CTA: NR = 2^lnr rows of one (block, prime); smem holds the NR
// c-rows (A) then the NR x-rows (X), each sm_len(LGC) words.
// SMALL (lgR == 0): the row is the whole transform; read the operand words,
// write scaled residues.
template <int P, int LGC, bool SMALL>
__device__ __forceinline__ void row_body(const ConvJob& job, const PlanTables& tab, int lnr) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGC);
  constexpr int T = sm_len(LGC);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int NR = 1 << lnr;
  const int b = blockIdx.z;
  const int q0 = blockIdx.x << lnr;
  const int lgR = job.lgR;
  const long long L = 1ll << job.lg;
  u32* sA = smem;
  u32* sX = smem + NR * T;
  const uint2* twf = tab.stw + (P * 2 + 0) * kTwN;
  const uint2* twi = tab.stw + (P * 2 + 1) * kTwN;
  u32* gA = job.buf + (((long long)b * 2 + 0) * 3 + P) * L;  // also the residue slot
  u32* gX = job.buf + (((long long)b * 2 + 1) * 3 + P) * L;
  const u32* wA = job.srcA + (long long)b * job.src_stride;
  const u32* wX = job.srcX + (long long)b * job.src_stride;

  // ---- pass 0: global -> (twiddle) -> DIF top stages -> smem (A and X share twiddles)
  if constexpr (PP.n > 1) {
    for (int task = threadIdx.x; task < (NR << SLO0); task += blockDim.x) {
      const int row = task >> SLO0, o = task & ((1 << SLO0) - 1);
      const int q = q0 + row;
      u32 v[2][1 << RS0];
      if constexpr (SMALL) {
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          const long long gi = o + (k << SLO0);
          v[0][k] = shoup(fetch_word(wA, gi, job.kA, job.maskA), 1u, PK<P>::one_sh, PK<P>::p);
          v[1][k] = shoup(fetch_word(wX, gi, job.kX, job.maskX), 1u, PK<P>::one_sh, PK<P>::p);
        }
      } else {
        const u32* ra = gA + ((long long)q << LGC) + o;
        const u32* rx = gX + ((long long)q << LGC) + o;
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          v[0][k] = ra[k << SLO0];
          v[1][k] = rx[k << SLO0];
        }
        const u32 k1 = (u32)brev(q, lgR);
        u32 m = tw_seed<P>(tab, 0, (u32)o * k1);
        const uint2 gam = __ldg(&tab.g[(P * 2 + 0) * kTwN + k1]);
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          v[0][k] = mont<P>(v[0][k], m);
          v[1][k] = mont<P>(v[1][k], m);
          m = shoup(m, gam, PK<P>::p);
        }
      }
      dif_rt<P, RS0, SLO0, 2>(v, twf + o);
      const int base = row * T + sm_idx(o);
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) {
        sA[base + k * sm_step(SLO0)] = v[0][k];
        sX[base + k * sm_step(SLO0)] = v[1][k];
      }
    }
    __syncthreads();
  }
  // ---- pass 1 (middle), forward, A and X
  if constexpr (PP.n == 3) {
    constexpr int RS1 = PP.rs[1], SLO1 = PP.slo[1];
    constexpr int LGG = LGC - RS1;  // groups per row (log2)
    for (int task = threadIdx.x; task < (NR << LGG); task += blockDim.x) {
      const int row = task >> LGG, g = task & ((1 << LGG) - 1);
      const int o = g & ((1 << SLO1) - 1), blk = g >> SLO1;
      const int base = row * T + sm_idx((blk << (SLO1 + RS1)) + o);
      u32 v[2][1 << RS1];
#pragma unroll
      for (int k = 0; k < (1 << RS1); ++k) {
        v[0][k] = sA[base + k * sm_step(SLO1)];
        v[1][k] = sX[base + k * sm_step(SLO1)];
      }
      dif_rt<P, RS1, SLO1, 2>(v, twf + o);
#pragma unroll
      for (int k = 0; k < (1 << RS1); ++k) {
        sA[base + k * sm_step(SLO1)] = v[0][k];
        sX[base + k * sm_step(SLO1)] = v[1][k];
      }
    }
    __syncthreads();
  }
  // ---- last DIF pass (lowest stages) + pointwise + first DIT pass
  constexpr int RSL = PP.rs[PP.n - 1];
  {
    constexpr int LGG = LGC - RSL;
    for (int task = threadIdx.x; task < (NR << LGG); task += blockDim.x) {
      const int row = task >> LGG, g = task & ((1 << LGG) - 1);
      u32 a[1][1 << RSL], x[1][1 << RSL];
      int base = 0;
      if constexpr (PP.n == 1) {  // whole transform in registers, straight from global
        const int q = q0 + row;
        if constexpr (SMALL) {
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            a[0][k] = shoup(fetch_word(wA, k, job.kA, job.maskA), 1u, PK<P>::one_sh, PK<P>::p);
            x[0][k] = shoup(fetch_word(wX, k, job.kX, job.maskX), 1u, PK<P>::one_sh, PK<P>::p);
          }
        } else {
          const u32 k1 = (u32)brev(q, lgR);
          u32 m = tw_seed<P>(tab, 0, 0u);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 0) * kTwN + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            a[0][k] = mont<P>(gA[((long long)q << LGC) + k], m);
            x[0][k] = mont<P>(gX[((long long)q << LGC) + k], m);
            m = shoup(m, gam, PK<P>::p);
          }
        }
      } else {
        base = row * T + sm_idx(g << RSL);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) a[0][k] = sA[base + k];
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) x[0][k] = sX[base + k];
      }
      dif_ct<P, RSL, 1>(a);
      dif_ct<P, RSL, 1>(x);
#pragma unroll
      for (int k = 0; k < (1 << RSL); ++k) x[0][k] = mont<P>(a[0][k], x[0][k]);
      dit_ct<P, RSL>(x[0]);
      if constexpr (PP.n == 1) {
        const int q = q0 + row;
        if constexpr (SMALL) {
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k)
            if (k < job.nRes)
              gA[k] = red(shoup(x[0][k], tab.scale[P], tab.scale_sh[P], PK<P>::p), PK<P>::p);
        } else {
          const u32 k1 = (u32)brev(q, lgR);
          u32 m = tw_seed<P>(tab, 1, 0u);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 1) * kTwN + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            gX[((long long)q << LGC) + k] = mont<P>(red(x[0][k], PK<P>::two_p), m);
            m = shoup(m, gam, PK<P>::p);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) sX[base + k] = x[0][k];
      }
    }
  }
  if constexpr (PP.n > 1) {
    __syncthreads();
    // ---- pass 1 inverse (X)
    if constexpr (PP.n == 3) {
      constexpr int RS1 = PP.rs[1], SLO1 = PP.slo[1];
      constexpr int LGG = LGC - RS1;
      for (int task = threadIdx.x; task < (NR << LGG); task += blockDim.x) {
        const int row = task >> LGG, g = task & ((1 << LGG) - 1);
        const int o = g & ((1 << SLO1) - 1), blk = g >> SLO1;
        const int base = row * T + sm_idx((blk << (SLO1 + RS1)) + o);
        u32 v[1 << RS1];
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) v[k] = sX[base + k * sm_step(SLO1)];
        dit_rt<P, RS1, SLO1>(v, twi + o);
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) sX[base + k * sm_step(SLO1)] = v[k];
      }
      __syncthreads();
    }
    // ---- pass 0 inverse (X) -> inverse twiddle -> global (or scaled residues)
    for (int task = threadIdx.x; task < (NR << SLO0); task += blockDim.x) {
      const int row = task >> SLO0, o = task & ((1 << SLO0) - 1);
      const int q = q0 + row;
      const int base = row * T + sm_idx(o);
      u32 v[1 << RS0];
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) v[k] = sX[base + k * sm_step(SLO0)];
      dit_rt<P, RS0, SLO0>(v, twi + o);
      if constexpr (SMALL) {
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          const long long gi = o + (k << SLO0);
          if (gi < job.nRes)
            gA[gi] = red(shoup(v[k], tab.scale[P], tab.scale_sh[P], PK<P>::p), PK<P>::p);
        }
      } else {
        const u32 k1 = (u32)brev(q, lgR);
        u32 m = tw_seed<P>(tab, 1, (u32)o * k1);
        const uint2 gam = __ldg(&tab.g[(P * 2 + 1) * kTwN + k1]);
        u32* rx = gX + ((long long)q << LGC) + o;
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          rx[k << SLO0] = mont<P>(red(v[k], PK<P>::two_p), m);
          m = shoup(m, gam, PK<P>::p);
        }
      }
    }
  }
}

template <int LGC, bool SMALL>
__global__ void __launch_bounds__(256) k_row(ConvJob job, PlanTables tab, int lnr) {
  switch (blockIdx.y) {
    case 0: row_body<0, LGC, SMALL>(job, tab, lnr); break;
    case 1: row_body<1, LGC, SMALL>(job, tab, lnr); break;
    default: row_body<2, LGC, SMALL>(job, tab, lnr); break;
  }
}

// ---------------------------------------------------------------------------
// Column passes.  CTA: CT = 2^lct adjacent columns x R rows, interleaved in
// smem as s[sm_idx(row) * CT + t]; lanes walk columns (coalesced, twiddle
// broadcast).  Forward: operand words -> DIF -> buf; inverse: buf -> DIT ->
// scaled residues.
template <int P, int LGR>
__device__ __forceinline__ void col_fwd_body(const ConvJob& job, const PlanTables& tab, int lct) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int CT = 1 << lct;
  const int b = blockIdx.z >> 1, op = blockIdx.z & 1;
  const int lgC = job.lgC;
  const long long L = 1ll << job.lg;
  const int c0 = blockIdx.x << lct;
  const u32* src = (op ? job.srcX : job.srcA) + (long long)b * job.src_stride;
  const long long kv = op ? job.kX : job.kA;
  const u32 mask = op ? job.maskX : job.maskA;
  u32* dst = job.buf + (((long long)b * 2 + op) * 3 + P) * L;
  const uint2* twf = tab.stw + (P * 2 + 0) * kTwN;

  if constexpr (PP.n == 1) {
    for (int t = threadIdx.x; t < CT; t += blockDim.x) {
      u32 v[1][1 << LGR];
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k)
        v[0][k] = shoup(fetch_word(src, ((long long)k << lgC) + c0 + t, kv, mask), 1u,
                        PK<P>::one_sh, PK<P>::p);
      dif_ct<P, LGR, 1>(v);
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) dst[((long long)k << lgC) + c0 + t] = v[0][k];
    }
  } else {
    for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
      const int t = task & (CT - 1), o = task >> lct;
      u32 v[1][1 << RS0];
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) {
        const long long gi = ((long long)(o + (k << SLO0)) << lgC) + c0 + t;
        v[0][k] = shoup(fetch_word(src, gi, kv, mask), 1u, PK<P>::one_sh, PK<P>::p);
      }
      dif_rt<P, RS0, SLO0, 1>(v, twf + o);
      const int base = sm_idx(o) * CT + t;
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) smem[base + k * sm_step(SLO0) * CT] = v[0][k];
    }
    __syncthreads();
    if constexpr (PP.n == 3) {
      constexpr int RS1 = PP.rs[1], SLO1 = PP.slo[1];
      for (int task = threadIdx.x; task < (CT << (LGR - RS1)); task += blockDim.x) {
        const int t = task & (CT - 1), g = task >> lct;
        const int o = g & ((1 << SLO1) - 1), blk = g >> SLO1;
        const int base = sm_idx((blk << (SLO1 + RS1)) + o) * CT + t;
        u32 v[1][1 << RS1];
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) v[0][k] = smem[base + k * sm_step(SLO1) * CT];
        dif_rt<P, RS1, SLO1, 1>(v, twf + o);
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) smem[base + k * sm_step(SLO1) * CT] = v[0][k];
      }
      __syncthreads();
    }
    for (int task = threadIdx.x; task < (CT << (LGR - 5)); task += blockDim.x) {
      const int t = task & (CT - 1), g = task >> lct;
      const int base = (33 * g) * CT + t;
      u32 v[1][32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[0][k] = smem[base + k * CT];
      dif_ct<P, 5, 1>(v);
      u32* d = dst + ((long long)(g << 5) << lgC) + c0 + t;
#pragma unroll
      for (int k = 0; k < 32; ++k) d[(long long)k << lgC] = v[0][k];
    }
  }
}

template <int P, int LGR>
__device__ __forceinline__ void col_inv_body(const ConvJob& job, const PlanTables& tab, int lct) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int CT = 1 << lct;
  const int b = blockIdx.z;
  const int lgC = job.lgC;
  const long long L = 1ll << job.lg;
  const int c0 = blockIdx.x << lct;
  const u32* src = job.buf + (((long long)b * 2 + 1) * 3 + P) * L;
  u32* res = job.buf + (((long long)b * 2 + 0) * 3 + P) * L;
  const uint2* twi = tab.stw + (P * 2 + 1) * kTwN;
  const u32 sc = tab.scale[P], sc_sh = tab.scale_sh[P];

  if constexpr (PP.n == 1) {
    for (int t = threadIdx.x; t < CT; t += blockDim.x) {
      u32 v[1 << LGR];
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) v[k] = src[((long long)k << lgC) + c0 + t];
      dit_ct<P, LGR>(v);
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) {
        const long long gi = ((long long)k << lgC) + c0 + t;
        if (gi < job.nRes) res[gi] = red(shoup(v[k], sc, sc_sh, PK<P>::p), PK<P>::p);
      }
    }
  } else {
    for (int task = threadIdx.x; task < (CT << (LGR - 5)); task += blockDim.x) {
      const int t = task & (CT - 1), g = task >> lct;
      const u32* s = src + ((long long)(g << 5) << lgC) + c0 + t;
      u32 v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = s[(long long)k << lgC];
      dit_ct<P, 5>(v);
      const int base = (33 * g) * CT + t;
#pragma unroll
      for (int k = 0; k < 32; ++k) smem[base + k * CT] = v[k];
    }
    __syncthreads();
    if constexpr (PP.n == 3) {
      constexpr int RS1 = PP.rs[1], SLO1 = PP.slo[1];
      for (int task = threadIdx.x; task < (CT << (LGR - RS1)); task += blockDim.x) {
        const int t = task & (CT - 1), g = task >> lct;
        const int o = g & ((1 << SLO1) - 1), blk = g >> SLO1;
        const int base = sm_idx((blk << (SLO1 + RS1)) + o) * CT + t;
        u32 v[1 << RS1];
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) v[k] = smem[base + k * sm_step(SLO1) * CT];
        dit_rt<P, RS1, SLO1>(v, twi + o);
#pragma unroll
        for (int k = 0; k < (1 << RS1); ++k) smem[base + k * sm_step(SLO1) * CT] = v[k];
      }
      __syncthreads();
    }
    for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
      const int t = task & (CT - 1), o = task >> lct;
      const int base = sm_idx(o) * CT + t;
      u32 v[1 << RS0];
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) v[k] = smem[base + k * sm_step(SLO0) * CT];
      dit_rt<P, RS0, SLO0>(v, twi + o);
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) {
        const long long gi = ((long long)(o + (k << SLO0)) << lgC) + c0 + t;
        if (gi < job.nRes) res[gi] = red(shoup(v[k], sc, sc_sh, PK<P>::p), PK<P>::p);
      }
    }
  }
}

template <int LGR>
__global__ void __launch_bounds__(256) k_col_fwd(ConvJob job, PlanTables tab, int lct) {
  switch (blockIdx.y) {
    case 0: col_fwd_body<0, LGR>(job, tab, lct); break;
    case 1: col_fwd_body<1, LGR>(job, tab, lct); break;
    default: col_fwd_body<2, LGR>(job, tab, lct); break;
  }
}
template <int LGR>
__global__ void __launch_bounds__(256) k_col_inv(ConvJob job, PlanTables tab, int lct) {
  switch (blockIdx.y) {
    case 0: col_inv_body<0, LGR>(job, tab, lct); break;
    case 1: col_inv_body<1, LGR>(job, tab, lct); break;
    default: col_inv_body<2, LGR>(job, tab, lct); break;
  }
}

// ---------------------------------------------------------------------------
// Carry: CRT of the three residues, overlap-add of the 96-bit coefficients at
// 32-bit stride, + D, carry-lookahead scan (decoupled look-back across tiles),
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

__device__ __forceinline__ void crt3(u32 r0, u32 r1, u32 r2, u32& w0, u32& w1, u32& w2) {
  const CrtConst& k = c_crt;
  const u32 v0 = r0;
  const u32 x1 = r1 + 2u * k.p1 - v0;
  const u32 v1 = red(shoup(x1, k.inv01, k.inv01_sh, k.p1), k.p1);
  u32 u = v0 + shoup(v1, k.p0m2, k.p0m2_sh, k.p2);  // [0, 4 p2)
  u = red(u, 2u * k.p2);
  const u32 x2 = r2 + 2u * k.p2 - u;
  const u32 v2 = red(shoup(x2, k.inv012, k.inv012_sh, k.p2), k.p2);
  const u64 lo = (u64)v0 + (u64)k.p0 * v1;  // < 2^61
  const u64 prod_lo = k.p0p1 * (u64)v2;
  u64 prod_hi = __umul64hi(k.p0p1, (u64)v2);
  const u64 s = lo + prod_lo;
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
  const u32* dw = job.srcD ? job.srcD + (long long)b * job.src_stride : nullptr;
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
      const u32 d = dw ? fetch_word(dw, w, job.kD, job.maskD) : 0u;
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
  if (job.out_words) {
    u32* out = job.out_words + (long long)b * job.mw;
#pragma unroll
    for (int j = 0; j < kCarryItems; ++j) {
      const long long oj = w0 + j - ws;
      if (oj >= 0 && oj < job.mw) out[oj] = sh ? ((T[j] >> sh) | (T[j + 1] << (32 - sh))) : T[j];
    }
  } else {  // LSF bytes, word-aligned block starts
    uint8_t* out = job.out_bytes + (long long)b * job.out_stride;
#pragma unroll
    for (int j = 0; j < kCarryItems; ++j) {
      const long long oj = w0 + j - ws;
      if (oj >= 0 && oj < job.mw) {
        const u32 y = sh ? ((T[j] >> sh) | (T[j + 1] << (32 - sh))) : T[j];
        if (4 * oj + 4 <= job.rbytes) {
          reinterpret_cast<u32*>(out)[oj] = y;
        } else {
          for (int q = 0; q < 4 && 4 * oj + q < job.rbytes; ++q)
            out[4 * oj + q] = (uint8_t)(y >> (8 * q));
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch over compile-time transform sizes

typedef void (*ConvKernel)(ConvJob, PlanTables, int);

static ConvKernel row_kernel(int lg, bool small) {
  switch (lg) {
#define PAB_ROW(L) \
  case L: return small ? k_row<L, true> : k_row<L, false>;
    PAB_ROW(1) PAB_ROW(2) PAB_ROW(3) PAB_ROW(4) PAB_ROW(5) PAB_ROW(6) PAB_ROW(7) PAB_ROW(8)
    PAB_ROW(9) PAB_ROW(10) PAB_ROW(11) PAB_ROW(12)
#undef PAB_ROW
    default: return nullptr;
  }
}
static ConvKernel col_kernel(int lg, bool inv) {
  switch (lg) {
#define PAB_COL(L) \
  case L: return inv ? k_col_inv<L> : k_col_fwd<L>;
    PAB_COL(6) PAB_COL(7) PAB_COL(8) PAB_COL(9) PAB_COL(10) PAB_COL(11) PAB_COL(12)
#undef PAB_COL
    default: return nullptr;
  }
}

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
    const size_t sm = (size_t)sm_len(job.lgC) * 2 * 4;
    prof::Scope ps_("k_row_single", st);
    row_kernel(job.lgC, true)<<<dim3(1, kNumPrimes, job.batch), threads, sm, st>>>(job, tab, 0);
    return;
  }
  const int lct = col_lct(job.lgR, job.lgC);
  const size_t smc = (size_t)sm_len(job.lgR) * (1u << lct) * 4;
  {
    prof::Scope ps_("k_col_fwd", st);
    col_kernel(job.lgR, false)<<<dim3(1u << (job.lgC - lct), kNumPrimes, job.batch * 2), threads,
                                 smc, st>>>(job, tab, lct);
  }
  int lnr = 13 - job.lgC;  // 8K words of rows (A+X: 16K words) per CTA
  if (lnr < 0) lnr = 0;
  if (lnr > job.lgR) lnr = job.lgR;
  const size_t smr = (size_t)sm_len(job.lgC) * (2u << lnr) * 4;
  {
    prof::Scope ps_("k_row", st);
    row_kernel(job.lgC, false)<<<dim3(1u << (job.lgR - lnr), kNumPrimes, job.batch), threads, smr,
                                 st>>>(job, tab, lnr);
  }
  {
    prof::Scope ps_("k_col_inv", st);
    col_kernel(job.lgR, true)<<<dim3(1u << (job.lgC - lct), kNumPrimes, job.batch), threads, smc,
                                st>>>(job, tab, lct);
  }
}

void launch_carry(const ConvJob& job, cudaStream_t st) {
  prof::Scope ps_("k_carry", st);
  k_carry<<<dim3(job.tiles, job.batch), kCarryThreads, 0, st>>>(job);
}

// Opt every dynamic-smem kernel into > 48 KB once per device.
void set_kernel_attrs() {
  for (int lg = 1; lg <= 12; ++lg) {
    for (int s = 0; s < 2; ++s) {
      ConvKernel k = row_kernel(lg, s != 0);
      if (k) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      ConvKernel c = col_kernel(lg, s != 0);
      if (c) cudaFuncSetAttribute(c, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
  }
}

}  // namespace pab
