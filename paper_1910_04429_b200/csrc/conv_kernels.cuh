// Size-specialised NTT conv kernels (instantiated per transform size in
// conv_lg*.cu so they compile in parallel).  See pa_kernels.cu for the pipeline.
#pragma once
#include "ntt_core.cuh"
#include "pa_kernels.cuh"

namespace pab {

typedef void (*ConvKernel)(ConvJob, PlanTables, int);
struct ConvKernels {
  ConvKernel row, row_small, row_tw4;
  ConvKernel col_fwd, col_inv;      // column passes with lgC == LG (lg even)
  ConvKernel col_fwd1, col_inv1;    // column passes with lgC == LG + 1 (lg odd)
  ConvKernel col_fwd_all, col_fwd_all1;  // all-primes forward column pass (lgC == LG, LG + 1)
  // mixed radix M = 3, 5 (index 0, 1) with LGR2 == LG and lgC = LG + 2 + dc (dc = 0..2)
  ConvKernel colm_fwd[2][3], colm_inv[2][3];
  ConvKernel colm_fwd_all[2][3];
};

__device__ __forceinline__ int brev(int x, int bits) {
  return bits == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - bits));
}

// Operand in coefficient units: cw = 2 reads 64-bit coefficients (words 2i, 2i+1;
// 8-byte aligned), cw = 1 single words.  Coefficients >= kc are zero; the last
// one is masked with (mlo, mhi) (bits >= n of the operand's last word).
struct OpView {
  const u32* src;
  int kc;
  u32 mlo, mhi;
  int cw;
  bool a8;   // cw = 2: the row is 8-byte aligned (else two 4-byte loads per coefficient)
  bool odd;  // cw = 2: odd word count, the last coefficient has no high word
};
__device__ __forceinline__ OpView op_view(const ConvJob& job, int op, int b) {
  OpView v;
  v.src = (op ? job.srcX : job.srcA) + (long long)b * job.src_stride;
  const long long kv = op ? job.kX : job.kA;
  const u32 mask = op ? job.maskX : job.maskA;
  v.cw = job.cw;
  v.a8 = (reinterpret_cast<uintptr_t>(v.src) & 7) == 0;
  v.odd = (kv & 1) != 0;
  if (job.cw == 2) {
    v.kc = (int)((kv + 1) >> 1);
    v.mlo = (kv & 1) ? mask : 0xFFFFFFFFu;
    v.mhi = (kv & 1) ? 0u : mask;
  } else {
    v.kc = (int)kv;
    v.mlo = mask;
    v.mhi = 0u;
  }
  return v;
}
// coefficient (lo, hi) -> residue in [0, 2p)
// The low word needs no multiply: 2^32 < 6p for every prime, so it is below 6p and
// two subtract-and-min steps by 2p bring it (or its sum with the high word's Shoup
// product, which stays below 2^32) into [0, 2p).  An IMAD.HI holds the FMA pipe 4
// clk and an IMAD 2 (profiles/r2/pipe_rates.json); these are ALU-pipe ops.
template <int P>
__device__ __forceinline__ u32 coef_red(u32 lo, u32 hi, int cw) {
  static_assert(6ull * kPrimes[P] > (1ull << 32), "low word must be below 6p");
  const u32 a = red(lo, PK<P>::two_p);  // < max(2p, 2^32 - 2p) < 4p
  if (cw == 1) return red(a, PK<P>::two_p);
  // a + s < 2^32: a < 2p gives < 4p, else a < 2^32 - 2p and s < 2p
  const u32 s = a + shoup(hi, PK<P>::r32, PK<P>::r32_sh, PK<P>::p);
  return red(red(s, PK<P>::two_p), PK<P>::two_p);
}
// the two words of 64-bit coefficient gi (cw = 2): one 8-byte load on 8-byte
// aligned rows, else two 4-byte loads; the last coefficient of an odd word
// count has no high word (it is not read: it may lie past the row)
__device__ __forceinline__ uint2 ld_coef2(const OpView& o, int gi, bool last) {
  // two 4-byte loads, the second predicated (no branch between loads, so the
  // compiler can issue a task's loads together); hot paths use 8-byte loads directly
  const u32* w = o.src + 2 * gi;
  const u32 lo = __ldg(w);
  const u32 hi = (last && o.odd) ? 0u : __ldg(w + 1);
  return make_uint2(lo, hi);
}
// coefficient gi known to be valid and unmasked (gi < kc - 1)
template <int P>
__device__ __forceinline__ u32 coef_fast(const OpView& o, int gi) {
  if (o.cw == 2) {
    const uint2 w = ld_coef2(o, gi, false);
    return coef_red<P>(w.x, w.y, 2);
  }
  return coef_red<P>(__ldg(o.src + gi), 0u, 1);
}
// raw coefficient words (lo, hi; hi = 0 for cw = 1) at any index: zero at or
// beyond kc, last one masked
__device__ __forceinline__ uint2 coef_raw_at(const OpView& o, int gi) {
  uint2 w = make_uint2(0u, 0u);
  if (gi < o.kc) {
    if (o.cw == 2) {
      w = ld_coef2(o, gi, gi == o.kc - 1);
    } else {
      w.x = __ldg(o.src + gi);
    }
    if (gi == o.kc - 1) {
      w.x &= o.mlo;
      w.y &= o.mhi;
    }
  }
  return w;
}

// any coefficient index: zero at or beyond kc, last one masked
template <int P>
__device__ __forceinline__ u32 coef_at(const OpView& o, int gi) {
  u32 lo = 0u, hi = 0u;
  if (gi < o.kc) {
    if (o.cw == 2) {
      const uint2 w = ld_coef2(o, gi, gi == o.kc - 1);
      lo = w.x;
      hi = w.y;
    } else {
      lo = __ldg(o.src + gi);
    }
    if (gi == o.kc - 1) {
      lo &= o.mlo;
      hi &= o.mhi;
    }
  }
  return coef_red<P>(lo, hi, o.cw);
}

// Forward column grid (1-D): chunks of fwd_chunk blocks, then prime, then
// block, operand, column tile.  All primes of a chunk read the same operand
// words, which stay L2-resident across the chunk's five prime sweeps, while
// the CTAs resident together run one prime's code.
struct FwdIdx {
  int prime, b, op, tile;
};
__device__ __forceinline__ FwdIdx fwd_idx(const ConvJob& job, int lct) {
  const unsigned tc = 1u << (job.lgC - lct);
  const unsigned per_block = 2u * tc;  // CTAs of one (block, prime)
  const unsigned span = per_block * (unsigned)job.pn * (unsigned)job.fwd_chunk;
  const unsigned id = blockIdx.x;
  const unsigned c = id / span;
  const unsigned local = id - c * span;
  const int b0 = (int)c * job.fwd_chunk;
  const int nb = min(job.fwd_chunk, job.batch - b0);
  const unsigned per_prime = per_block * (unsigned)nb;
  FwdIdx r;
  const unsigned pi = local / per_prime;
  r.prime = job.p0 + (int)pi;
  const unsigned rem = local - pi * per_prime;
  r.b = b0 + (int)(rem / per_block);
  const unsigned w = rem - (rem / per_block) * per_block;
  r.op = (int)(w / tc);
  r.tile = (int)(w - (unsigned)r.op * tc);
  return r;
}

// Operand staging for the all-primes forward column kernel: rows [0, rows) x
// CT columns of raw coefficients (uint2: lo, hi; hi = 0 for cw = 1) at
// stage[row * CT + t] via cp.async, so the whole tile's loads are in flight at
// once and are then reused by every prime.  Coefficients >= kc are zero, the
// last one is masked.
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((u32)__cvta_generic_to_shared(s)),
               "l"(g));
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((u32)__cvta_generic_to_shared(s)),
               "l"(g));
}
template <int LCT = -1>
__device__ __forceinline__ void stage_operand(const OpView& ov, uint2* stage, int rows, int lct_in,
                                              int lgC, int c0) {
  const int lct = LCT >= 0 ? LCT : lct_in;
  const int CT = 1 << lct;
  if (ov.cw == 2 && ov.a8 && ((rows - 1) << lgC) + c0 + CT - 1 < ov.kc - 1) {
    // every staged coefficient valid and unmasked (all but the operand's last tiles)
    for (int e = threadIdx.x; e < (rows << lct); e += blockDim.x) {
      const int gi = ((e >> lct) << lgC) + c0 + (e & (CT - 1));
      cp_async8(stage + e, ov.src + 2 * gi);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    return;
  }
  for (int e = threadIdx.x; e < (rows << lct); e += blockDim.x) {
    const int gi = ((e >> lct) << lgC) + c0 + (e & (CT - 1));
    if (gi < ov.kc - 1) {
      if (ov.cw == 2) {
        if (ov.a8) {
          cp_async8(stage + e, ov.src + 2 * gi);
        } else {
          cp_async4(stage + e, ov.src + 2 * gi);
          cp_async4(reinterpret_cast<u32*>(stage + e) + 1, ov.src + 2 * gi + 1);
        }
      } else {
        cp_async4(stage + e, ov.src + gi);
        reinterpret_cast<u32*>(stage + e)[1] = 0u;
      }
    } else {
      stage[e] = coef_raw_at(ov, gi);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
}

// staged raw coefficient (row, t) -> residue in [0, 2p); rows >= srows are zero
template <int P>
__device__ __forceinline__ u32 coef_staged(const uint2* stage, int row, int t, int lct, int srows,
                                           int cw) {
  if (row >= srows) return 0u;
  const uint2 w = stage[(row << lct) + t];
  return coef_red<P>(w.x, w.y, cw);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-stream-serialization attribute may become resident while its
// predecessor in the stream still runs; pdl_wait() blocks until that grid has
// completed and its writes are visible, pdl_launch() lets this grid's own
// successor start launching.  Both are no-ops under an ordinary launch.
// Every kernel of the hash calls them first, so completion orders transitively.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// conv kernels run one prime per grid index IDX (primes p0 .. p0 + pn - 1).  Kernels
// without cross-prime data reuse (row, inverse column) put the prime in the
// slowest grid dimension so CTAs resident together run the same prime's
// code: one body is ~20-40 KB of straight-line SASS, and mixing primes on an
// SM starves instruction fetch (ncu: stall_no_instructions dominant).
#define PAB_PRIME_SWITCH(X, IDX) \
  switch (IDX) {                 \
    case 0: X(0); break;         \
    case 1: X(1); break;         \
    case 2: X(2); break;         \
    case 3: X(3); break;         \
    default: X(4); break;        \
  }
static_assert(kNumPrimes == 5, "PAB_PRIME_SWITCH covers five primes");

// four-step twiddle seed w_L^e * 2^32 (Montgomery form, lazy [0, 2p)), e < L
template <int P>
__device__ __forceinline__ u32 tw_seed(const PlanTables& tab, int dir, u32 e) {
  const u32 lo = __ldg(&tab.tlo_m[(P * 2 + dir) * kTwN + (e & (kTwN - 1))]);
  const uint2 hi = __ldg(&tab.thi[(P * 2 + dir) * tab.thi_stride + (e >> kTwLg)]);
  return shoup(lo, hi, PK<P>::p);
}

// column frequency of storage row q: the column DFT (radix-m stage, then
// 2^lgR pow2 DIF) leaves row q = s * 2^lgR + pos holding k1 = s + m * brev(pos)
__device__ __forceinline__ u32 row_k1(int q, int m, int lgR) {
  return (u32)((q >> lgR) + m * brev(q & ((1 << lgR) - 1), lgR));
}

// ---------------------------------------------------------------------------
// Row pass.  CTA: NR = 2^lnr rows of one (block, prime); smem holds the NR
// c-rows (A) then the NR x-rows (X), each sm_len(LGC) words.
// SMALL (lgR == 0): the row is the whole transform; read the operand words,
// write scaled residues.
#ifndef PAB_ROW_REG2_MIN
#define PAB_ROW_REG2_MIN 7  // last row pass keeps A and X in registers together above this lgC (C2 k_row -2%)
#endif
// TW4: the four-step twiddles come from the precomputed tables (tab.tw4) only;
// otherwise either path, chosen by tab.tw4 at run time.  The table-only variant
// keeps the generated path's code out of the instruction stream (k_row<12> is
// ~3.7K instructions per prime).
template <int P, int LGC, bool SMALL, bool TW4 = false>
__device__ __forceinline__ void row_body(const ConvJob& job, const PlanTables& tab, int lnr) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGC);
  constexpr int T = sm_len(LGC);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int NR = 1 << lnr;
  // grid (batch, R / NR, prime): the blocks of a batch run row group q together,
  // so the four-step twiddle rows they share are read from DRAM once (ncu at
  // 3 * 2^20: 1.66 GB of table re-reads per launch with the row group fastest)
  const int b = SMALL ? blockIdx.y : blockIdx.x;
  const int q0 = SMALL ? 0 : (int)(blockIdx.y << lnr);
  const int lgR = job.lgR;
  const long long L = job.L;
  u32* sA = smem;
  u32* sX = smem + NR * T;
  const uint2* twf = tab.stw + (P * 2 + 0) * kTwN;
  const uint2* twi = tab.stw + (P * 2 + 1) * kTwN;
  u32* gA = job.buf + (((long long)b * 2 + 0) * job.np + P) * L;  // also the residue slot
  u32* gX = job.buf + (((long long)b * 2 + 1) * job.np + P) * L;
  const OpView vA = op_view(job, 0, b), vX = op_view(job, 1, b);

  // ---- pass 0: global -> (twiddle) -> DIF top stages -> smem (A and X share twiddles)
  if constexpr (PP.n > 1) {
    for (int task = threadIdx.x; task < (NR << SLO0); task += blockDim.x) {
      const int row = task >> SLO0, o = task & ((1 << SLO0) - 1);
      const int q = q0 + row;
      u32 v[2][1 << RS0];
      if constexpr (SMALL) {
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          const int gi = o + (k << SLO0);
          v[0][k] = coef_at<P>(vA, gi);
          v[1][k] = coef_at<P>(vX, gi);
        }
      } else {
        const u32* ra = gA + ((long long)q << LGC) + o;
        const u32* rx = gX + ((long long)q << LGC) + o;
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          v[0][k] = ra[k << SLO0];
          v[1][k] = rx[k << SLO0];
        }
        if (TW4 || tab.tw4) {  // precomputed Shoup twiddles (coalesced, L2-resident)
          const uint2* tp = tab.tw4 + (long long)(P * 2 + 0) * L + ((long long)q << LGC) + o;
#pragma unroll
          for (int k = 0; k < (1 << RS0); ++k) {
            const uint2 w = __ldg(tp + (k << SLO0));
            v[0][k] = shoup(v[0][k], w, PK<P>::p);
            v[1][k] = shoup(v[1][k], w, PK<P>::p);
          }
        } else {
          const u32 k1 = row_k1(q, job.m, lgR);
          u32 m = tw_seed<P>(tab, 0, (u32)o * k1);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 0) * tab.tstride + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RS0); ++k) {
            v[0][k] = mont<P>(v[0][k], m);
            v[1][k] = mont<P>(v[1][k], m);
            m = shoup(m, gam, PK<P>::p);
          }
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
      if constexpr (PP.n == 1) {  // whole transform in registers, straight from global
        u32 a[1][1 << RSL], x[1][1 << RSL];
        const int q = q0 + row;
        if constexpr (SMALL) {
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            a[0][k] = coef_at<P>(vA, k);
            x[0][k] = coef_at<P>(vX, k);
          }
        } else {
          const u32 k1 = row_k1(q, job.m, lgR);
          u32 m = tw_seed<P>(tab, 0, 0u);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 0) * tab.tstride + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            a[0][k] = mont<P>(gA[((long long)q << LGC) + k], m);
            x[0][k] = mont<P>(gX[((long long)q << LGC) + k], m);
            m = shoup(m, gam, PK<P>::p);
          }
        }
        dif_ct<P, RSL, 1>(a);
        dif_ct<P, RSL, 1>(x);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) x[0][k] = mont<P>(a[0][k], x[0][k]);
        dit_ct<P, RSL>(x[0]);
        if constexpr (SMALL) {
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k)
            if (k < job.nRes)
              gA[k] = red(shoup(x[0][k], tab.scale[P], tab.scale_sh[P], PK<P>::p), PK<P>::p);
        } else {
          const u32 k1 = row_k1(q, job.m, lgR);
          u32 m = tw_seed<P>(tab, 1, 0u);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 1) * tab.tstride + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RSL); ++k) {
            gX[((long long)q << LGC) + k] = mont<P>(red(x[0][k], PK<P>::two_p), m);
            m = shoup(m, gam, PK<P>::p);
          }
        }
      } else if constexpr (LGC > PAB_ROW_REG2_MIN) {
        const int base = row * T + sm_idx(g << RSL);
        u32 a[1][1 << RSL], x[1][1 << RSL];
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) a[0][k] = sA[base + k];
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) x[0][k] = sX[base + k];
        dif_ct<P, RSL, 1>(a);
        dif_ct<P, RSL, 1>(x);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) x[0][k] = mont<P>(a[0][k], x[0][k]);
        dit_ct<P, RSL>(x[0]);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) sX[base + k] = x[0][k];
      } else {
        // lgC <= 8 (measured faster): A and X one after the other (32 live
        // values, not 64; 79 -> 64 registers): A's spectrum goes back to smem
        // and is re-read per point for the pointwise product.
        const int base = row * T + sm_idx(g << RSL);
        u32 v[1][1 << RSL];
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) v[0][k] = sA[base + k];
        dif_ct<P, RSL, 1>(v);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) sA[base + k] = v[0][k];
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) v[0][k] = sX[base + k];
        dif_ct<P, RSL, 1>(v);
        asm volatile("" ::: "memory");  // compiler barrier: re-read A (tasks may be < 32 per warp)
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) v[0][k] = mont<P>(sA[base + k], v[0][k]);
        dit_ct<P, RSL>(v[0]);
#pragma unroll
        for (int k = 0; k < (1 << RSL); ++k) sX[base + k] = v[0][k];
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
        u32* rx = gX + ((long long)q << LGC) + o;
        if (TW4 || tab.tw4) {
          const uint2* tp = tab.tw4 + (long long)(P * 2 + 1) * L + ((long long)q << LGC) + o;
#pragma unroll
          for (int k = 0; k < (1 << RS0); ++k)
            rx[k << SLO0] = shoup(v[k], __ldg(tp + (k << SLO0)), PK<P>::p);
        } else {
          const u32 k1 = row_k1(q, job.m, lgR);
          u32 m = tw_seed<P>(tab, 1, (u32)o * k1);
          const uint2 gam = __ldg(&tab.g[(P * 2 + 1) * tab.tstride + k1]);
#pragma unroll
          for (int k = 0; k < (1 << RS0); ++k) {
            rx[k << SLO0] = mont<P>(red(v[k], PK<P>::two_p), m);
            m = shoup(m, gam, PK<P>::p);
          }
        }
      }
    }
  }
}

template <int LGC, bool SMALL, bool TW4 = false>
__global__ void __launch_bounds__(256) k_row(ConvJob job, PlanTables tab, int lnr) {
  pdl_enter();
#define PAB_B(P_) row_body<P_, LGC, SMALL, TW4>(job, tab, lnr);
  PAB_PRIME_SWITCH(PAB_B, job.p0 + (int)blockIdx.z)
#undef PAB_B
}

// ---------------------------------------------------------------------------
// Column passes.  CTA: CT = 2^lct adjacent columns x R rows, interleaved in
// smem as s[sm_idx(row) * CT + t]; lanes walk columns (coalesced, twiddle
// broadcast).  Forward: operand words -> DIF -> buf; inverse: buf -> DIT ->
// scaled residues.
// LCT >= 0: the tile width is the compile-time col_lct (smem offsets fold into
// immediates: the radix-32 pass's 32 loads were ~5 instructions each with a
// runtime width); -1: runtime lct_in.
template <int P, int LGR, int LGC, bool STAGED = false, int LCT = -1>
__device__ __forceinline__ void col_fwd_body(const ConvJob& job, const PlanTables& tab, int lct_in,
                                             int b, int op, int tile,
                                             const uint2* stage = nullptr,
                                             const uint2* s_tw = nullptr) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int lct = LCT >= 0 ? LCT : lct_in;
  const int CT = 1 << lct;
  constexpr int lgC = LGC;
  const long long L = job.L;
  const int c0 = tile << lct;
  const OpView ov = op_view(job, op, b);
  u32* dst = job.buf + (((long long)b * 2 + op) * job.np + P) * L;
  const uint2* twf = tab.stw + (P * 2 + 0) * kTwN;

  if constexpr (PP.n == 1) {
    for (int t = threadIdx.x; t < CT; t += blockDim.x) {
      u32 v[1][1 << LGR];
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k)
        v[0][k] = coef_at<P>(ov, (k << lgC) + c0 + t);
      dif_ct<P, LGR, 1>(v);
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) dst[((long long)k << lgC) + c0 + t] = v[0][k];
    }
  } else {
    // operand rows >= R/2 are all zero when kc <= L/2 (always for the hash):
    // skip their loads and turn the first DIF stage into one multiply
    const bool half = ov.kc <= (L >> 1);
    const int ilast = ov.kc - 1;
    for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
      const int t = task & (CT - 1), o = task >> lct;
      const int col = c0 + t;
      u32 v[1][1 << RS0];
      if constexpr (STAGED) {  // raw coefficients of rows o + k 2^SLO0 from the staged tile
        constexpr int NK = 1 << RS0;
        if (half) {
#pragma unroll
          for (int k = 0; k < NK / 2; ++k) {
            const uint2 w = stage[((o + (k << SLO0)) << lct) + t];
            v[0][k] = coef_red<P>(w.x, w.y, ov.cw);
          }
          dif_rt_half<P, RS0, SLO0, true>(v, s_tw + o);
        } else {
#pragma unroll
          for (int k = 0; k < NK; ++k) {
            const uint2 w = stage[((o + (k << SLO0)) << lct) + t];
            v[0][k] = coef_red<P>(w.x, w.y, ov.cw);
          }
          dif_rt<P, RS0, SLO0, 1, true>(v, s_tw + o);
        }
      } else if (half) {
        const int g0 = (o << lgC) + col;
        constexpr int kTop = ((1 << (RS0 - 1)) - 1) << (SLO0 + lgC);
        if (g0 + kTop < ilast && ov.cw == 2) {  // every coefficient valid and unmasked:
          // all loads first (8-byte rows: one load each), then the reductions
          uint2 raw[1 << (RS0 - 1)];
          if (ov.a8) {
            const uint2* s2 = reinterpret_cast<const uint2*>(ov.src);
#pragma unroll
            for (int k = 0; k < (1 << (RS0 - 1)); ++k) raw[k] = __ldg(s2 + g0 + (k << (SLO0 + lgC)));
          } else {
#pragma unroll
            for (int k = 0; k < (1 << (RS0 - 1)); ++k) {
              const u32* w = ov.src + 2 * (g0 + (k << (SLO0 + lgC)));
              raw[k] = make_uint2(__ldg(w), __ldg(w + 1));
            }
          }
#pragma unroll
          for (int k = 0; k < (1 << (RS0 - 1)); ++k) v[0][k] = coef_red<P>(raw[k].x, raw[k].y, 2);
        } else if (g0 + kTop < ilast) {
#pragma unroll
          for (int k = 0; k < (1 << (RS0 - 1)); ++k)
            v[0][k] = coef_fast<P>(ov, g0 + (k << (SLO0 + lgC)));
        } else {
#pragma unroll
          for (int k = 0; k < (1 << (RS0 - 1)); ++k)
            v[0][k] = coef_at<P>(ov, g0 + (k << (SLO0 + lgC)));
        }
        dif_rt_half<P, RS0, SLO0>(v, twf + o);
      } else {
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k)
          v[0][k] = coef_at<P>(ov, ((o + (k << SLO0)) << lgC) + col);
        dif_rt<P, RS0, SLO0, 1>(v, twf + o);
      }
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

template <int P, int LGR, int LGC, int LCT = -1>
__device__ __forceinline__ void col_inv_body(const ConvJob& job, const PlanTables& tab,
                                             int lct_in) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR);
  constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
  const int lct = LCT >= 0 ? LCT : lct_in;
  const int CT = 1 << lct;
  const int b = blockIdx.y;  // grid (C / CT, batch, prime)
  constexpr int lgC = LGC;
  const long long L = job.L;
  const int c0 = blockIdx.x << lct;
  const u32* src = job.buf + (((long long)b * 2 + 1) * job.np + P) * L;
  u32* res = job.buf + (((long long)b * 2 + 0) * job.np + P) * L;
  const uint2* twi = tab.stw + (P * 2 + 1) * kTwN;

  if constexpr (PP.n == 1) {
    for (int t = threadIdx.x; t < CT; t += blockDim.x) {
      u32 v[1 << LGR];
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) v[k] = src[((long long)k << lgC) + c0 + t];
      dit_ct<P, LGR>(v);
#pragma unroll
      for (int k = 0; k < (1 << LGR); ++k) {
        const long long gi = ((long long)k << lgC) + c0 + t;
        if (gi < job.nRes) res[gi] = red(red(v[k], PK<P>::two_p), PK<P>::p);  // scale is in the twiddles
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
    // residues are needed only below nRes; when nRes <= L/2 the top DIT stage
    // produces just its lower half
    const bool half = job.nRes <= (L >> 1);
    const int nres = (int)(job.nRes < L ? job.nRes : L);
    for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
      const int t = task & (CT - 1), o = task >> lct;
      const int base = sm_idx(o) * CT + t;
      u32 v[1 << RS0];
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) v[k] = smem[base + k * sm_step(SLO0) * CT];
      if (half) {
        dit_rt_half<P, RS0, SLO0>(v, twi + o);
#pragma unroll
        for (int k = 0; k < (1 << (RS0 - 1)); ++k) {
          const int gi = ((o + (k << SLO0)) << lgC) + c0 + t;
          if (gi < nres) res[gi] = red(red(v[k], PK<P>::two_p), PK<P>::p);  // scale is in the twiddles
        }
      } else {
        dit_rt<P, RS0, SLO0>(v, twi + o);
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          const int gi = ((o + (k << SLO0)) << lgC) + c0 + t;
          if (gi < nres) res[gi] = red(red(v[k], PK<P>::two_p), PK<P>::p);  // scale is in the twiddles
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Mixed-radix column passes: columns of length R = M * 2^LGR2 (M = 3 or 5).
// Forward: radix-M stage over rows {j + t*R2} (from the operand words) with
// twiddles w_R^(j*s) -> M interleaved sub-columns s of length R2 (smem rows
// s*R2 + j) -> pow2 DIF of each -> buf.  Inverse mirrors it.  lgC is runtime.

// one smem->smem pow2 pass over the M sub-transforms (interleaved layout)
template <int P, int M, int LGR2, int RS, int SLO, bool DIF>
__device__ __forceinline__ void colm_pass(u32* smem, int lct, const uint2* __restrict__ tw) {
  const int CT = 1 << lct;
  constexpr int T2 = sm_len(LGR2);
  constexpr int LGG = LGR2 - RS;
  for (int task = threadIdx.x; task < ((CT * M) << LGG); task += blockDim.x) {
    const int t = task & (CT - 1), rest = task >> lct;
    const int g = rest & ((1 << LGG) - 1), s = rest >> LGG;
    const int o = g & ((1 << SLO) - 1), blk = g >> SLO;
    const int base = (s * T2 + sm_idx((blk << (SLO + RS)) + o)) * CT + t;
    u32 v[1][1 << RS];
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) v[0][k] = smem[base + k * sm_step(SLO) * CT];
    if constexpr (DIF) {
      if constexpr (SLO == 0) dif_ct<P, RS, 1>(v);
      else dif_rt<P, RS, SLO, 1>(v, tw + o);
    } else {
      if constexpr (SLO == 0) dit_ct<P, RS>(v[0]);
      else dit_rt<P, RS, SLO>(v[0], tw + o);
    }
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) smem[base + k * sm_step(SLO) * CT] = v[0][k];
  }
}

template <int P, int M, int LGR2, int LGC, bool STAGED = false>
__device__ __forceinline__ void colm_fwd_body(const ConvJob& job, const PlanTables& tab, int lct,
                                             int b, int op, int tile,
                                             const uint2* stage = nullptr, int srows = 0) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR2);
  constexpr int R2 = 1 << LGR2, T2 = sm_len(LGR2);
  const int CT = 1 << lct;
  constexpr int lgC = LGC;
  const long long L = job.L;
  const int c0 = tile << lct;
  const OpView ov = op_view(job, op, b);
  u32* dst = job.buf + (((long long)b * 2 + op) * job.np + P) * L;
  const uint2* twf = tab.stw + (P * 2 + 0) * kTwN;
  const uint2* trad = tab.trad + (P * 2 + 0) * tab.tstride;
  if constexpr (!STAGED) {  // L2 prefetch of this CTA's operand lines (first use is the radix pass)
    const int rows = min((ov.kc + (1 << LGC) - 1) >> LGC, M << LGR2);
    const int lpr = (CT * ov.cw * 4 + 127) >> 7;  // 128-byte lines per row segment
    const char* end = reinterpret_cast<const char*>(ov.src + (size_t)ov.kc * ov.cw);
    for (int i = threadIdx.x; i < rows * lpr; i += blockDim.x) {
      const int row = i / lpr, ln = i - row * lpr;
      const char* p =
          reinterpret_cast<const char*>(ov.src + (size_t)((row << LGC) + c0) * ov.cw) + (ln << 7);
      if (p < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    }
  }
  constexpr bool FUSE = PP.n >= 2 && M * (1 << PP.rs[0]) <= 32;  // register budget
  if constexpr (FUSE) {
    // radix-M stage fused with the first pow2 pass (when M * 2^RS0 <= 32 values fit in
    // registers without losing occupancy): a task (column t, offset o) loads
    // the M * 2^RS0 words of rows {o + k*2^SLO0 + s*R2}, runs the 2^RS0 radix-M DFTs
    // (+ twiddles w_R^(j*s)), then the top RS0 DIF stages of all M sub-columns with
    // shared table twiddles, and stores once to smem.
    constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
    constexpr int NK = 1 << RS0;
    // operand rows >= R/2 are zero when kc <= L/2 (always for the hash): of the
    // radix-M inputs (rows j + s R2, j = o + k 2^SLO0) only sub-columns s < M/2,
    // and s = M/2 for j < R2/2 (k < NK/2), can be nonzero -- compile-time per
    // (s, k), so their loads all issue before any use (ncu at 1e8: the first use
    // of each load was 25% of stall samples) and the known zeros fold away.
    if (ov.kc <= (L >> 1)) {
      const uint2* src2 = reinterpret_cast<const uint2*>(ov.src);
      auto pass = [&](auto s8_c) {
        constexpr bool S8 = decltype(s8_c)::value;
        for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
          const int t = task & (CT - 1), o = task >> lct;
          // every loaded coefficient of the task below kc - 1: no checks, no mask
          const int gtop = ((o + ((NK / 2 - 1) << SLO0) + (M / 2) * R2) << lgC) + c0 + t;
          const bool inner = !STAGED && S8 && gtop < ov.kc - 1;
          uint2 raw[M][NK];
#pragma unroll
          for (int k = 0; k < NK; ++k) {
#pragma unroll
            for (int s = 0; s < M; ++s) {
              raw[s][k] = make_uint2(0u, 0u);
              if (s < M / 2 || (s == M / 2 && k < NK / 2)) {
                const int row = o + (k << SLO0) + s * R2;
                const int gi = (row << lgC) + c0 + t;
                if (STAGED) {  // staged raw words (last one already masked)
                  if (row < srows) raw[s][k] = stage[(row << lct) + t];
                } else if (inner) {
                  raw[s][k] = __ldg(src2 + gi);
                } else if (gi < ov.kc) {
                  if (ov.cw == 2) {
                    // S8: 8-byte rows of whole coefficients (one 8-byte load each)
                    raw[s][k] = S8 ? __ldg(src2 + gi) : ld_coef2(ov, gi, gi == ov.kc - 1);
                  } else {
                    raw[s][k].x = __ldg(ov.src + gi);
                  }
                }
              }
            }
          }
          u32 v[M][NK];
#pragma unroll
          for (int k = 0; k < NK; ++k) {
            const int j = o + (k << SLO0);
            u32 a[M];
#pragma unroll
            for (int s = 0; s < M; ++s) {
              if (s < M / 2 || (s == M / 2 && k < NK / 2)) {
                const int gi = ((j + s * R2) << lgC) + c0 + t;
                uint2 w = raw[s][k];
                if (!STAGED && !inner && gi == ov.kc - 1) {
                  w.x &= ov.mlo;
                  w.y &= ov.mhi;
                }
                a[s] = coef_red<P>(w.x, w.y, ov.cw);
              } else {
                a[s] = 0u;
              }
            }
            radix_m<P, M, false>(a);
#pragma unroll
            for (int s = 0; s < M; ++s)
              v[s][k] = s ? shoup(a[s], __ldg(trad + j * s), PK<P>::p) : a[0];
          }
          dif_rt<P, RS0, SLO0, M>(v, twf + o);
#pragma unroll
          for (int s = 0; s < M; ++s)
#pragma unroll
            for (int k = 0; k < NK; ++k)
              smem[(s * T2 + sm_idx(o + (k << SLO0))) * CT + t] = v[s][k];
        }
      };
      if (ov.cw == 2 && ov.a8 && !ov.odd) {  // S8 = whole 8-byte coefficients only
        pass(std::integral_constant<bool, true>{});
      } else {
        pass(std::integral_constant<bool, false>{});
      }
    } else
    for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
      const int t = task & (CT - 1), o = task >> lct;
      u32 v[M][1 << RS0];
#pragma unroll
      for (int k = 0; k < (1 << RS0); ++k) {
        const int j = o + (k << SLO0);
        u32 a[M];
#pragma unroll
        for (int s = 0; s < M; ++s) {
          a[s] = STAGED ? coef_staged<P>(stage, j + s * R2, t, lct, srows, ov.cw)
                     : coef_at<P>(ov, ((j + s * R2) << lgC) + c0 + t);
        }
        radix_m<P, M, false>(a);
#pragma unroll
        for (int s = 0; s < M; ++s)
          v[s][k] = s ? shoup(a[s], __ldg(trad + j * s), PK<P>::p) : a[0];
      }
      dif_rt<P, RS0, SLO0, M>(v, twf + o);
#pragma unroll
      for (int s = 0; s < M; ++s)
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k)
          smem[(s * T2 + sm_idx(o + (k << SLO0))) * CT + t] = v[s][k];
    }
    __syncthreads();
    if constexpr (PP.n == 3) {
      colm_pass<P, M, LGR2, PP.rs[1], PP.slo[1], true>(smem, lct, twf);
      __syncthreads();
    }
  } else {
  // radix-M stage straight from the operand words.  kc <= L/2 (the hash): rows
  // >= R/2 are zero -- sub-columns s > M/2 always, s = M/2 for j >= R2/2 -- so
  // the two halves of j run as compile-time variants with only the nonzero
  // loads, all issued first (plain 8-byte loads where the task is inside kc - 1)
  auto radix_task = [&](auto hi_c, int task) {
    constexpr bool HI = decltype(hi_c)::value;  // j >= R2/2
    const int t = task & (CT - 1), j = task >> lct;
    constexpr int STOP = HI ? M / 2 : M / 2 + 1;  // sub-columns s < STOP can be nonzero
    const int gtop = ((j + (STOP - 1) * R2) << lgC) + c0 + t;
    const bool fast = ov.cw == 2 && ov.a8 && gtop < ov.kc - 1;
    uint2 raw[M];
#pragma unroll
    for (int s = 0; s < M; ++s) {
      raw[s] = make_uint2(0u, 0u);
      if (s < STOP) {
        const int gi = ((j + s * R2) << lgC) + c0 + t;
        raw[s] = fast ? __ldg(reinterpret_cast<const uint2*>(ov.src) + gi) : coef_raw_at(ov, gi);
      }
    }
    u32 a[M];
#pragma unroll
    for (int s = 0; s < M; ++s) a[s] = s < STOP ? coef_red<P>(raw[s].x, raw[s].y, ov.cw) : 0u;
    radix_m<P, M, false>(a);
#pragma unroll
    for (int s = 1; s < M; ++s) a[s] = shoup(a[s], __ldg(trad + j * s), PK<P>::p);
#pragma unroll
    for (int s = 0; s < M; ++s) smem[(s * T2 + sm_idx(j)) * CT + t] = a[s];
  };
  if (!STAGED && ov.kc <= (L >> 1)) {
    for (int task = threadIdx.x; task < (CT << (LGR2 - 1)); task += blockDim.x)
      radix_task(std::integral_constant<bool, false>{}, task);
    for (int task = (CT << (LGR2 - 1)) + threadIdx.x; task < (CT << LGR2); task += blockDim.x)
      radix_task(std::integral_constant<bool, true>{}, task);
  } else {
  for (int task = threadIdx.x; task < (CT << LGR2); task += blockDim.x) {
    const int t = task & (CT - 1), j = task >> lct;
    u32 a[M];
#pragma unroll
    for (int s = 0; s < M; ++s) {
      a[s] = STAGED ? coef_staged<P>(stage, j + s * R2, t, lct, srows, ov.cw)
                     : coef_at<P>(ov, ((j + s * R2) << lgC) + c0 + t);
    }
    radix_m<P, M, false>(a);
#pragma unroll
    for (int s = 1; s < M; ++s) a[s] = shoup(a[s], __ldg(trad + j * s), PK<P>::p);
#pragma unroll
    for (int s = 0; s < M; ++s) smem[(s * T2 + sm_idx(j)) * CT + t] = a[s];
  }
  }
  __syncthreads();
  if constexpr (PP.n >= 2) {
    colm_pass<P, M, LGR2, PP.rs[0], PP.slo[0], true>(smem, lct, twf);
    __syncthreads();
  }
  if constexpr (PP.n == 3) {
    colm_pass<P, M, LGR2, PP.rs[1], PP.slo[1], true>(smem, lct, twf);
    __syncthreads();
  }
  }
  // last pow2 pass (stages RSL-1..0, compile-time twiddles) -> global rows s*R2 + pos
  constexpr int RSL = PP.rs[PP.n - 1];
  constexpr int LGG = LGR2 - RSL;
  for (int task = threadIdx.x; task < ((CT * M) << LGG); task += blockDim.x) {
    const int t = task & (CT - 1), rest = task >> lct;
    const int g = rest & ((1 << LGG) - 1), s = rest >> LGG;
    const int base = (s * T2 + sm_idx(g << RSL)) * CT + t;
    u32 v[1][1 << RSL];
#pragma unroll
    for (int k = 0; k < (1 << RSL); ++k) v[0][k] = smem[base + k * CT];
    dif_ct<P, RSL, 1>(v);
    u32* d = dst + ((long long)(s * R2 + (g << RSL)) << lgC) + c0 + t;
#pragma unroll
    for (int k = 0; k < (1 << RSL); ++k) d[(long long)k << lgC] = v[0][k];
  }
}

template <int P, int M, int LGR2, int LGC>
__device__ __forceinline__ void colm_inv_body(const ConvJob& job, const PlanTables& tab, int lct) {
  extern __shared__ u32 smem[];
  constexpr PassPlan PP = pass_plan(LGR2);
  constexpr int R2 = 1 << LGR2, T2 = sm_len(LGR2);
  const int CT = 1 << lct;
  const int b = blockIdx.y;  // grid (C / CT, batch, prime)
  constexpr int lgC = LGC;
  const long long L = job.L;
  const int c0 = blockIdx.x << lct;
  const u32* src = job.buf + (((long long)b * 2 + 1) * job.np + P) * L;
  u32* res = job.buf + (((long long)b * 2 + 0) * job.np + P) * L;
  const uint2* twi = tab.stw + (P * 2 + 1) * kTwN;
  const uint2* trad = tab.trad + (P * 2 + 1) * tab.tstride;
  // first pow2 DIT pass (stages 0..RSL-1) from global
  constexpr int RSL = PP.rs[PP.n - 1];
  {
    constexpr int LGG = LGR2 - RSL;
    for (int task = threadIdx.x; task < ((CT * M) << LGG); task += blockDim.x) {
      const int t = task & (CT - 1), rest = task >> lct;
      const int g = rest & ((1 << LGG) - 1), s = rest >> LGG;
      const u32* sp = src + ((long long)(s * R2 + (g << RSL)) << lgC) + c0 + t;
      u32 v[1 << RSL];
#pragma unroll
      for (int k = 0; k < (1 << RSL); ++k) v[k] = sp[(long long)k << lgC];
      dit_ct<P, RSL>(v);
      const int base = (s * T2 + sm_idx(g << RSL)) * CT + t;
#pragma unroll
      for (int k = 0; k < (1 << RSL); ++k) smem[base + k * CT] = v[k];
    }
  }
  __syncthreads();
  if constexpr (PP.n == 3) {
    colm_pass<P, M, LGR2, PP.rs[1], PP.slo[1], false>(smem, lct, twi);
    __syncthreads();
  }
  const int nres = (int)(job.nRes < L ? job.nRes : L);
  constexpr bool FUSE = PP.n >= 2 && M * (1 << PP.rs[0]) <= 32;  // register budget
  if constexpr (FUSE) {
    // top pow2 DIT stages of the M sub-columns fused with the inverse radix-M stage
    constexpr int RS0 = PP.rs[0], SLO0 = PP.slo[0];
    // HALF (nres <= L/2, always for the hash): rows >= R/2 are never stored, which
    // is sub-columns s > M/2, and s = M/2 for j >= R2/2 (k >= NK/2) -- compile-time
    // per (s, k), so their outputs and radix-M arithmetic fold away
    auto pass = [&](auto half_c) {
      constexpr bool HALF = decltype(half_c)::value;
      for (int task = threadIdx.x; task < (CT << SLO0); task += blockDim.x) {
        const int t = task & (CT - 1), o = task >> lct;
        u32 v[M][1 << RS0];
#pragma unroll
        for (int s = 0; s < M; ++s) {
#pragma unroll
          for (int k = 0; k < (1 << RS0); ++k)
            v[s][k] = smem[(s * T2 + sm_idx(o + (k << SLO0))) * CT + t];
          dit_rt<P, RS0, SLO0>(v[s], twi + o);
        }
#pragma unroll
        for (int k = 0; k < (1 << RS0); ++k) {
          const int j = o + (k << SLO0);
          u32 a[M];
          a[0] = red(v[0][k], PK<P>::two_p);
#pragma unroll
          for (int s = 1; s < M; ++s) a[s] = shoup(v[s][k], __ldg(trad + j * s), PK<P>::p);
          radix_m<P, M, true>(a);
#pragma unroll
          for (int s = 0; s < M; ++s) {
            if (HALF && !(s < M / 2 || (s == M / 2 && k < (1 << RS0) / 2))) continue;
            const int gi = ((j + s * R2) << lgC) + c0 + t;
            if (gi < nres) res[gi] = red(a[s], PK<P>::p);  // [0, 2p) -> canonical; scale in the twiddles
          }
        }
      }
    };
    if (job.nRes <= (L >> 1)) {
      pass(std::integral_constant<bool, true>{});
    } else {
      pass(std::integral_constant<bool, false>{});
    }
    return;
  }
  if constexpr (PP.n >= 2) {
    colm_pass<P, M, LGR2, PP.rs[0], PP.slo[0], false>(smem, lct, twi);
    __syncthreads();
  }
  // inverse radix-M stage: twiddle w_R^(-j*s), inverse DFT -> canonical residues.
  // nres <= L/2 (the hash): rows >= R/2 are never stored -- sub-columns s > M/2,
  // and s = M/2 for j >= R2/2 -- so the two halves of j run as compile-time
  // variants and the dead outputs fold away
  auto inv_task = [&](auto mode_c, int task) {
    constexpr int MODE = decltype(mode_c)::value;  // 0: all outputs, 1: j < R2/2, 2: j >= R2/2
    constexpr int STOP = MODE == 0 ? M : (MODE == 1 ? M / 2 + 1 : M / 2);
    const int t = task & (CT - 1), j = task >> lct;
    u32 a[M];
    a[0] = red(smem[sm_idx(j) * CT + t], PK<P>::two_p);
#pragma unroll
    for (int s = 1; s < M; ++s)
      a[s] = shoup(smem[(s * T2 + sm_idx(j)) * CT + t], __ldg(trad + j * s), PK<P>::p);
    radix_m<P, M, true>(a);
#pragma unroll
    for (int s = 0; s < STOP; ++s) {
      const int gi = ((j + s * R2) << lgC) + c0 + t;
      if (gi < nres) res[gi] = red(a[s], PK<P>::p);  // [0, 2p) -> canonical; scale in the twiddles
    }
  };
  if (job.nRes <= (L >> 1)) {
    for (int task = threadIdx.x; task < (CT << (LGR2 - 1)); task += blockDim.x)
      inv_task(std::integral_constant<int, 1>{}, task);
    for (int task = (CT << (LGR2 - 1)) + threadIdx.x; task < (CT << LGR2); task += blockDim.x)
      inv_task(std::integral_constant<int, 2>{}, task);
  } else {
    for (int task = threadIdx.x; task < (CT << LGR2); task += blockDim.x)
      inv_task(std::integral_constant<int, 0>{}, task);
  }
}

template <int M, int LGR2, int LGC>
#ifndef PAB_COLM3_FWD_REGS
#define PAB_COLM3_FWD_REGS 64
#endif
__global__ void __maxnreg__(M == 3 ? PAB_COLM3_FWD_REGS : 48) k_colm_fwd(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  constexpr int lct = col_lct_rows((long long)M << LGR2, LGC);  // compile-time tile width
  if (lct_in != lct) __trap();
  const FwdIdx ix = fwd_idx(job, lct);
#define PAB_B(P_) colm_fwd_body<P_, M, LGR2, LGC>(job, tab, lct, ix.b, ix.op, ix.tile);
  PAB_PRIME_SWITCH(PAB_B, ix.prime)
#undef PAB_B
}
template <int M, int LGR2, int LGC>
__global__ void __launch_bounds__(512) k_colm_inv(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  constexpr int lct = col_lct_rows((long long)M << LGR2, LGC);  // compile-time tile width
  if (lct_in != lct) __trap();
#define PAB_B(P_) colm_inv_body<P_, M, LGR2, LGC>(job, tab, lct);
  PAB_PRIME_SWITCH(PAB_B, job.p0 + (int)blockIdx.z)
#undef PAB_B
}

template <int LGR, int LGC>
__global__ void __launch_bounds__(256, 5) k_col_fwd(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  constexpr int LCT = col_lct(LGR, LGC);
  if (lct_in != LCT) __trap();  // the launcher's width is this constant
  const FwdIdx ix = fwd_idx(job, LCT);
#define PAB_B(P_) col_fwd_body<P_, LGR, LGC, false, LCT>(job, tab, LCT, ix.b, ix.op, ix.tile);
  PAB_PRIME_SWITCH(PAB_B, ix.prime)
#undef PAB_B
}
// All primes of one (block, operand, column tile) per CTA: the raw operand tile
// is staged once (cp.async) and transformed for each prime in turn.  1-D grid:
// tile fastest, then operand, then block.  Dynamic smem: the transform panel
// plus the stage (rows x CT x 8 bytes).
template <int LGR, int LGC>
__global__ void __launch_bounds__(256) k_col_fwd_all(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  extern __shared__ u32 smem[];
  constexpr int lct = col_lct(LGR, LGC);
  if (lct_in != lct) __trap();  // the launcher's width is this constant
  constexpr int CT = 1 << lct;
  const unsigned tc = 1u << (LGC - lct);
  const int tile = (int)(blockIdx.x % tc);
  const int rest = (int)(blockIdx.x / tc);
  const int op = rest & 1, b = rest >> 1;
  const OpView ov = op_view(job, op, b);
  const bool half = ov.kc <= (job.L >> 1);
  const int rows = half ? (1 << (LGR - 1)) : (1 << LGR);
  uint2* stage = reinterpret_cast<uint2*>(smem + sm_len(LGR) * CT);
  // the first pass's stage twiddles (entries < 2^(SLO0 + RS0)) of every prime
  constexpr PassPlan PP = pass_plan(LGR);
  constexpr int NTW = 1 << (PP.slo[0] + PP.rs[0]);
  uint2* s_tw = stage + (rows << lct);
  for (int i = threadIdx.x; i < job.np * NTW; i += blockDim.x)
    s_tw[i] = __ldg(tab.stw + ((i / NTW) * 2) * kTwN + (i % NTW));
  stage_operand<lct>(ov, stage, rows, lct, LGC, tile << lct);  // (its barrier covers s_tw too)
  // small launches (few blocks) spread the primes over grid.y, one per CTA
  const int q0 = gridDim.y > 1 ? job.p0 + (int)blockIdx.y : job.p0;
  const int qn = gridDim.y > 1 ? 1 : job.pn;
  sfor<kNumPrimes>([&](auto pc) {
    constexpr int P = decltype(pc)::value;
    if (P >= q0 && P < q0 + qn) {
      col_fwd_body<P, LGR, LGC, true, lct>(job, tab, lct, b, op, tile, stage, s_tw + P * NTW);
      __syncthreads();  // the next prime reuses the transform panel
    }
  });
}

// Mixed radix, all primes per CTA: stages the operand rows holding nonzero
// coefficients (row < ceil(kc / C)) once, then each prime's radix-M + pow2
// column DFT reads them from smem.
template <int M, int LGR2, int LGC>
__global__ void __maxnreg__(48) k_colm_fwd_all(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  extern __shared__ u32 smem[];
  // half-width tiles (the launcher's lcta), compile-time
  constexpr int lct = col_lct_rows((long long)M << LGR2, LGC) - 1 < 2
                          ? 2 : col_lct_rows((long long)M << LGR2, LGC) - 1;
  if (lct_in != lct) __trap();
  constexpr int CT = 1 << lct;
  const unsigned tc = 1u << (LGC - lct);
  const int tile = (int)(blockIdx.x % tc);
  const int rest = (int)(blockIdx.x / tc);
  const int op = rest & 1, b = rest >> 1;
  const OpView ov = op_view(job, op, b);
  const int R = M << LGR2;
  int rows = (ov.kc + (1 << LGC) - 1) >> LGC;
  if (rows > R) rows = R;
  uint2* stage = reinterpret_cast<uint2*>(smem + M * sm_len(LGR2) * CT);
  stage_operand(ov, stage, rows, lct, LGC, tile << lct);
  const int q0 = gridDim.y > 1 ? job.p0 + (int)blockIdx.y : job.p0;  // as k_col_fwd_all
  const int qn = gridDim.y > 1 ? 1 : job.pn;
  sfor<kNumPrimes>([&](auto pc) {
    constexpr int P = decltype(pc)::value;
    if (P >= q0 && P < q0 + qn) {
      colm_fwd_body<P, M, LGR2, LGC, true>(job, tab, lct, b, op, tile, stage, rows);
      __syncthreads();  // the next prime reuses the transform panel
    }
  });
}

template <int LGR, int LGC>
__global__ void __launch_bounds__(256) k_col_inv(ConvJob job, PlanTables tab, int lct_in) {
  pdl_enter();
  constexpr int LCT = col_inv_lct(LGR, LGC);
  if (lct_in != LCT) __trap();  // the launcher's width is this constant
#define PAB_B(P_) col_inv_body<P_, LGR, LGC, LCT>(job, tab, LCT);
  PAB_PRIME_SWITCH(PAB_B, job.p0 + (int)blockIdx.z)
#undef PAB_B
}


// Each size compiles only what can run: forward column passes in the variant
// the launcher uses for it (all-primes staged for pow2 columns up to 2^8 and
// mixed radix up to 2^7 per sub-column, per-prime above), no clamped duplicates.
template <int LG, int DC>
void set_colm(ConvKernels& k) {  // mixed radix, columns of M * 2^LG, rows 2^(LG + 2 + DC)
  constexpr int C = LG + 2 + DC;
  if constexpr (C <= 12) {
    k.colm_inv[0][DC] = k_colm_inv<3, LG, C>;
    k.colm_inv[1][DC] = k_colm_inv<5, LG, C>;
    if constexpr (LG <= 7) {
      k.colm_fwd_all[0][DC] = k_colm_fwd_all<3, LG, C>;
      k.colm_fwd_all[1][DC] = k_colm_fwd_all<5, LG, C>;
    } else {
      k.colm_fwd[0][DC] = k_colm_fwd<3, LG, C>;
      k.colm_fwd[1][DC] = k_colm_fwd<5, LG, C>;
    }
  }
}

template <int LG>
ConvKernels make_conv_kernels() {
  ConvKernels k{};
  k.row = k_row<LG, false>;
  k.row_small = k_row<LG, true>;
  // table-only variant where the generated path's code costs i-cache (lgC = 12:
  // k_row -2%); at lgC <= 11 ptxas schedules it in fewer registers and it loses 1-3%
  if constexpr (LG == 12) k.row_tw4 = k_row<LG, false, true>;
  if constexpr (LG >= 6) {
    k.col_inv = k_col_inv<LG, LG>;
    if constexpr (LG <= 8) {
      k.col_fwd_all = k_col_fwd_all<LG, LG>;
    } else {
      k.col_fwd = k_col_fwd<LG, LG>;
    }
    if constexpr (LG < 12) {
      k.col_inv1 = k_col_inv<LG, LG + 1>;
      if constexpr (LG <= 8) {
        k.col_fwd_all1 = k_col_fwd_all<LG, LG + 1>;
      } else {
        k.col_fwd1 = k_col_fwd<LG, LG + 1>;
      }
    }
  }
  if constexpr (LG >= 3 && LG <= 10) {
    set_colm<LG, 0>(k);
    set_colm<LG, 1>(k);
    set_colm<LG, 2>(k);
  }
  return k;
}

}  // namespace pab

// one translation unit per size: defines conv_kernels_<LG>()
#define PAB_DEFINE_CONV(LG) \
  namespace pab {           \
  ConvKernels conv_kernels_##LG() { return make_conv_kernels<LG>(); } \
  }
