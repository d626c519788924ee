// In-shared-memory batched NTT passes ("panels").
//
// A panel holds several transforms of length N = 2^lgN in one of two layouts,
// both with one pad word per 16 elements of a transform:
//  * interleaved (column passes): element i of transform t at
//    ((i + i/16) << lnc) + t; tasks are numbered transform-fastest, so the
//    lanes of a warp walk adjacent columns (coalesced global access, twiddle
//    broadcast);
//  * transform-major (row passes): element i of transform t at
//    t * tstride + i + i/16; tasks are numbered group-fastest.
// Every radix pass starts at a stage that is a multiple of 4, which together
// with the padding keeps the strided register passes bank-conflict free.
//
// A transform of lgN stages is run as radix-2^RS register passes (RS <= 4):
// each thread task loads 2^RS elements at stride 2^s_lo, performs RS
// butterfly stages in registers, and stores them back.  Stage twiddles come
// from a per-prime table tw[h + e] = w_{2h}^{+-e} (Shoup pairs), h = 2^stage,
// for sub-transforms of up to 4096 points.  Tasks are numbered transform-
// fastest, so when a panel holds >= 32 transforms (column passes) all lanes of
// a warp read the same twiddle (broadcast).
//
// This replaces the reference's radix-2 _transform over Z/(2^N'+1)
// (pkg/src/modpa/ntt.py:178-201): DIF here is the forward transform (natural
// order in, bit-reversed out) and DIT with inverse twiddles the inverse
// (bit-reversed in, natural out), so no bit-reversal permutation is ever done.
#pragma once
#include "modarith.cuh"

namespace pab {

__device__ __forceinline__ int pidx(int i, int t, int lnc) {
  return ((i + (i >> 4)) << lnc) + t;
}
__host__ __device__ constexpr int tm_stride(int lgN) { return (1 << lgN) + ((1 << lgN) >> 4); }
__device__ __forceinline__ int tidx(int i, int t, int lgN) { return t * tm_stride(lgN) + i + (i >> 4); }
__host__ __device__ constexpr int panel_words(int lgN, int lnc) {
  return ((1 << lgN) + ((1 << lgN) >> 4)) << lnc;
}

// RS DIF stages (s = s_lo+RS-1 down to s_lo) on registers v[k] = x[base + o + k*2^s_lo].
template <int RS, bool LAST>
__device__ __forceinline__ void dif_regs(u32 (&v)[1 << RS], int o, int s_lo,
                                         const uint2* __restrict__ tw, u32 p, u32 two_p) {
#pragma unroll
  for (int st = 0; st < RS; ++st) {
    const int hr = 1 << (RS - 1 - st);
    const int sg = RS - 1 - st;  // stage index relative to s_lo
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) {
      if (k & hr) continue;
      if (LAST) {  // s_lo == 0 and o == 0: twiddle index is compile-time
        const int e = k & (hr - 1);
        if (e == 0) {
          dif_bfly1(v[k], v[k + hr], two_p);
        } else {
          uint2 w = __ldg(&tw[(1 << sg) + e]);
          dif_bfly(v[k], v[k + hr], w, p, two_p);
        }
      } else {
        const int e = o + ((k & (hr - 1)) << s_lo);
        uint2 w = __ldg(&tw[(1 << (sg + s_lo)) + e]);
        dif_bfly(v[k], v[k + hr], w, p, two_p);
      }
    }
  }
}

// RS DIT stages (s = s_lo up to s_lo+RS-1); inverse twiddle table.
template <int RS, bool FIRST>
__device__ __forceinline__ void dit_regs(u32 (&v)[1 << RS], int o, int s_lo,
                                         const uint2* __restrict__ tw, u32 p, u32 two_p) {
#pragma unroll
  for (int st = 0; st < RS; ++st) {
    const int hr = 1 << st;
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) {
      if (k & hr) continue;
      if (FIRST) {
        const int e = k & (hr - 1);
        if (e == 0) {
          dit_bfly1(v[k], v[k + hr], two_p);
        } else {
          uint2 w = __ldg(&tw[(1 << st) + e]);
          dit_bfly(v[k], v[k + hr], w, p, two_p);
        }
      } else {
        const int e = o + ((k & (hr - 1)) << s_lo);
        uint2 w = __ldg(&tw[(1 << (st + s_lo)) + e]);
        dit_bfly(v[k], v[k + hr], w, p, two_p);
      }
    }
  }
}

// Geometry of one register pass inside a panel.
struct PassGeo {
  int lgN;    // transform length log2
  int s_lo;   // lowest stage of this pass
  int lnt;    // log2 #transforms processed
  int lnc;    // log2 panel interleave (interleaved layout only)
  int tmul;   // physical transform index = t*tmul + toff
  int toff;
};

template <bool TM>
__device__ __forceinline__ int paddr(const PassGeo& g, int i, int t) {
  return TM ? tidx(i, t, g.lgN) : pidx(i, t, g.lnc);
}

template <int RS, bool TM>
__device__ __forceinline__ void task_pos(const PassGeo& g, int task, int& t, int& o, int& base) {
  int tl, grp;
  if (TM) {
    const int lg_groups = g.lgN - RS;
    tl = task >> lg_groups;
    grp = task & ((1 << lg_groups) - 1);
  } else {
    tl = task & ((1 << g.lnt) - 1);
    grp = task >> g.lnt;
  }
  t = tl * g.tmul + g.toff;
  o = grp & ((1 << g.s_lo) - 1);
  const int blk = grp >> g.s_lo;
  base = (blk << (g.s_lo + RS)) + o;
}

template <int RS, bool TM>
__device__ void panel_dif_pass(u32* s, const PassGeo g, const uint2* __restrict__ tw, u32 p,
                               u32 two_p) {
  const int tasks = 1 << (g.lgN - RS + g.lnt);
  for (int task = threadIdx.x; task < tasks; task += blockDim.x) {
    int t, o, base;
    task_pos<RS, TM>(g, task, t, o, base);
    u32 v[1 << RS];
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) v[k] = s[paddr<TM>(g, base + (k << g.s_lo), t)];
    if (g.s_lo == 0)
      dif_regs<RS, true>(v, 0, 0, tw, p, two_p);
    else
      dif_regs<RS, false>(v, o, g.s_lo, tw, p, two_p);
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) s[paddr<TM>(g, base + (k << g.s_lo), t)] = v[k];
  }
}

template <int RS, bool TM>
__device__ void panel_dit_pass(u32* s, const PassGeo g, const uint2* __restrict__ tw, u32 p,
                               u32 two_p) {
  const int tasks = 1 << (g.lgN - RS + g.lnt);
  for (int task = threadIdx.x; task < tasks; task += blockDim.x) {
    int t, o, base;
    task_pos<RS, TM>(g, task, t, o, base);
    u32 v[1 << RS];
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) v[k] = s[paddr<TM>(g, base + (k << g.s_lo), t)];
    if (g.s_lo == 0)
      dit_regs<RS, true>(v, 0, 0, tw, p, two_p);
    else
      dit_regs<RS, false>(v, o, g.s_lo, tw, p, two_p);
#pragma unroll
    for (int k = 0; k < (1 << RS); ++k) s[paddr<TM>(g, base + (k << g.s_lo), t)] = v[k];
  }
}

// Number of stages in the first (top) pass when lg stages are split in 4s.
__host__ __device__ constexpr int first_pass_stages(int lg) { return lg - 4 * ((lg - 1) / 4); }

// Full forward DIF over a panel (all transforms selected by lnt/tmul/toff).
template <bool TM>
__device__ __forceinline__ void panel_dif(u32* s, int lgN, int lnt, int lnc, int tmul, int toff,
                                          const uint2* __restrict__ tw, u32 p, u32 two_p) {
  int s_hi = lgN - 1;
  int rs = first_pass_stages(lgN);
  while (s_hi >= 0) {
    PassGeo g{lgN, s_hi - rs + 1, lnt, lnc, tmul, toff};
    switch (rs) {
      case 1: panel_dif_pass<1, TM>(s, g, tw, p, two_p); break;
      case 2: panel_dif_pass<2, TM>(s, g, tw, p, two_p); break;
      case 3: panel_dif_pass<3, TM>(s, g, tw, p, two_p); break;
      default: panel_dif_pass<4, TM>(s, g, tw, p, two_p); break;
    }
    __syncthreads();
    s_hi -= rs;
    rs = 4;
  }
}

// Full inverse DIT over a panel (no 1/N scaling).
template <bool TM>
__device__ __forceinline__ void panel_dit(u32* s, int lgN, int lnt, int lnc, int tmul, int toff,
                                          const uint2* __restrict__ tw, u32 p, u32 two_p) {
  const int top = first_pass_stages(lgN);
  int s_lo = 0;
  while (s_lo < lgN) {
    const int rs = (lgN - s_lo == top) ? top : 4;
    PassGeo g{lgN, s_lo, lnt, lnc, tmul, toff};
    switch (rs) {
      case 1: panel_dit_pass<1, TM>(s, g, tw, p, two_p); break;
      case 2: panel_dit_pass<2, TM>(s, g, tw, p, two_p); break;
      case 3: panel_dit_pass<3, TM>(s, g, tw, p, two_p); break;
      default: panel_dit_pass<4, TM>(s, g, tw, p, two_p); break;
    }
    __syncthreads();
    s_lo += rs;
  }
}

}  // namespace pab
