// Compile-time-specialised NTT building blocks (prime P, transform size, pass
// geometry are template parameters, so moduli and all small-stage twiddles
// become SASS immediates and every smem address is base + immediate).
//
// Transforms of length N = 2^LG run as radix-2^RS register passes:
//   * the last DIF pass (first DIT pass) always covers stages 0..4 (RS = 5,
//     s_lo = 0) with compile-time twiddles;
//   * the remaining stages run in passes of <= 4 stages whose lowest stage
//     s_lo >= 5, with twiddles read from the stage table tw[h + e] = w_{2h}^e.
// Shared-memory index of element i is i + i/32 (one pad word per 32): with
// s_lo in {0} U [5, ..] every lane pattern below is bank-conflict free.
//
// Reference counterpart: _transform / forward_ntt / inverse_ntt
// (pkg/src/modpa/ntt.py:178-222); DIF = forward (natural -> bit-reversed),
// DIT with inverse roots = inverse (bit-reversed -> natural), unscaled.
#pragma once
#include <utility>

#include "modarith.cuh"

namespace pab {

__host__ __device__ constexpr u32 cmul(u32 a, u32 b, u32 p) { return (u32)((u64)a * b % p); }
__host__ __device__ constexpr u32 cpow(u32 a, u64 e, u32 p) {
  u32 r = 1;
  while (e) {
    if (e & 1) r = cmul(r, a, p);
    a = cmul(a, a, p);
    e >>= 1;
  }
  return r;
}
__host__ __device__ constexpr u32 cshoup(u32 w, u32 p) { return (u32)(((u64)w << 32) / p); }
__host__ __device__ constexpr u32 cmont_neg_inv(u32 p) {
  u32 inv = 1;
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  return 0u - inv;
}
// w_N^e with w_N = g^((p-1)/N) (INV: w_N^-e); all roots derive from one generator
__host__ __device__ constexpr u32 croot_n(int P, bool inv, u64 N, u64 e) {
  const u32 p = kPrimes[P];
  const u64 x = (u64)(p - 1) / N * (e % N);
  return cpow(kGen[P], inv ? (u64)(p - 1) - x : x, p);
}
// w_{2^lgo}^e
__host__ __device__ constexpr u32 croot(int P, bool inv, int lgo, u64 e) {
  return croot_n(P, inv, (u64)1 << lgo, e);
}

template <int P>
struct PK {
  static constexpr u32 p = kPrimes[P];
  static constexpr u32 two_p = 2u * kPrimes[P];
  static constexpr u32 p_mont = cmont_neg_inv(kPrimes[P]);
  static constexpr u32 one_sh = cshoup(1u, kPrimes[P]);
  static constexpr u32 r32 = (u32)((1ull << 32) % kPrimes[P]);  // 2^32 mod p
  static constexpr u32 r32_sh = cshoup(r32, kPrimes[P]);
};

// ------------------------------------------------------------ static for
template <int... Is, class F>
__device__ __forceinline__ void sfor_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(std::make_integer_sequence<int, N>{}, f);
}

// ------------------------------------------------------------ pass plans
struct PassPlan {
  int n;       // number of passes
  int rs[3];   // stages per pass, DIF order (pass 0 = top stages)
  int slo[3];  // lowest stage of each pass
};
__host__ __device__ constexpr PassPlan pass_plan(int lg) {
  PassPlan pp{1, {lg, 0, 0}, {0, 0, 0}};
  if (lg <= 5) return pp;
  const int rem = lg - 5;
  int parts[2] = {0, 0};
  int np = 0;
  if (rem <= 4) {
    parts[np++] = rem;
  } else if (rem == 5) {
    parts[np++] = 3;
    parts[np++] = 2;
  } else if (rem == 6) {  // lg 11, 12: the heavier pass first (measured: k_row -5%)
    parts[np++] = 4;
    parts[np++] = 2;
  } else {  // rem == 7 (lg 12)
    parts[np++] = 4;
    parts[np++] = 3;
  }
  int s = lg;
  for (int i = 0; i < np; ++i) {
    s -= parts[i];
    pp.rs[i] = parts[i];
    pp.slo[i] = s;
  }
  pp.rs[np] = 5;
  pp.slo[np] = 0;
  pp.n = np + 1;
  return pp;
}

__host__ __device__ constexpr int sm_idx(int i) { return i + (i >> 5); }
__host__ __device__ constexpr int sm_len(int lg) { return (1 << lg) + ((1 << lg) >> 5); }
// smem distance between consecutive elements of a register group at stride 2^slo
__host__ __device__ constexpr int sm_step(int slo) { return slo >= 5 ? (1 << slo) + (1 << (slo - 5)) : (1 << slo); }

// ------------------------------------------------------------ butterflies
template <int P>
__device__ __forceinline__ void bf_dif(u32& x, u32& y, u32 w, u32 wp) {
  const u32 s = red(x + y, PK<P>::two_p);
  const u32 d = x - y + PK<P>::two_p;
  y = d * w - __umulhi(d, wp) * PK<P>::p;
  x = s;
}
template <int P>
__device__ __forceinline__ void bf_dif1(u32& x, u32& y) {
  const u32 s = red(x + y, PK<P>::two_p);
  y = red(x - y + PK<P>::two_p, PK<P>::two_p);
  x = s;
}
template <int P>
__device__ __forceinline__ void bf_dit(u32& x, u32& y, u32 w, u32 wp) {
  const u32 a = red(x, PK<P>::two_p);
  const u32 t = y * w - __umulhi(y, wp) * PK<P>::p;
  x = a + t;
  y = a - t + PK<P>::two_p;
}
template <int P>
__device__ __forceinline__ void bf_dit1(u32& x, u32& y) {
  const u32 a = red(x, PK<P>::two_p);
  const u32 t = red(y, PK<P>::two_p);
  x = a + t;
  y = a - t + PK<P>::two_p;
}
template <int P>
__device__ __forceinline__ u32 mont(u32 a, u32 b) { return montmul(a, b, PK<P>::p, PK<P>::p_mont); }

// DIF over RS stages with compile-time twiddles (s_lo = 0, o = 0); NV vectors.
template <int P, int RS, int NV>
__device__ __forceinline__ void dif_ct(u32 (&v)[NV][1 << RS]) {
  sfor<RS>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int hr = 1 << (RS - 1 - st);
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int e = k & (hr - 1);
        if constexpr (e == 0) {
#pragma unroll
          for (int j = 0; j < NV; ++j) bf_dif1<P>(v[j][k], v[j][k + hr]);
        } else {
          constexpr u32 w = croot(P, false, RS - st, e);
          constexpr u32 wp = cshoup(w, kPrimes[P]);
#pragma unroll
          for (int j = 0; j < NV; ++j) bf_dif<P>(v[j][k], v[j][k + hr], w, wp);
        }
      }
    });
  });
}

// DIT over RS stages (0..RS-1) with compile-time inverse twiddles.
template <int P, int RS>
__device__ __forceinline__ void dit_ct(u32 (&v)[1 << RS]) {
  sfor<RS>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int hr = 1 << st;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int e = k & (hr - 1);
        if constexpr (e == 0) {
          bf_dit1<P>(v[k], v[k + hr]);
        } else {
          constexpr u32 w = croot(P, true, st + 1, e);
          constexpr u32 wp = cshoup(w, kPrimes[P]);
          bf_dit<P>(v[k], v[k + hr], w, wp);
        }
      }
    });
  });
}

// DIF over stages SLO+RS-1 .. SLO with table twiddles; two = tw + o.
// (SMEM: `two` points into shared memory -- plain loads instead of __ldg)
template <int P, int RS, int SLO, int NV, bool SMEM = false>
__device__ __forceinline__ void dif_rt(u32 (&v)[NV][1 << RS], const uint2* __restrict__ two) {
  sfor<RS>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int sg = RS - 1 - st;
    constexpr int hr = 1 << sg;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int off = (1 << (sg + SLO)) + ((k & (hr - 1)) << SLO);
        const uint2 w = SMEM ? two[off] : __ldg(two + off);
#pragma unroll
        for (int j = 0; j < NV; ++j) bf_dif<P>(v[j][k], v[j][k + hr], w.x, w.y);
      }
    });
  });
}

// As dif_rt, but the upper half of the inputs (k >= 2^(RS-1)) is known to be
// zero (zero-padded operand): the first stage is y = x * w, x unchanged.
template <int P, int RS, int SLO, bool SMEM = false>
__device__ __forceinline__ void dif_rt_half(u32 (&v)[1][1 << RS], const uint2* __restrict__ two) {
  constexpr int H = 1 << (RS - 1);
  sfor<H>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    constexpr int off = (1 << (RS - 1 + SLO)) + (k << SLO);
    const uint2 w = SMEM ? two[off] : __ldg(two + off);
    v[0][k + H] = v[0][k] * w.x - __umulhi(v[0][k], w.y) * PK<P>::p;
  });
  sfor<RS - 1>([&](auto st_) {
    constexpr int st = decltype(st_)::value + 1;
    constexpr int sg = RS - 1 - st;
    constexpr int hr = 1 << sg;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int off = (1 << (sg + SLO)) + ((k & (hr - 1)) << SLO);
        const uint2 w = SMEM ? two[off] : __ldg(two + off);
        bf_dif<P>(v[0][k], v[0][k + hr], w.x, w.y);
      }
    });
  });
}

// DIT over stages SLO .. SLO+RS-1 with table (inverse) twiddles; two = tw + o.
template <int P, int RS, int SLO>
__device__ __forceinline__ void dit_rt(u32 (&v)[1 << RS], const uint2* __restrict__ two) {
  sfor<RS>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int hr = 1 << st;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int off = (1 << (st + SLO)) + ((k & (hr - 1)) << SLO);
        const uint2 w = __ldg(two + off);
        bf_dit<P>(v[k], v[k + hr], w.x, w.y);
      }
    });
  });
}

// As dit_rt, but only the lower half of the outputs (k < 2^(RS-1)) is needed:
// the last stage computes x + w*y only.
template <int P, int RS, int SLO>
__device__ __forceinline__ void dit_rt_half(u32 (&v)[1 << RS], const uint2* __restrict__ two) {
  sfor<RS - 1>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int hr = 1 << st;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int off = (1 << (st + SLO)) + ((k & (hr - 1)) << SLO);
        const uint2 w = __ldg(two + off);
        bf_dit<P>(v[k], v[k + hr], w.x, w.y);
      }
    });
  });
  constexpr int H = 1 << (RS - 1);
  sfor<H>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    constexpr int off = (1 << (RS - 1 + SLO)) + (k << SLO);
    const uint2 w = __ldg(two + off);
    const u32 a = red(v[k], PK<P>::two_p);
    v[k] = a + (v[k + H] * w.x - __umulhi(v[k + H], w.y) * PK<P>::p);
  });
}

// ------------------------------------------------------------ radix 3 / 5
// Length-M DFT of a[0..M) in place (INV: inverse roots), inputs in [0, 2p),
// outputs in [0, 2p).  Radix-3: y1,2 = a0 - s/2 +- c (a1 - a2), c = (w - w^2)/2.
// Radix-5: with u_k = a_k + a_{5-k}, v_k = a_k - a_{5-k}, C_k = (w^k + w^-k)/2,
// S_k = (w^k - w^-k)/2:  y1,4 = a0 + C1 u1 + C2 u2 +- (S1 v1 + S2 v2),
// y2,3 = a0 + C2 u1 + C1 u2 +- (S2 v1 - S1 v2).  Every product is a Shoup
// multiply by a compile-time constant.
template <int P, bool INV>
__device__ __forceinline__ void radix3(u32 (&a)[3]) {
  constexpr u32 p = kPrimes[P], tp = 2u * kPrimes[P];
  constexpr u32 h = (p + 1u) / 2u;  // 1/2
  constexpr u32 w1 = croot_n(P, INV, 3, 1), w2 = croot_n(P, INV, 3, 2);
  constexpr u32 c = cmul((w1 + p - w2) % p, h, p);
  constexpr u32 hs = cshoup(h, p), cs = cshoup(c, p);
  const u32 s = red(a[1] + a[2], tp);
  const u32 d = a[1] - a[2] + tp;
  const u32 y0 = red(a[0] + s, tp);
  const u32 t1 = s * h - __umulhi(s, hs) * p;
  const u32 t2 = d * c - __umulhi(d, cs) * p;
  const u32 u = red(a[0] - t1 + tp, tp);
  a[0] = y0;
  a[1] = red(u + t2, tp);
  a[2] = red(u - t2 + tp, tp);
}

template <int P, bool INV>
__device__ __forceinline__ void radix5(u32 (&a)[5]) {
  constexpr u32 p = kPrimes[P], tp = 2u * kPrimes[P];
  constexpr u32 h = (p + 1u) / 2u;
  constexpr u32 w1 = croot_n(P, INV, 5, 1), w2 = croot_n(P, INV, 5, 2);
  constexpr u32 w3 = croot_n(P, INV, 5, 3), w4 = croot_n(P, INV, 5, 4);
  constexpr u32 C1 = cmul((w1 + w4) % p, h, p), C2 = cmul((w2 + w3) % p, h, p);
  constexpr u32 S1 = cmul((w1 + p - w4) % p, h, p), S2 = cmul((w2 + p - w3) % p, h, p);
  constexpr u32 C1s = cshoup(C1, p), C2s = cshoup(C2, p), S1s = cshoup(S1, p),
                S2s = cshoup(S2, p);
  const u32 u1 = a[1] + a[4], v1 = a[1] - a[4] + tp;  // < 4p
  const u32 u2 = a[2] + a[3], v2 = a[2] - a[3] + tp;
  const u32 y0 = red(a[0] + red(red(u1, tp) + red(u2, tp), tp), tp);
  const u32 t1 = red((u1 * C1 - __umulhi(u1, C1s) * p) + (u2 * C2 - __umulhi(u2, C2s) * p), tp);
  const u32 t2 = red((u1 * C2 - __umulhi(u1, C2s) * p) + (u2 * C1 - __umulhi(u2, C1s) * p), tp);
  const u32 s1 = red((v1 * S1 - __umulhi(v1, S1s) * p) + (v2 * S2 - __umulhi(v2, S2s) * p), tp);
  const u32 s2 = red((v1 * S2 - __umulhi(v1, S2s) * p) - (v2 * S1 - __umulhi(v2, S1s) * p) + tp,
                     tp);
  const u32 b1 = red(a[0] + t1, tp), b2 = red(a[0] + t2, tp);
  a[0] = y0;
  a[1] = red(b1 + s1, tp);
  a[4] = red(b1 - s1 + tp, tp);
  a[2] = red(b2 + s2, tp);
  a[3] = red(b2 - s2 + tp, tp);
}

template <int P, int M, bool INV>
__device__ __forceinline__ void radix_m(u32 (&a)[M]) {
  if constexpr (M == 3) radix3<P, INV>(a);
  else if constexpr (M == 5) radix5<P, INV>(a);
}

}  // namespace pab
