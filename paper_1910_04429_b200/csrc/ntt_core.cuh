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

// primitive 2^23-th roots of unity (and inverses) of kPrimes (generator^((p-1)/2^23))
constexpr u32 kRoot23[kNumPrimes] = {15311432u, 872686320u, 273508579u};
constexpr u32 kIRoot23[kNumPrimes] = {469870224u, 354917575u, 109748732u};

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
// w_{2^lgo}^e (INV: inverse root)
__host__ __device__ constexpr u32 croot(int P, bool inv, int lgo, u64 e) {
  return cpow(inv ? kIRoot23[P] : kRoot23[P], e << (23 - lgo), kPrimes[P]);
}

template <int P>
struct PK {
  static constexpr u32 p = kPrimes[P];
  static constexpr u32 two_p = 2u * kPrimes[P];
  static constexpr u32 p_mont = cmont_neg_inv(kPrimes[P]);
  static constexpr u32 one_sh = cshoup(1u, kPrimes[P]);
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
  } else if (rem == 6) {
    parts[np++] = 3;
    parts[np++] = 3;
  } else {  // rem == 7 (lg 12)
    parts[np++] = 3;
    parts[np++] = 4;
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
template <int P, int RS, int SLO, int NV>
__device__ __forceinline__ void dif_rt(u32 (&v)[NV][1 << RS], const uint2* __restrict__ two) {
  sfor<RS>([&](auto st_) {
    constexpr int st = decltype(st_)::value;
    constexpr int sg = RS - 1 - st;
    constexpr int hr = 1 << sg;
    sfor<(1 << RS)>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      if constexpr ((k & hr) == 0) {
        constexpr int off = (1 << (sg + SLO)) + ((k & (hr - 1)) << SLO);
        const uint2 w = __ldg(two + off);
#pragma unroll
        for (int j = 0; j < NV; ++j) bf_dif<P>(v[j][k], v[j][k + hr], w.x, w.y);
      }
    });
  });
}

// As dif_rt, but the upper half of the inputs (k >= 2^(RS-1)) is known to be
// zero (zero-padded operand): the first stage is y = x * w, x unchanged.
template <int P, int RS, int SLO>
__device__ __forceinline__ void dif_rt_half(u32 (&v)[1][1 << RS], const uint2* __restrict__ two) {
  constexpr int H = 1 << (RS - 1);
  sfor<H>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    constexpr int off = (1 << (RS - 1 + SLO)) + (k << SLO);
    const uint2 w = __ldg(two + off);
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
        const uint2 w = __ldg(two + off);
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

}  // namespace pab
