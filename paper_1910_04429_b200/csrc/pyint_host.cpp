// Host-side layout conversions of the drop-in boundary: CPython int digits
// (30-bit payload in 32-bit slots, least significant first) <-> serialized
// blocks (ceil(n/8) bytes, LSF or MSF, pkg/src/modpa/pa.py:111-132).
//
// The reference's import_block / export_block are int.from_bytes /
// int.to_bytes; these do the same conversion at memory speed: four 30-bit
// digits are exactly 15 bytes, so the loops move 120-bit groups.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/pa_b200.h"

namespace {
constexpr uint32_t kMask30 = 0x3FFFFFFFu;

inline uint32_t dig_at(const uint32_t* d, uint64_t nd, uint64_t i) { return i < nd ? d[i] : 0u; }

#if defined(__x86_64__)
// 8 digits -> 30 bytes per 256-bit vector: pairs (d0 | d1 << 30) in 64-bit lanes,
// then (a | b << 60, b >> 4) per 128-bit half = 15 bytes each.  Returns the
// number of 30-byte groups written (stops 2 bytes early: each half stores 16).
__attribute__((target("avx2"))) uint64_t digits_to_bytes_avx2(const uint32_t* dig, uint64_t nd,
                                                              uint8_t* out, uint64_t nbytes) {
  const __m256i m30 = _mm256_set1_epi64x(0x3FFFFFFFll);
  const __m256i mhi = _mm256_set1_epi64x(0x0FFFFFFFC0000000ll);
  const __m256i keep_lo = _mm256_set_epi64x(0, -1, 0, -1);
  uint64_t g = 0;
  for (; 8 * g + 8 <= nd && 30 * g + 32 <= nbytes; ++g) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(dig + 8 * g));
    const __m256i t = _mm256_or_si256(_mm256_and_si256(x, m30),
                                      _mm256_and_si256(_mm256_srli_epi64(x, 2), mhi));
    const __m256i u = _mm256_unpackhi_epi64(_mm256_slli_epi64(t, 60), _mm256_srli_epi64(t, 4));
    const __m256i r = _mm256_or_si256(_mm256_and_si256(t, keep_lo), u);
    uint8_t* p = out + 30 * g;
    _mm_storeu_si128(reinterpret_cast<__m128i*>(p), _mm256_castsi256_si128(r));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(p + 15), _mm256_extracti128_si256(r, 1));
  }
  return g;
}
// (evaluated while the library loads, before main: run the CPU detection first)
const bool kHasAvx2 = [] {
  __builtin_cpu_init();
  return __builtin_cpu_supports("avx2") != 0;
}();
#endif

// 15-byte groups [g0, g1) <-> digits [4 g0, 4 g1); every store stays inside the
// groups' bytes, so ranges can run on different threads
void d2b_groups(const uint32_t* dig, uint64_t nd, uint8_t* out, uint64_t g0, uint64_t g1) {
  uint64_t g = g0;
#if defined(__x86_64__)
  if (kHasAvx2)
    g += 2 * digits_to_bytes_avx2(dig + 4 * g0, nd > 4 * g0 ? nd - 4 * g0 : 0, out + 15 * g0,
                                  15 * (g1 - g0));
#endif
  for (; g < g1; ++g) {  // 4 digits -> 15 bytes
    const uint64_t i = 4 * g;
    uint32_t d0, d1, d2, d3;
    if (i + 4 <= nd) {
      d0 = dig[i], d1 = dig[i + 1], d2 = dig[i + 2], d3 = dig[i + 3];
    } else {
      d0 = dig_at(dig, nd, i), d1 = dig_at(dig, nd, i + 1), d2 = dig_at(dig, nd, i + 2),
      d3 = dig_at(dig, nd, i + 3);
    }
    const uint64_t lo = (uint64_t)d0 | ((uint64_t)d1 << 30) | ((uint64_t)d2 << 60);
    const uint64_t hi = ((uint64_t)d2 >> 4) | ((uint64_t)d3 << 26);  // 56 bits
    uint8_t* p = out + 15 * g;
    const uint64_t up = (lo >> 56) | (hi << 8);  // bytes 7 .. 14 (one overlapping 8-byte store)
    std::memcpy(p, &lo, 8);
    std::memcpy(p + 7, &up, 8);
  }
}

void b2d_groups(const uint8_t* in, uint32_t* dig, uint64_t g0, uint64_t g1) {
  for (uint64_t g = g0; g < g1; ++g) {  // 15 bytes -> 4 digits
    const uint8_t* p = in + 15 * g;
    uint64_t lo, hi;
    std::memcpy(&lo, p, 8);
    std::memcpy(&hi, p + 7, 8);  // bytes 7 .. 14
    hi >>= 8;
    uint32_t* d = dig + 4 * g;
    d[0] = (uint32_t)lo & kMask30;
    d[1] = (uint32_t)(lo >> 30) & kMask30;
    d[2] = (uint32_t)((lo >> 60) | (hi << 4)) & kMask30;
    d[3] = (uint32_t)(hi >> 26) & kMask30;
  }
}

// run f(g0, g1) over [0, groups): on up to 8 threads above 4 MB (one thread moves
// ~2-10 GB/s here; a 10^8-bit operand is 12.5 MB), chunks of an even group count
template <class F>
void over_groups(uint64_t groups, F f) {
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = 15 * groups < ((uint64_t)4 << 20) || hw < 2 ? 1u : (hw > 8 ? 8u : hw);
  if (nt == 1) {
    f(0, groups);
    return;
  }
  const uint64_t per = ((groups + nt - 1) / nt + 1) & ~1ull;
  std::vector<std::thread> th;
  for (uint64_t g0 = 0; g0 < groups; g0 += per)
    th.emplace_back(f, g0, g0 + per < groups ? g0 + per : groups);
  for (auto& t : th) t.join();
}
}  // namespace

extern "C" {

int pab_digits_to_bytes(const uint32_t* dig, uint64_t nd, uint8_t* out, uint64_t nbytes,
                        int byte_order) {
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF) return PAB_EINVAL;
  if ((nd && !dig) || (nbytes && !out)) return PAB_EINVAL;
  const uint64_t groups = nbytes / 15;
  over_groups(groups, [&](uint64_t g0, uint64_t g1) { d2b_groups(dig, nd, out, g0, g1); });
  // tail: fewer than 15 bytes
  uint64_t acc = 0;
  int have = 0;
  uint64_t i = 4 * groups;
  for (uint64_t k = 15 * groups; k < nbytes; ++k) {
    if (have < 8) {
      acc |= (uint64_t)dig_at(dig, nd, i++) << have;
      have += 30;
    }
    out[k] = (uint8_t)acc;
    acc >>= 8;
    have -= 8;
  }
  if (byte_order == PAB_ORDER_MSF) std::reverse(out, out + nbytes);
  return PAB_OK;
}

int pab_bytes_to_digits(const uint8_t* in, uint64_t nbytes, int byte_order, uint32_t* dig,
                        uint64_t nd) {
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF) return PAB_EINVAL;
  if ((nbytes && !in) || (nd && !dig)) return PAB_EINVAL;
  const bool msf = byte_order == PAB_ORDER_MSF;
  auto byte_at = [&](uint64_t k) -> uint64_t {  // LSF byte k
    return k < nbytes ? (msf ? in[nbytes - 1 - k] : in[k]) : 0u;
  };
  uint64_t i = 0;
  if (!msf) {
    const uint64_t full = std::min(nd / 4, nbytes / 15);  // whole 15-byte groups
    over_groups(full, [&](uint64_t g0, uint64_t g1) { b2d_groups(in, dig, g0, g1); });
    i = 4 * full;
  }
  for (; i < nd; ++i) {  // bits [30 i, 30 i + 30) byte by byte
    const uint64_t b0 = 30 * i;
    const uint64_t k0 = b0 >> 3;
    const int sh = (int)(b0 & 7);
    uint64_t v = 0;
    for (int q = 0; q < 5; ++q) v |= byte_at(k0 + q) << (8 * q);
    dig[i] = (uint32_t)(v >> sh) & kMask30;
  }
  return PAB_OK;
}

}  // extern "C"
