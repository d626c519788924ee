// Kernel-facing data structures and launchers for the PA hash pipeline.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "modarith.cuh"

namespace pab {

// Device twiddle tables for one plan (one transform length L = 2^lg).
// All arrays are [prime][dir] with dir 0 = forward (w), 1 = inverse (w^-1).
struct PlanTables {
  const uint2* stw;    // [3][2][4096] stage twiddles tw[h+e] = w_{2h}^e, Shoup pairs
  const u32* tlo_m;    // [3][2][4096] Montgomery form of w_L^e, e < 4096
  const uint2* thi;    // [3][2][4096] Shoup pairs of w_L^(4096 j)
  u32 scale[3];        // L^-1 * 2^32 mod p (undoes the transform length and the
  u32 scale_sh[3];     // Montgomery factor of the pointwise product), Shoup pair
};

struct CrtConst {
  u32 p0, p1, p2;
  u32 inv01, inv01_sh;     // p0^-1 mod p1
  u32 p0m2, p0m2_sh;       // p0 mod p2
  u32 inv012, inv012_sh;   // (p0 p1)^-1 mod p2
  u64 p0p1;
};

// One convolution-product job over a batch of independent blocks:
//   T = (A * X + D) mod 2^n_mod_bits (as words), out = T >> shift (mw words).
struct ConvJob {
  int batch;
  int lg, lgR, lgC;            // L = 2^lg = R * C (R = 1: single-pass path)
  long long kA, kX, kD;        // valid input words per block (A, X, D)
  long long in_stride;         // words between consecutive blocks' operand slots
  const u32* words;            // [batch][3][in_stride]: slot 0 = A, 1 = X, 2 = D
  u32* buf;                    // [batch][2][3][L] transform buffers
  long long nT;                // T words computed
  long long nRes;              // residues stored (min(nT, L))
  long long n_mod_bits;        // T is reduced mod 2^n_mod_bits
  long long shift;             // output = T >> shift
  long long mw;                // output words per block
  u32* out_words;              // [batch][mw]
  unsigned long long* tile_state;  // [batch][tiles] look-back states (zeroed)
  u32* tile_ctr;               // [batch] tile tickets (zeroed)
  int tiles;                   // carry tiles per block
};

constexpr int kCarryThreads = 256;
constexpr int kCarryItems = 8;
constexpr int kCarryTile = kCarryThreads * kCarryItems;

void upload_constants(const PrimeInfo* primes, const CrtConst& crt);

// bytes (LSF or MSF) -> u32 words, zero-padded to kw words, bits >= n cleared.
void launch_pack(const uint8_t* in, long long in_stride_bytes, long long n_bits, int msf,
                 int batch, u32* words, long long word_stride, long long kw, cudaStream_t st);
// u32 words -> ceil(m/8) bytes per block (LSF or MSF).
void launch_unpack(const u32* words, long long word_stride, long long m_bits, int msf, int batch,
                   uint8_t* out, long long out_stride_bytes, cudaStream_t st);
// transform + pointwise + inverse -> residues in buf slot A; then carry.
void launch_conv(const ConvJob& job, const PlanTables& tab, cudaStream_t st);
void launch_carry(const ConvJob& job, cudaStream_t st);

}  // namespace pab
