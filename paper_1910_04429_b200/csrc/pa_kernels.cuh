// Kernel-facing data structures and launchers for the PA hash pipeline.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "modarith.cuh"

namespace pab {

// Device twiddle tables for one plan (one transform length L = m * 2^lg).
// Arrays are [prime][dir][...] with dir 0 = forward (w), 1 = inverse (w^-1);
// primes whose 2-adicity is below lg have zero entries (unused: cw = 1 jobs).
struct PlanTables {
  const uint2* stw;    // stage twiddles tw[h+e] = w_{2h}^e (Shoup pairs), h <= 2048
  const u32* tlo_m;    // [5][2][4096] Montgomery form of w_L^e, e < 4096
  const uint2* thi;    // [5][2][thi_stride] Shoup pairs of w_L^(4096 j)
  const uint2* g;      // [5][2][R] Shoup pairs of w_L^(k1 * 2^slo0(lgC)), k1 < R (row twiddle step)
  const uint2* trad;   // [5][2][R] Shoup pairs of w_R^e, e < R (radix-m column stage), or null
  int tstride;         // R: stride of g and trad
  int thi_stride;      // stride of thi (>= L / 4096)
  const uint2* tw4;    // [5][2][L] full four-step twiddles w_L^(+-c*brev(q)) at [q*C + c],
                       // Shoup pairs; only for small L (L2-resident), else null
  u32 scale[kNumPrimes];     // L^-1 * 2^32 mod p: undoes the length and the Montgomery
  u32 scale_sh[kNumPrimes];  // factor of the pointwise product (Shoup companions)
};

// One convolution-product job over a batch of independent blocks:
//   T = (A * X + D) mod 2^n_mod_bits (as 32-bit words), out = T >> shift.
struct ConvJob {
  int batch;
  int cw;                      // words per coefficient: 2 (five primes) or 1 (three primes)
  int np;                      // primes (buffer layout, CRT): 5 if cw == 2 else 3
  int p0, pn;                  // primes [p0, p0 + pn) this job's convolution computes
                               // (all of them unless the primes are split over GPUs)
  int m;                       // radix of the column length: L = m * 2^lg
  int lg, lgR, lgC;            // R = m * 2^lgR rows (columns of length R), C = 2^lgC
  long long L;                 // transform length (R = 1: single-CTA path)
  // operands as little-endian 32-bit words; block b at src + b * src_stride
  const u32* srcA;
  const u32* srcX;
  const u32* srcD;             // may be null (no addend)
  long long src_stride;        // in words (even when cw == 2: 8-byte aligned coefficients)
  long long kA, kX, kD;        // valid words per block
  u32 maskA, maskX, maskD;     // applied to the last valid word (bits >= n)
  u32* buf;                    // [batch][2][np][L] transform buffers (slot A reused for residues)
  long long nT;                // T words computed
  long long nRes;              // residues stored per prime (coefficients: <= L)
  long long n_mod_bits;        // T is reduced mod 2^n_mod_bits
  long long shift;             // output = T >> shift
  long long mw;                // output words per block
  u32* out_words;              // [batch][mw], or null: write LSF bytes directly
  uint8_t* out_bytes;          // block b at out_bytes + b * out_stride, rbytes each
  long long out_stride;
  long long rbytes;
  unsigned long long* tile_state;  // [batch][tiles] look-back states (zeroed)
  u32* tile_ctr;               // [batch] tile tickets (zeroed)
  int tiles;                   // carry tiles per block
  int fwd_chunk;               // forward column pass: blocks per L2-resident chunk (grid order)
};

// Column-pass tile widths (columns per CTA, log2), shared by the launcher and the
// kernels so the kernels can take them as compile-time constants.
__host__ __device__ constexpr int col_lct(int lgR, int lgC) {
  int lct = 14 - lgR;  // ~16K words per CTA
  if (lct > 5) lct = 5;
  if (lct < 13 - lgR) lct = 13 - lgR;  // the radix-32 pass has >= 256 tasks (one per thread)
  if (lct < 3) lct = 3;
  if (lct > lgC) lct = lgC;
  return lct;
}
// pow2 inverse: half-width tiles in 128-thread CTAs while >= 32 columns wide
__host__ __device__ constexpr int col_inv_lct(int lgR, int lgC) {
  return col_lct(lgR, lgC) - (col_lct(lgR, lgC) >= 6 ? 1 : 0);
}
__host__ __device__ constexpr int col_lct_rows(long long R, int lgC) {  // ~16K words per CTA
  int lct = 5;
  while (lct > 3 && (R << lct) > 16384) --lct;
  if (lct > lgC) lct = lgC;
  return lct;
}

constexpr int kCarryWarps = 8;                           // warps per carry CTA
constexpr int kCarryRows = 8;                            // 32-word rows per warp
constexpr int kCarryThreads = 32 * kCarryWarps;
constexpr int kCarryTile = 32 * kCarryWarps * kCarryRows;  // words per tile
constexpr int kCarryTileMin = 1000;  // smallest tile of any carry kernel (sizes the look-back state)

constexpr int kTinyBits = 2048;  // single-warp schoolbook path (n <= kTinyBits)

void launch_tiny(const uint8_t* x, const uint8_t* c, const uint8_t* d, long long stride, int n_bits,
                 int r_bits, int msf, int batch, uint8_t* out, long long out_stride,
                 cudaStream_t st);
void set_kernel_attrs();

// bytes (LSF or MSF) -> u32 words, zero-padded to kw words, bits >= n cleared.
void launch_pack(const uint8_t* in, long long in_stride_bytes, long long n_bits, int msf,
                 int batch, u32* words, long long word_stride, long long kw, cudaStream_t st);
// u32 words -> ceil(m/8) bytes per block (LSF or MSF).
void launch_unpack(const u32* words, long long word_stride, long long m_bits, int msf, int batch,
                   uint8_t* out, long long out_stride_bytes, cudaStream_t st);
// CPython 30-bit int digits (least significant first) <-> u32 words.
struct DigitOperands {
  const u32* d[3];
  long long nd[3];  // digits present (beyond: zero)
};
void launch_digits_pack(const DigitOperands& ops, int nops, long long n_bits, u32* words,
                        long long word_stride, long long kw, cudaStream_t st);
void launch_digits_unpack(const u32* words, long long m_bits, u32* dig, long long nd,
                          cudaStream_t st);
// forward transforms + pointwise + inverse -> residues in buf slot A.
void launch_conv(const ConvJob& job, const PlanTables& tab, cudaStream_t st);
// CRT + carry + mask + shift -> output.
void launch_carry(const ConvJob& job, cudaStream_t st);
// gen_seed(n, derive_block_seed(master, first + j)) for j < batch on the GPU
// (SHAKE-256, pkg/src/modpa/pa.py:138-172): c and d rows at j * stride bytes,
// ceil(n/8) bytes each in byte order msf; word_io = LSF rows 8-byte aligned.
constexpr int kMaxSeedMaster = 1024;  // master seed material bytes (kernel parameter)
struct SeedMaster {
  uint8_t b[kMaxSeedMaster];
};
// fixed_index >= 0: the bench protocol -- block j's material is the integer
// first + j and the derive_block_seed label index is fixed_index (master unused)
void launch_seed_expand(const SeedMaster& master, int mlen, unsigned long long first, int batch,
                        long long n_bits, int msf, int word_io, uint8_t* c, uint8_t* d,
                        long long stride, cudaStream_t st, long long fixed_index = -1);
void seed_expand_raw(const SeedMaster& master, int mlen, unsigned long long first, int batch,
                     long long n_bits, int msf, int word_io, uint8_t* c, uint8_t* d,
                     long long stride, cudaStream_t st, long long fixed_index);
// a kernel set exists for this geometry (L = m * 2^(lgR + lgC))
bool conv_supported(int m, int lgR, int lgC);

}  // namespace pab
