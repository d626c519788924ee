// Fused convolution for L = 2^15 on a cluster of two CTAs (thread-block
// cluster + distributed shared memory, sm_100a).
//
// The four-step path (k_col_fwd -> k_row -> k_col_inv) passes each block's
// transforms through HBM three times.  At L = 2^15 (n up to 1,048,576 bits:
// BASELINE C1 / C2) one transform is 128 KB of residues, so a (block, prime)
// pair fits on two SMs: CTA r of the cluster holds the spectrum of operand r
// (0: c, 1: x) in its own shared memory, and the two CTAs finish the product
// together through DSMEM:
//
//   1. each CTA: its operand's coefficients -> 15 DIF stages in smem
//      (radix-32 register passes over stages 14..10, 9..5, 4..0; natural in,
//      bit-reversed out); the top stage is a multiply, the upper half being zero;
//   2. cluster barrier;
//   3. CTA r owns spectrum half r: pointwise Montgomery product of its own and
//      the peer's spectrum (one DSMEM load per point), then DIT stages 0..13
//      of that half in its own smem;
//   4. cluster barrier;
//   5. DIT stage 14 for the low half of the outputs only (coefficients < L/2:
//      the hash keeps K' <= L/2), split over the two CTAs, one operand local and
//      one remote; residues [0, p) to the workspace slot the carry kernel reads.
//
// The L^-1 * 2^32 scale (length and the Montgomery factor of the pointwise
// product) rides in operand c's coefficient reduction (two Shoup products,
// as the unscaled reduction already costs).  HBM traffic per (block, prime):
// the two operands in, K' residues out.
//
// Reference: the whole of ssa_multiply's transform part, pkg/src/modpa/ntt.py:178-284
// (forward_ntt x2, pointwise_mul, inverse_ntt), restated as one exact
// cyclic convolution modulo one NTT prime.
#include <cooperative_groups.h>

#include "conv_kernels.cuh"

namespace cg = cooperative_groups;

namespace pab {

namespace {

constexpr int kLg = 15;
constexpr int kL = 1 << kLg;
constexpr int kHalf = kL / 2;

// coefficient gi of the operand, times `s` mod p (s in Shoup form for the low
// and the high word), in [0, 2p); zero at or beyond kc, the last one masked
template <int P>
__device__ __forceinline__ u32 coef_scaled(const OpView& o, int gi, u32 s_lo, u32 s_lo_sh,
                                           u32 s_hi, u32 s_hi_sh) {
  const uint2 w = coef_raw_at(o, gi);
  return red(shoup(w.x, s_lo, s_lo_sh, PK<P>::p) + shoup(w.y, s_hi, s_hi_sh, PK<P>::p),
             PK<P>::two_p);
}

template <int P>
__device__ __forceinline__ void fused_body(const ConvJob& job, const PlanTables& tab, int b) {
  extern __shared__ u32 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();  // 0: operand c (A), 1: operand x (X)
  const int t = threadIdx.x;
  const uint2* twf = tab.stwL + (P * 2 + 0) * kL;  // tw[h + e] = w_2h^e, h < 2^14
  const uint2* twi = tab.stwL + (P * 2 + 1) * kL;

  // ---- 1. forward DIF of operand r
  {
    const OpView ov = op_view(job, r, b);
    // c carries L^-1 * 2^32 (undone by the transforms and the Montgomery product)
    const u32 s_lo = r ? 1u : tab.scale[P], s_lo_sh = r ? PK<P>::one_sh : tab.scale_sh[P];
    const u32 s_hi = r ? PK<P>::r32 : tab.scale2[P];
    const u32 s_hi_sh = r ? PK<P>::r32_sh : tab.scale2_sh[P];
    // pass F1, stages 14..10: elements t + 1024 k; k >= 16 are the zero upper half
    u32 v[1][32];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[0][k] = coef_scaled<P>(ov, t + (k << 10), s_lo, s_lo_sh, s_hi, s_hi_sh);
    dif_rt_half<P, 5, 10>(v, twf + t);
#pragma unroll
    for (int k = 0; k < 32; ++k) smem[sm_idx(t + (k << 10))] = v[0][k];
  }
  __syncthreads();
  {  // pass F2, stages 9..5: elements 1024 blk + o + 32 k
    const int o = t & 31, base = (t >> 5) * 1024 + o;
    u32 v[1][32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[0][k] = smem[sm_idx(base + (k << 5))];
    dif_rt<P, 5, 5, 1>(v, twf + o);
#pragma unroll
    for (int k = 0; k < 32; ++k) smem[sm_idx(base + (k << 5))] = v[0][k];
  }
  __syncthreads();
  {  // pass F3, stages 4..0: 32 contiguous elements (compile-time twiddles)
    const int base = t * 32;
    u32 v[1][32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[0][k] = smem[sm_idx(base + k)];
    dif_ct<P, 5, 1>(v);
#pragma unroll
    for (int k = 0; k < 32; ++k) smem[sm_idx(base + k)] = v[0][k];
  }
  // ---- 2. both spectra complete
  cl.sync();
  const u32* peer = cl.map_shared_rank(smem, r ^ 1);
  const int h0 = r * kHalf;  // this CTA's half of the (bit-reversed) spectrum
  // ---- 3. pointwise product + DIT stages 0..13 of half r (overwrites only
  // this CTA's half r; the peer reads half r ^ 1 of this CTA's smem)
  if (t < kHalf / 32) {  // pass I1: 32 contiguous points, stages 0..4
    const int base = h0 + t * 32;
    u32 v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int i = sm_idx(base + k);
      v[k] = mont<P>(smem[i], peer[i]);
    }
    dit_ct<P, 5>(v);
#pragma unroll
    for (int k = 0; k < 32; ++k) smem[sm_idx(base + k)] = v[k];
  }
  __syncthreads();
  if (t < kHalf / 32) {  // pass I2, stages 5..9: elements h0 + 1024 blk + o + 32 k
    const int o = t & 31, base = h0 + (t >> 5) * 1024 + o;
    u32 v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = smem[sm_idx(base + (k << 5))];
    dit_rt<P, 5, 5>(v, twi + o);
#pragma unroll
    for (int k = 0; k < 32; ++k) smem[sm_idx(base + (k << 5))] = v[k];
  }
  __syncthreads();
  {  // pass I3, stages 10..13: elements h0 + t + 1024 k, k < 16 (all threads)
    const int base = h0 + t;
    u32 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = smem[sm_idx(base + (k << 10))];
    dit_rt<P, 4, 10>(v, twi + t);
#pragma unroll
    for (int k = 0; k < 16; ++k) smem[sm_idx(base + (k << 10))] = v[k];
  }
  // ---- 4. both halves through stage 13
  cl.sync();
  // ---- 5. stage 14, low outputs only: out[k] = a_k + w^-k b_k, a_k in CTA 0's
  // half 0, b_k in CTA 1's half 1; CTA r writes k in [r 2^13, (r + 1) 2^13)
  {
    const u32* lo = r ? peer : smem;
    const u32* hi = r ? smem : peer;
    u32* res = job.buf + (((long long)b * 2 + 0) * job.np + P) * job.L;
    const int nres = (int)job.nRes;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = r * (kHalf / 2) + t + (k << 10);
      const uint2 w = __ldg(twi + kHalf + i);
      const u32 a = red(lo[sm_idx(i)], PK<P>::two_p);
      const u32 x = a + shoup(hi[sm_idx(kHalf + i)], w, PK<P>::p);
      if (i < nres) res[i] = red(red(x, PK<P>::two_p), PK<P>::p);
    }
  }
  cl.sync();  // the peer may still be reading this CTA's smem
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1)
    k_conv_fused15(ConvJob job, PlanTables tab) {
  const int b = blockIdx.x >> 1;
#define PAB_B(P_) fused_body<P_>(job, tab, b);
  PAB_PRIME_SWITCH(PAB_B, job.p0 + (int)blockIdx.y)
#undef PAB_B
}

}  // namespace

size_t fused15_smem_bytes() { return (size_t)sm_len(kLg) * 4; }

bool fused15_applies(const ConvJob& job, const PlanTables& tab) {
  if (job.m != 1 || job.L != kL || job.cw != 2 || !tab.stwL) return false;
  const long long ka = (job.kA + 1) / 2, kx = (job.kX + 1) / 2;  // coefficients
  return ka <= kHalf && kx <= kHalf && job.nRes <= kHalf;
}

void set_fused15_attrs() {
  cudaFuncSetAttribute(k_conv_fused15, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused15_smem_bytes());
}

void launch_fused15(const ConvJob& job, const PlanTables& tab, cudaStream_t st) {
  k_conv_fused15<<<dim3(2 * job.batch, job.pn), 1024, fused15_smem_bytes(), st>>>(job, tab);
}

}  // namespace pab
