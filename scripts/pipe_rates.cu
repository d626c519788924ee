// Per-instruction issue cost of the integer ops the NTT butterflies use, on B200.
// Each mode is a stream of independent chains of one instruction (or a fixed mix);
// the result is warp-instructions per clock per SM sub-partition (SMSP).  Built and
// run by scripts/gpu_pipe_rates.sh; output kept as profiles/r2/pipe_rates.json.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kChains = 8;

enum Mode {
  M_IMAD = 0,     // mad.lo.u32
  M_HI,           // mul.hi.u32 (IMAD.HI.U32)
  M_WIDE,         // mul.wide.u32, both halves consumed (IMAD.WIDE.U32)
  M_IADD3,        // add (IADD3)
  M_VMNMX,        // add + min fused (VIADDMNMX.U32)
  M_LOP3,         // lop3
  M_SHOUP,        // mul.hi + mul.lo + mad.lo (the Shoup product alone)
  M_BFLY,         // full DIF butterfly: IADD, VIADDMNMX, IADD3, HI, LO, MAD
  M_IMAD_IADD,    // 1 IMAD : 1 IADD3 (both pipes, expect 2x)
  M_HI_IADD2,     // 1 HI : 2 IADD3
  M_HI_IADD4,     // 1 HI : 4 IADD3
  M_WIDE_IADD2,   // 1 WIDE : 2 IADD3
  M_MONT,         // Montgomery product (WIDE, LO, HI + 3 alu)
  M_SHOUP_WIDE,   // 1 HI : 1 LOP3
  M_BFLY_ASM,     // the butterfly with its two-operand add pinned as add.u32 (stays IADD3)
  M_IADD3_IMM,    // three-operand IADD3 (register + register + immediate)
  M_SUB,          // two-register subtract
  M_COUNT
};

template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains], b[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = seed * (threadIdx.x + 17 * i + 1);
    b[i] = seed ^ (i * 0x9E3779B9u + threadIdx.x);
  }
  const uint32_t p = 943718401u, tp = 2u * p;
  uint32_t w = seed * 77u + 12345u, wp = seed * 99u + 54321u, pm = seed * 3u + 0xdeadbeefu;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      uint32_t x = a[i], y = b[i];
      if (MODE == M_IMAD) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(w), "r"(wp));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y) : "r"(w), "r"(wp));
      } else if (MODE == M_HI) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(wp));
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
      } else if (MODE == M_WIDE) {
        // one WIDE + one LOP3 (alu pipe) per product, so no register-pair moves are needed
        uint64_t t = (uint64_t)x * wp;
        x = (uint32_t)t ^ (uint32_t)(t >> 32);
        t = (uint64_t)y * w;
        y = (uint32_t)t ^ (uint32_t)(t >> 32);
      } else if (MODE == M_IADD3) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(w));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
      } else if (MODE == M_VMNMX) {
        x = min(x, x - tp);
        y = min(y, y - tp);
      } else if (MODE == M_LOP3) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(w), "r"(wp));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y) : "r"(w), "r"(wp));
      } else if (MODE == M_SHOUP) {
        uint32_t q = __umulhi(x, wp);
        x = x * w - q * p;
        q = __umulhi(y, wp);
        y = y * w - q * p;
      } else if (MODE == M_BFLY) {
        uint32_t s = x + y;
        s = min(s, s - tp);
        uint32_t d = x - y + tp;
        uint32_t q = __umulhi(d, wp);
        y = d * w - q * p;
        x = s;
      } else if (MODE == M_IMAD_IADD) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(w), "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
      } else if (MODE == M_HI_IADD2) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(w));
      } else if (MODE == M_HI_IADD4) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(w));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(w));
      } else if (MODE == M_WIDE_IADD2) {
        uint32_t lo;
        asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %2; mov.b64 {%1, %0}, t;}" : "+r"(x), "=r"(lo) : "r"(wp));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(lo));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y) : "r"(w));
      } else if (MODE == M_MONT) {
        uint64_t t = (uint64_t)x * y;
        uint32_t lo = (uint32_t)t, hi = (uint32_t)(t >> 32);
        uint32_t m = lo * pm;
        uint32_t mh = __umulhi(m, p);
        y = hi + mh + (lo != 0u ? 1u : 0u);
        x = min(y + x, y + x - tp);
      } else if (MODE == M_BFLY_ASM) {
        uint32_t s;
        asm volatile("add.u32 %0, %1, %2;" : "=r"(s) : "r"(x), "r"(y));
        s = min(s, s - tp);
        uint32_t d = x - y + tp;
        uint32_t q = __umulhi(d, wp);
        y = d * w - q * p;
        x = s;
      } else if (MODE == M_IADD3_IMM) {
        x = x + y + 0x1234u;
        y = y + x + 0x77u;
      } else if (MODE == M_SUB) {
        asm volatile("sub.u32 %0, %0, %1;" : "+r"(x) : "r"(w));
        asm volatile("sub.u32 %0, %0, %1;" : "+r"(y) : "r"(wp));
      } else if (MODE == M_SHOUP_WIDE) {  // 1 HI : 1 LOP3
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(wp));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y) : "r"(w), "r"(wp));
      }
      a[i] = x;
      b[i] = y;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc ^= a[i] ^ b[i];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
double run(int sms, int mhz, double warp_instr_per_inner) {
  uint32_t* d;
  cudaMalloc(&d, 4);
  const int blocks = sms * 8, threads = 256;
  k<MODE><<<blocks, threads>>>(d, 3);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(d, 3 + rep);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(d);
  // warp-instructions per clock per SMSP
  const double winstr = (double)blocks * (threads / 32) * kIters * kChains * warp_instr_per_inner;
  const double clocks = best * 1e-3 * mhz * 1e6;
  return winstr / clocks / (sms * 4.0);
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  int mhz = 0;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  mhz /= 1000;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %d, \"unit\": \"units per clock per SMSP (1 warp instruction per clock = 1.0)\"", prop.name, sms, mhz);
  printf(", \"imad\": %.4f", run<M_IMAD>(sms, mhz, 2));
  printf(", \"imad_hi\": %.4f", run<M_HI>(sms, mhz, 2));
  printf(", \"imad_wide\": %.4f", run<M_WIDE>(sms, mhz, 2));
  printf(", \"iadd3\": %.4f", run<M_IADD3>(sms, mhz, 2));
  printf(", \"viaddmnmx\": %.4f", run<M_VMNMX>(sms, mhz, 2));
  printf(", \"lop3\": %.4f", run<M_LOP3>(sms, mhz, 2));
  printf(", \"shoup_products\": %.4f", run<M_SHOUP>(sms, mhz, 2));
  printf(", \"butterflies\": %.4f", run<M_BFLY>(sms, mhz, 1));
  printf(", \"imad_plus_iadd_pairs\": %.4f", run<M_IMAD_IADD>(sms, mhz, 1));
  printf(", \"hi_plus_2iadd_groups\": %.4f", run<M_HI_IADD2>(sms, mhz, 1));
  printf(", \"hi_plus_4iadd_groups\": %.4f", run<M_HI_IADD4>(sms, mhz, 1));
  printf(", \"wide_plus_2iadd_groups\": %.4f", run<M_WIDE_IADD2>(sms, mhz, 1));
  printf(", \"mont_products\": %.4f", run<M_MONT>(sms, mhz, 1));
  printf(", \"hi_plus_lop3_pairs\": %.4f", run<M_SHOUP_WIDE>(sms, mhz, 1));
  printf(", \"butterflies_add_pinned\": %.4f", run<M_BFLY_ASM>(sms, mhz, 1));
  printf(", \"iadd3_three_operand\": %.4f", run<M_IADD3_IMM>(sms, mhz, 2));
  printf(", \"sub_two_register\": %.4f", run<M_SUB>(sms, mhz, 2));
  printf("}\n");
  return 0;
}
