// Integer-pipe throughput on B200 (the denominator of the NTT int roofline).
// Streams of independent IADD3 / LOP3 (ALU pipe), IMAD (FMA pipe), IMAD.HI,
// and a 4:3 ALU:FMA mix shaped like the Shoup butterfly, over all SMs.
// Prints one JSON object; used as profiles/int_peak.json.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int MODE>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains], b[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = seed * (threadIdx.x + 17 * i + 1);
    b[i] = seed ^ (i * 0x9E3779B9u + threadIdx.x);
  }
  const uint32_t p = 998244353u, w = 12345u, wp = 54321u;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if (MODE == 0) {  // ALU: 4 x 3-input add
        a[i] = a[i] + b[i] + 0x1234u;
        b[i] = b[i] + a[i] + 0x77u;
        a[i] = a[i] + b[i] + 0x55u;
        b[i] = b[i] + a[i] + 0x99u;
      } else if (MODE == 1) {  // FMA: 4 x IMAD
        a[i] = a[i] * b[i] + 0x1234u;
        b[i] = b[i] * a[i] + 0x77u;
        a[i] = a[i] * b[i] + 0x55u;
        b[i] = b[i] * a[i] + 0x99u;
      } else if (MODE == 2) {  // IMAD.HI
        a[i] = __umulhi(a[i], b[i]) + a[i];
        b[i] = __umulhi(b[i], a[i]) + b[i];
      } else {  // Shoup DIF butterfly: 4 ALU + 3 FMA-pipe (IMAD.HI, 2 IMAD)
        uint32_t s = a[i] + b[i];
        s = min(s, s - 2 * p);
        uint32_t d = a[i] - b[i] + 2 * p;
        uint32_t q = __umulhi(d, wp);
        b[i] = d * w - q * p;
        a[i] = s;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc ^= a[i] ^ b[i];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
double run(int blocks, int threads, double ops_per_inner) {
  uint32_t* d;
  cudaMalloc(&d, 4);
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
  const double ops = (double)blocks * threads * kIters * kChains * ops_per_inner;
  return ops / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const int blocks = sms * 8, threads = 256;
  // warm the clocks
  run<3>(blocks, threads, 7.0);
  const double alu = run<0>(blocks, threads, 4.0);   // 4 IADD3 per inner
  const double fma = run<1>(blocks, threads, 4.0);   // 4 IMAD
  const double hi = run<2>(blocks, threads, 4.0);    // 2 IMAD.HI + 2 IADD
  const double bfly = run<3>(blocks, threads, 7.0);  // canonical 7 ops / butterfly
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"alu_iadd3_tops\": %.3f, \"fma_imad_tops\": %.3f, "
         "\"imad_hi_mix_tops\": %.3f, \"shoup_butterfly_tops\": %.3f, "
         "\"shoup_butterflies_per_s\": %.4e, \"int32_tops\": %.3f, \"clock_attr_mhz\": %.0f, "
         "\"note\": \"int32_tops = canonical-op rate of the Shoup DIF butterfly stream "
         "(7 ops each), the mix the NTT issues\"}\n",
         prop.name, sms, alu, fma, hi, bfly, bfly / 7.0 * 1e12, bfly, clk_khz / 1e3);
  return 0;
}
