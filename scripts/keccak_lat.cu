// Development aid: cycles per Keccak-f[1600] on one dependent chain, for the
// state layouts considered for k_seed_expand (shake.cu).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#define FULL 0xFFFFFFFFu
__constant__ uint32_t RC[48];
__constant__ int RHO[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39, 41, 45, 15, 21, 8, 18, 2, 61, 56, 14};
__device__ __forceinline__ uint32_t rotv(uint32_t v, uint32_t k) { return __funnelshift_l(v, v, k); }

struct Ctx { uint32_t colmask; int xm1, xp1, xp2, pi_src, c1, c2, c3, c4; uint32_t swap, rke, rko, iota; };
__device__ Ctx ctx(int t) {
  Ctx c; const int u = t < 25 ? t : 0; const int x = u % 5, y = u / 5;
  c.colmask = t < 25 ? (0x108421u << x) : 0xFE000000u;
  c.xm1 = (x + 4) % 5 + 5 * y; c.xp1 = (x + 1) % 5 + 5 * y; c.xp2 = (x + 2) % 5 + 5 * y;
  c.c1 = x + 5 * ((y + 1) % 5); c.c2 = x + 5 * ((y + 2) % 5); c.c3 = x + 5 * ((y + 3) % 5); c.c4 = x + 5 * ((y + 4) % 5);
  const int sx = ((3 * (y - 3 * x)) % 5 + 5) % 5, sy = x; c.pi_src = sx + 5 * sy;
  const int r = RHO[c.pi_src]; c.swap = r & 1; c.rke = (r + 1) >> 1; c.rko = r >> 1; if (!c.swap) c.rke = c.rko;
  c.iota = t == 0 ? FULL : 0u; return c;
}
template <int MODE>
__device__ __forceinline__ void f25(uint32_t& e, uint32_t& o, const Ctx& c) {
#pragma unroll 4
  for (int round = 0; round < 24; ++round) {
    uint32_t ce, co;
    if (MODE == 0) { ce = __reduce_xor_sync(c.colmask, e); co = __reduce_xor_sync(c.colmask, o); }
    else {
      ce = e ^ __shfl_sync(FULL, e, c.c1) ^ __shfl_sync(FULL, e, c.c2) ^ __shfl_sync(FULL, e, c.c3) ^ __shfl_sync(FULL, e, c.c4);
      co = o ^ __shfl_sync(FULL, o, c.c1) ^ __shfl_sync(FULL, o, c.c2) ^ __shfl_sync(FULL, o, c.c3) ^ __shfl_sync(FULL, o, c.c4);
    }
    const uint32_t me = __shfl_sync(FULL, ce, c.xm1), mo = __shfl_sync(FULL, co, c.xm1);
    const uint32_t pe = __shfl_sync(FULL, ce, c.xp1), po = __shfl_sync(FULL, co, c.xp1);
    e ^= me ^ __funnelshift_l(po, po, 1); o ^= mo ^ pe;
    const uint32_t se = __shfl_sync(FULL, e, c.pi_src), so = __shfl_sync(FULL, o, c.pi_src);
    const uint32_t be = rotv(c.swap ? so : se, c.rke), bo = rotv(c.swap ? se : so, c.rko);
    const uint32_t b1e = __shfl_sync(FULL, be, c.xp1), b1o = __shfl_sync(FULL, bo, c.xp1);
    const uint32_t b2e = __shfl_sync(FULL, be, c.xp2), b2o = __shfl_sync(FULL, bo, c.xp2);
    e = be ^ (~b1e & b2e); o = bo ^ (~b1o & b2o);
    e ^= RC[2 * round] & c.iota; o ^= RC[2 * round + 1] & c.iota;
  }
}
template <int MODE>
__global__ void k(int iters, uint32_t* out, long long* cyc) {
  const int t = threadIdx.x & 31; const Ctx c = ctx(t);
  uint32_t e = t, o = t * 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) f25<MODE>(e, o, c);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = e ^ o;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  uint32_t h[48]; for (int i = 0; i < 48; ++i) h[i] = i * 2654435761u; cudaMemcpyToSymbol(RC, h, sizeof h);
  uint32_t* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 8);
  const int iters = 200;
  for (int blocks : {1, 2048}) {
    k<0><<<blocks, 32>>>(iters, out, cyc); cudaDeviceSynchronize();
    k<0><<<blocks, 32>>>(iters, out, cyc); cudaDeviceSynchronize();
    printf("redux  blocks %d: %.0f cycles/permutation (%s)\n", blocks, (double)*cyc / iters, cudaGetErrorString(cudaGetLastError()));
    k<1><<<blocks, 32>>>(iters, out, cyc); cudaDeviceSynchronize();
    k<1><<<blocks, 32>>>(iters, out, cyc); cudaDeviceSynchronize();
    printf("shfl   blocks %d: %.0f cycles/permutation\n", blocks, (double)*cyc / iters);
  }
  return 0;
}
