// C ABI (include/pa_b200.h): plans, twiddle tables, workspaces, host paths.
//
// Reference seams replaced (pkg/src/modpa): compress pa.py:175-190,
// pa_round pa.py:193-217 (validation stays in Python), mul bignum.py:194-231,
// fused_mul_add bignum.py:234-238, import/export layout pa.py:111-132.
// The reference's SSA plan (ntt.py:69-108) chooses a Fermat-ring geometry;
// here the plan is the transform length L = 2^lg >= 2*ceil(n/32) - 1 of a
// three-prime word convolution and its four-step split L = R * C.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pa_b200.h"
#include "ntt_core.cuh"
#include "pa_kernels.cuh"

namespace pab {
void profile_enable(bool enable);
int profile_collect(const char** names, int* counts, double* ms, int cap);
}

using namespace pab;

namespace {

thread_local std::string g_err;
constexpr int kTw4MaxLg = 18;  // full four-step twiddle tables up to L = 2^18 (12 MiB, L2-resident)

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  const int code = (e == cudaErrorMemoryAllocation) ? PAB_ENOMEM : PAB_ECUDA;
  return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                          \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// ---------------------------------------------------------------- host math
u64 powmod(u64 a, u64 e, u64 m) {
  u64 r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = r * a % m;
    a = a * a % m;
    e >>= 1;
  }
  return r;
}
u32 inv_mod(u32 a, u32 p) { return (u32)powmod(a, p - 2, p); }
u32 shoup_of(u32 w, u32 p) { return (u32)(((u64)w << 32) / p); }

PrimeInfo prime_info(u32 p) {
  PrimeInfo pi;
  pi.p = p;
  pi.two_p = 2 * p;
  u32 inv = 1;  // p^-1 mod 2^32 by Newton
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  pi.p_mont = 0u - inv;
  pi.one_sh = shoup_of(1, p);
  return pi;
}

// root of unity of order 2^k (dir 1: its inverse); the same roots the device
// code derives at compile time (ntt_core.cuh: croot)
u32 root_pow2(int prime, int k, int dir) {
  const u32 p = kPrimes[prime];
  const u32 w23 = dir ? kIRoot23[prime] : kRoot23[prime];
  return (u32)powmod(w23, (u64)1 << (kMaxLg - k), p);
}

// ------------------------------------------------------------ device state
struct Plan {
  int lg, lgR, lgC;
  u32* tlo_m = nullptr;
  uint2* thi = nullptr;
  uint2* g = nullptr;
  uint2* tw4 = nullptr;
  u32 scale[kNumPrimes], scale_sh[kNumPrimes];
};

struct HostCtx {  // cached buffers for the host-pointer entry points
  cudaStream_t stream = nullptr;
  uint8_t* mapped = nullptr;      // pinned, device-mapped staging for tiny blocks
  uint8_t* mapped_dev = nullptr;
  size_t mapped_bytes = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  uint8_t* dev_io = nullptr;
  size_t dev_io_bytes = 0;
  std::mutex mu;
};

struct DevState {
  bool ready = false;
  uint2* stw = nullptr;
  std::map<int, Plan> plans;
  HostCtx host;
};

std::mutex g_mu;
std::map<int, std::unique_ptr<DevState>> g_dev;

int ensure_device(int dev, DevState** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto& slot = g_dev[dev];
  if (!slot) slot.reset(new DevState());
  DevState* ds = slot.get();
  if (!ds->ready) {
    for (int i = 0; i < kNumPrimes; ++i) {  // the compiled-in roots must be primitive 2^23-th
      const u32 p = kPrimes[i];
      if (powmod(kRoot23[i], (u64)1 << (kMaxLg - 1), p) != p - 1 ||
          (u64)kRoot23[i] * kIRoot23[i] % p != 1)
        return fail(PAB_ECUDA, "internal: bad root-of-unity constants");
    }
    PrimeInfo pis[kNumPrimes];
    for (int i = 0; i < kNumPrimes; ++i) pis[i] = prime_info(kPrimes[i]);
    CrtConst crt;
    crt.p0 = kPrimes[0];
    crt.p1 = kPrimes[1];
    crt.p2 = kPrimes[2];
    crt.inv01 = inv_mod(crt.p0 % crt.p1, crt.p1);
    crt.inv01_sh = shoup_of(crt.inv01, crt.p1);
    crt.p0m2 = crt.p0 % crt.p2;
    crt.p0m2_sh = shoup_of(crt.p0m2, crt.p2);
    crt.inv012 = inv_mod((u32)(((u64)crt.p0 * crt.p1) % crt.p2), crt.p2);
    crt.inv012_sh = shoup_of(crt.inv012, crt.p2);
    crt.p0p1 = (u64)crt.p0 * crt.p1;
    upload_constants(pis, crt);
    CK(cudaGetLastError(), "upload constants");
    // stage twiddles tw[h + e] = w_{2h}^{+-e}
    std::vector<uint2> stw((size_t)kNumPrimes * 2 * kTwN);
    for (int i = 0; i < kNumPrimes; ++i) {
      const u32 p = kPrimes[i];
      for (int dir = 0; dir < 2; ++dir) {
        uint2* t = &stw[((size_t)i * 2 + dir) * kTwN];
        t[0] = make_uint2(1, shoup_of(1, p));
        for (int s = 0; s < kTwLg; ++s) {
          const int h = 1 << s;
          const u32 w = root_pow2(i, s + 1, dir);
          u64 x = 1;
          for (int e = 0; e < h; ++e) {
            t[h + e] = make_uint2((u32)x, shoup_of((u32)x, p));
            x = x * w % p;
          }
        }
      }
    }
    CK(cudaMalloc(&ds->stw, stw.size() * sizeof(uint2)), "alloc twiddles");
    CK(cudaMemcpy(ds->stw, stw.data(), stw.size() * sizeof(uint2), cudaMemcpyHostToDevice),
       "upload twiddles");
    set_kernel_attrs();
    CK(cudaGetLastError(), "kernel attributes");
    ds->ready = true;
  }
  *out = ds;
  return PAB_OK;
}

int current_device(DevState** ds) {
  int dev = 0;
  CK(cudaGetDevice(&dev), "cudaGetDevice");
  return ensure_device(dev, ds);
}

void split_lg(int lg, int* lgR, int* lgC) {
  if (lg <= kTwLg) {
    *lgR = 0;
    *lgC = lg;
  } else {
    *lgR = lg / 2;
    *lgC = lg - lg / 2;
  }
}

int get_plan(DevState* ds, int lg, const Plan** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = ds->plans.find(lg);
  if (it != ds->plans.end()) {
    *out = &it->second;
    return PAB_OK;
  }
  Plan pl;
  pl.lg = lg;
  split_lg(lg, &pl.lgR, &pl.lgC);
  std::vector<u32> tlo((size_t)kNumPrimes * 2 * kTwN, 0);
  std::vector<uint2> thi((size_t)kNumPrimes * 2 * kTwN, make_uint2(0, 0));
  std::vector<uint2> gt((size_t)kNumPrimes * 2 * kTwN, make_uint2(0, 0));
  // row-pass twiddle step: w_L^(k1 * 2^slo0), slo0 = lowest stage of the row's top pass
  const int slo0 = pass_plan(pl.lgC).slo[0];
  for (int i = 0; i < kNumPrimes; ++i) {
    const u32 p = kPrimes[i];
    const u64 r32 = ((u64)1 << 32) % p;
    for (int dir = 0; dir < 2; ++dir) {
      const u32 wL = root_pow2(i, lg, dir);
      if (pl.lgR > 0) {
        const u64 gstep = powmod(wL, (u64)1 << slo0, p);
        u64 y = 1;
        for (int k = 0; k < (1 << pl.lgR); ++k) {
          gt[((size_t)i * 2 + dir) * kTwN + k] = make_uint2((u32)y, shoup_of((u32)y, p));
          y = y * gstep % p;
        }
      }
      u64 x = 1;
      for (int e = 0; e < kTwN; ++e) {
        tlo[((size_t)i * 2 + dir) * kTwN + e] = (u32)(x * r32 % p);
        x = x * wL % p;
      }
      const u64 step = powmod(wL, kTwN, p);
      x = 1;
      for (int j = 0; j < kTwN; ++j) {
        thi[((size_t)i * 2 + dir) * kTwN + j] = make_uint2((u32)x, shoup_of((u32)x, p));
        x = x * step % p;
      }
    }
    const u64 linv = inv_mod((u32)(((u64)1 << lg) % p), p);
    pl.scale[i] = (u32)(linv * r32 % p);
    pl.scale_sh[i] = shoup_of(pl.scale[i], p);
  }
  CK(cudaMalloc(&pl.tlo_m, tlo.size() * sizeof(u32)), "alloc plan tables");
  CK(cudaMalloc(&pl.thi, thi.size() * sizeof(uint2)), "alloc plan tables");
  CK(cudaMalloc(&pl.g, gt.size() * sizeof(uint2)), "alloc plan tables");
  CK(cudaMemcpy(pl.g, gt.data(), gt.size() * sizeof(uint2), cudaMemcpyHostToDevice),
     "upload plan tables");
  CK(cudaMemcpy(pl.tlo_m, tlo.data(), tlo.size() * sizeof(u32), cudaMemcpyHostToDevice),
     "upload plan tables");
  CK(cudaMemcpy(pl.thi, thi.data(), thi.size() * sizeof(uint2), cudaMemcpyHostToDevice),
     "upload plan tables");
  // full four-step twiddle tables for small L (<= 2^kTw4MaxLg): 48 L bytes, L2-resident
  if (pl.lgR > 0 && lg <= kTw4MaxLg) {
    const size_t L = (size_t)1 << lg;
    const int C = 1 << pl.lgC, R = 1 << pl.lgR;
    std::vector<uint2> t4((size_t)kNumPrimes * 2 * L);
    for (int i = 0; i < kNumPrimes; ++i) {
      const u32 p = kPrimes[i];
      for (int dir = 0; dir < 2; ++dir) {
        const u32 wL = root_pow2(i, lg, dir);
        uint2* t = &t4[((size_t)i * 2 + dir) * L];
        for (int q = 0; q < R; ++q) {
          int k1 = 0;  // bit reversal of q in lgR bits
          for (int b = 0; b < pl.lgR; ++b) k1 |= ((q >> b) & 1) << (pl.lgR - 1 - b);
          const u64 step = powmod(wL, (u64)k1, p);
          u64 x = 1;
          for (int c = 0; c < C; ++c) {
            t[(size_t)q * C + c] = make_uint2((u32)x, shoup_of((u32)x, p));
            x = x * step % p;
          }
        }
      }
    }
    CK(cudaMalloc(&pl.tw4, t4.size() * sizeof(uint2)), "alloc twiddle tables");
    CK(cudaMemcpy(pl.tw4, t4.data(), t4.size() * sizeof(uint2), cudaMemcpyHostToDevice),
       "upload twiddle tables");
  }
  auto res = ds->plans.emplace(lg, pl);
  *out = &res.first->second;
  return PAB_OK;
}

PlanTables tables_of(const DevState* ds, const Plan* pl) {
  PlanTables t;
  t.stw = ds->stw;
  t.tlo_m = pl->tlo_m;
  t.thi = pl->thi;
  t.g = pl->g;
  t.tw4 = pl->tw4;
  for (int i = 0; i < kNumPrimes; ++i) {
    t.scale[i] = pl->scale[i];
    t.scale_sh[i] = pl->scale_sh[i];
  }
  return t;
}

// P = p0 p1 p2 as a double-free bound check: k * (2^32-1)^2 < P.
bool crt_bound_ok(u64 k) {
  // compare with 128-bit arithmetic: P / (2^32-1)^2 ~ 2^25.35
  unsigned __int128 P = (unsigned __int128)kPrimes[0] * kPrimes[1] * kPrimes[2];
  unsigned __int128 w = (unsigned __int128)0xFFFFFFFFu * 0xFFFFFFFFu;
  return (unsigned __int128)k * w < P;
}

int lg_for(u64 len) {  // smallest lg with 2^lg >= len, at least 6
  int lg = 6;
  while (((u64)1 << lg) < len) ++lg;
  return lg;
}

constexpr u64 kMaxChunk = 16384;
  // blocks per launch (grid.y/z <= 65535)

u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }
u64 round_up(u64 a, u64 b) { return ceil_div(a, b) * b; }

// Workspace layout for a conv job over `batch` blocks.
struct Layout {
  u64 in_stride;   // words per operand slot
  u64 L;
  u64 tiles;
  u64 mw;
  size_t off_words, off_buf, off_out, off_state, off_ctr, total;
};

Layout layout_for(u64 kmax, int lg, u64 nT, u64 mw, u64 batch) {
  Layout ly;
  ly.in_stride = round_up(kmax > 0 ? kmax : 1, 64);
  ly.L = (u64)1 << lg;
  ly.tiles = ceil_div(nT, kCarryTile);
  ly.mw = mw;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += round_up(bytes, 256);
    return o;
  };
  ly.off_words = take(batch * 3 * ly.in_stride * 4);
  ly.off_buf = take(batch * 6 * ly.L * 4);
  ly.off_out = take(batch * mw * 4);
  ly.off_state = take(batch * ly.tiles * 8);
  ly.off_ctr = take(batch * 4);
  ly.total = off;
  return ly;
}

struct HashGeo {
  u64 K;    // words per operand
  int lg;
  u64 mw;
};

int hash_geo(u64 n, u64 r, HashGeo* g) {
  if (n < 1) return fail(PAB_EINVAL, "block length must be >= 1");
  if (r < 1 || r > n) return fail(PAB_EINVAL, "output length r must satisfy 1 <= r <= n");
  if (n > pab_max_bits()) return fail(PAB_ERANGE, "block length exceeds pab_max_bits()");
  g->K = ceil_div(n, 32);
  g->lg = lg_for(2 * g->K - 1);
  g->mw = ceil_div(r, 32);
  return PAB_OK;
}

ConvJob make_job(const Layout& ly, void* ws, int lg, int batch) {
  ConvJob j;
  std::memset(&j, 0, sizeof(j));
  char* base = (char*)ws;
  j.batch = batch;
  j.lg = lg;
  int lgR, lgC;
  split_lg(lg, &lgR, &lgC);
  j.lgR = lgR;
  j.lgC = lgC;
  j.buf = (u32*)(base + ly.off_buf);
  j.out_words = (u32*)(base + ly.off_out);
  j.mw = (long long)ly.mw;
  j.tile_state = (unsigned long long*)(base + ly.off_state);
  j.tile_ctr = (u32*)(base + ly.off_ctr);
  j.tiles = (int)ly.tiles;
  j.maskA = j.maskX = j.maskD = 0xFFFFFFFFu;
  return j;
}

bool aligned4(const void* p) { return ((uintptr_t)p & 3) == 0; }

}  // namespace

// ================================================================== C ABI
extern "C" {

int pab_version(void) { return 100; }

const char* pab_last_error(void) { return g_err.c_str(); }

uint64_t pab_max_bits(void) { return (uint64_t)32 << (kMaxLg - 1); }  // 2K-1 <= 2^23

int pab_plan_info(uint64_t n_bits, int* lg, int* lg_rows, int* lg_cols) {
  HashGeo g;
  int rc = hash_geo(n_bits, 1, &g);
  if (rc) return rc;
  int a, b;
  split_lg(g.lg, &a, &b);
  if (lg) *lg = g.lg;
  if (lg_rows) *lg_rows = a;
  if (lg_cols) *lg_cols = b;
  return PAB_OK;
}

size_t pab_hash_workspace_bytes(uint64_t n_bits, uint32_t batch) {
  HashGeo g;
  if (hash_geo(n_bits, 1, &g)) return 0;
  // output words are bounded by K; size for the largest r
  return layout_for(g.K, g.lg, g.K, g.K, batch ? batch : 1).total;
}

int pab_hash_batch(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t in_stride,
                   uint64_t n_bits, uint64_t r_bits, uint32_t batch, int byte_order,
                   uint8_t* out, uint64_t out_stride, void* workspace, size_t workspace_bytes,
                   void* stream) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  if (batch == 0) return PAB_OK;
  if (!x || !c || !d || !out || !workspace) return fail(PAB_EINVAL, "null pointer argument");
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  const u64 nbytes = ceil_div(n_bits, 8), rbytes = ceil_div(r_bits, 8);
  if (in_stride < nbytes || out_stride < rbytes)
    return fail(PAB_EINVAL, "stride smaller than the block byte length");
  DevState* ds;
  if ((rc = current_device(&ds))) return rc;
  const Plan* pl;
  if ((rc = get_plan(ds, g.lg, &pl))) return rc;
  const PlanTables tab = tables_of(ds, pl);
  cudaStream_t st = (cudaStream_t)stream;
  // blocks per chunk that fit the workspace
  u64 chunk = batch < kMaxChunk ? batch : kMaxChunk;  // grid y/z limits
  while (chunk > 0 && layout_for(g.K, g.lg, g.K, g.mw, chunk).total > workspace_bytes) chunk /= 2;
  if (chunk == 0) return fail(PAB_EINVAL, "workspace too small for one block");
  const int msf = byte_order == PAB_ORDER_MSF;
  // LSF blocks whose words can be read in place (the common case): no pack kernel
  const bool direct_in = !msf && nbytes % 4 == 0 && in_stride % 4 == 0 && aligned4(x) &&
                         aligned4(c) && aligned4(d);
  const bool direct_out = !msf && out_stride % 4 == 0 && aligned4(out);
  const u32 mask = (n_bits & 31) ? ((1u << (n_bits & 31)) - 1u) : 0xFFFFFFFFu;
  for (u64 b0 = 0; b0 < batch; b0 += chunk) {
    const int nb = (int)((batch - b0) < chunk ? (batch - b0) : chunk);
    const Layout ly = layout_for(g.K, g.lg, g.K, g.mw, nb);
    ConvJob job = make_job(ly, workspace, g.lg, nb);
    job.kA = job.kX = job.kD = (long long)g.K;
    job.maskA = job.maskX = job.maskD = mask;
    job.nT = (long long)g.K;
    job.nRes = (long long)g.K;
    job.n_mod_bits = (long long)n_bits;
    job.shift = (long long)(n_bits - r_bits);
    job.mw = (long long)g.mw;
    CK(cudaMemsetAsync((char*)workspace + ly.off_state, 0, ly.total - ly.off_state, st), "memset");
    if (direct_in) {
      job.srcA = (const u32*)(c + b0 * in_stride);
      job.srcX = (const u32*)(x + b0 * in_stride);
      job.srcD = (const u32*)(d + b0 * in_stride);
      job.src_stride = (long long)(in_stride / 4);
    } else {
      u32* words = (u32*)((char*)workspace + ly.off_words);
      const long long ws = (long long)ly.in_stride;
      launch_pack(c + b0 * in_stride, (long long)in_stride, (long long)n_bits, msf, nb, words,
                  3 * ws, (long long)g.K, st);
      launch_pack(x + b0 * in_stride, (long long)in_stride, (long long)n_bits, msf, nb, words + ws,
                  3 * ws, (long long)g.K, st);
      launch_pack(d + b0 * in_stride, (long long)in_stride, (long long)n_bits, msf, nb,
                  words + 2 * ws, 3 * ws, (long long)g.K, st);
      job.srcA = words;
      job.srcX = words + ws;
      job.srcD = words + 2 * ws;
      job.src_stride = 3 * ws;
    }
    if (direct_out) {
      job.out_words = nullptr;
      job.out_bytes = out + b0 * out_stride;
      job.out_stride = (long long)out_stride;
      job.rbytes = (long long)rbytes;
    }
    launch_conv(job, tab, st);
    launch_carry(job, st);
    if (!direct_out)
      launch_unpack(job.out_words, job.mw, (long long)r_bits, msf, nb, out + b0 * out_stride,
                    (long long)out_stride, st);
    CK(cudaGetLastError(), "kernel launch");
  }
  return PAB_OK;
}

static int host_ensure(HostCtx& h, size_t ws_bytes, size_t io_bytes) {
  if (!h.stream) CK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking), "stream");
  if (h.ws_bytes < ws_bytes) {
    if (h.ws) cudaFree(h.ws);
    h.ws = nullptr;
    h.ws_bytes = 0;
    CK(cudaMalloc(&h.ws, ws_bytes), "workspace alloc");
    h.ws_bytes = ws_bytes;
  }
  if (h.dev_io_bytes < io_bytes) {
    if (h.dev_io) cudaFree(h.dev_io);
    h.dev_io = nullptr;
    h.dev_io_bytes = 0;
    CK(cudaMalloc(&h.dev_io, io_bytes), "io alloc");
    h.dev_io_bytes = io_bytes;
  }
  return PAB_OK;
}

int pab_hash_host(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                  uint64_t r_bits, uint32_t batch, int byte_order, uint8_t* out, int device) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  if (batch == 0) return PAB_OK;
  CK(cudaSetDevice(device), "cudaSetDevice");
  DevState* ds;
  if ((rc = ensure_device(device, &ds))) return rc;
  HostCtx& h = ds->host;
  std::lock_guard<std::mutex> lk(h.mu);
  const u64 nbytes = ceil_div(n_bits, 8), rbytes = ceil_div(r_bits, 8);
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  // tiny blocks: one kernel over mapped pinned memory (one launch, one sync)
  const size_t tiny_io = (size_t)batch * (3 * nbytes + rbytes);
  if (n_bits <= (u64)kTinyBits && tiny_io <= ((size_t)1 << 20)) {
    if (!h.stream) CK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking), "stream");
    if (!h.mapped) {
      h.mapped_bytes = (size_t)1 << 20;
      CK(cudaHostAlloc((void**)&h.mapped, h.mapped_bytes, cudaHostAllocMapped), "host alloc");
      CK(cudaHostGetDevicePointer((void**)&h.mapped_dev, h.mapped, 0), "mapped pointer");
    }
    std::memcpy(h.mapped, x, batch * nbytes);
    std::memcpy(h.mapped + batch * nbytes, c, batch * nbytes);
    std::memcpy(h.mapped + 2 * batch * nbytes, d, batch * nbytes);
    uint8_t* dout = h.mapped_dev + 3 * batch * nbytes;
    launch_tiny(h.mapped_dev, h.mapped_dev + batch * nbytes, h.mapped_dev + 2 * batch * nbytes,
                (long long)nbytes, (int)n_bits, (int)r_bits, byte_order == PAB_ORDER_MSF,
                (int)batch, dout, (long long)rbytes, h.stream);
    CK(cudaGetLastError(), "kernel launch");
    CK(cudaStreamSynchronize(h.stream), "synchronize");
    std::memcpy(out, h.mapped + 3 * batch * nbytes, batch * rbytes);
    return PAB_OK;
  }
  const u64 in_stride = round_up(nbytes, 16), out_stride = round_up(rbytes, 16);
  // at most ~2 GiB of transform workspace per chunk
  u64 chunk = batch;
  while (chunk > 1 && pab_hash_workspace_bytes(n_bits, (uint32_t)chunk) > ((size_t)2 << 30))
    chunk /= 2;
  const size_t ws_bytes = pab_hash_workspace_bytes(n_bits, (uint32_t)chunk);
  const size_t io_bytes = (size_t)batch * (3 * in_stride + out_stride);
  if ((rc = host_ensure(h, ws_bytes, io_bytes))) return rc;
  uint8_t* dx = h.dev_io;
  uint8_t* dc = dx + batch * in_stride;
  uint8_t* dd = dc + batch * in_stride;
  uint8_t* dout = dd + batch * in_stride;
  CK(cudaMemcpy2DAsync(dx, in_stride, x, nbytes, nbytes, batch, cudaMemcpyHostToDevice, h.stream),
     "H2D x");
  CK(cudaMemcpy2DAsync(dc, in_stride, c, nbytes, nbytes, batch, cudaMemcpyHostToDevice, h.stream),
     "H2D c");
  CK(cudaMemcpy2DAsync(dd, in_stride, d, nbytes, nbytes, batch, cudaMemcpyHostToDevice, h.stream),
     "H2D d");
  rc = pab_hash_batch(dx, dc, dd, in_stride, n_bits, r_bits, batch, byte_order, dout, out_stride,
                      h.ws, h.ws_bytes, h.stream);
  if (rc) return rc;
  CK(cudaMemcpy2DAsync(out, rbytes, dout, out_stride, rbytes, batch, cudaMemcpyDeviceToHost,
                       h.stream),
     "D2H out");
  CK(cudaStreamSynchronize(h.stream), "synchronize");
  return PAB_OK;
}

size_t pab_mul_workspace_bytes(uint64_t a_bytes, uint64_t b_bytes) {
  const u64 ka = ceil_div(a_bytes, 4), kb = ceil_div(b_bytes, 4);
  if (ka == 0 || kb == 0) return 256;
  const u64 nT = ka + kb;
  const int lg = lg_for(ka + kb - 1);
  return layout_for(ka > kb ? ka : kb, lg, nT, nT, 1).total;
}

int pab_mul(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes, uint8_t* out,
            void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const u64 ka = ceil_div(a_bytes, 4), kb = ceil_div(b_bytes, 4);
  if (a_bytes + b_bytes == 0) return PAB_OK;
  if (ka == 0 || kb == 0) {
    CK(cudaMemsetAsync(out, 0, a_bytes + b_bytes, st), "memset");
    return PAB_OK;
  }
  const u64 nT = ka + kb;
  const int lg = lg_for(ka + kb - 1);
  if (lg > kMaxLg || !crt_bound_ok(ka < kb ? ka : kb))
    return fail(PAB_ERANGE, "operands exceed the exact three-prime convolution range");
  const Layout ly = layout_for(ka > kb ? ka : kb, lg, nT, nT, 1);
  if (workspace_bytes < ly.total) return fail(PAB_EINVAL, "workspace too small");
  int rc;
  DevState* ds;
  if ((rc = current_device(&ds))) return rc;
  const Plan* pl;
  if ((rc = get_plan(ds, lg, &pl))) return rc;
  ConvJob job = make_job(ly, workspace, lg, 1);
  job.kA = (long long)ka;
  job.kX = (long long)kb;
  job.kD = 0;
  job.nT = (long long)nT;
  job.nRes = (long long)(nT < ly.L ? nT : ly.L);
  job.n_mod_bits = 32ll * (long long)nT;
  job.shift = 0;
  job.mw = (long long)nT;
  CK(cudaMemsetAsync((char*)workspace + ly.off_state, 0, ly.total - ly.off_state, st), "memset");
  u32* words = (u32*)((char*)workspace + ly.off_words);
  launch_pack(a, (long long)a_bytes, 8ll * (long long)a_bytes, 0, 1, words, 0, (long long)ka, st);
  launch_pack(b, (long long)b_bytes, 8ll * (long long)b_bytes, 0, 1, words + ly.in_stride, 0,
              (long long)kb, st);
  job.srcA = words;
  job.srcX = words + ly.in_stride;
  job.srcD = nullptr;
  job.src_stride = 0;
  launch_conv(job, tables_of(ds, pl), st);
  launch_carry(job, st);
  launch_unpack(job.out_words, job.mw, 8ll * (long long)(a_bytes + b_bytes), 0, 1, out,
                (long long)(a_bytes + b_bytes), st);
  CK(cudaGetLastError(), "kernel launch");
  return PAB_OK;
}

int pab_mul_host(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes,
                 uint8_t* out, int device) {
  CK(cudaSetDevice(device), "cudaSetDevice");
  DevState* ds;
  int rc;
  if ((rc = ensure_device(device, &ds))) return rc;
  HostCtx& h = ds->host;
  std::lock_guard<std::mutex> lk(h.mu);
  const size_t ws = pab_mul_workspace_bytes(a_bytes, b_bytes);
  const size_t io = round_up(a_bytes + 1, 256) + round_up(b_bytes + 1, 256) +
                    round_up(a_bytes + b_bytes + 1, 256);
  if ((rc = host_ensure(h, ws, io))) return rc;
  uint8_t* da = h.dev_io;
  uint8_t* db = da + round_up(a_bytes + 1, 256);
  uint8_t* dout = db + round_up(b_bytes + 1, 256);
  if (a_bytes) CK(cudaMemcpyAsync(da, a, a_bytes, cudaMemcpyHostToDevice, h.stream), "H2D a");
  if (b_bytes) CK(cudaMemcpyAsync(db, b, b_bytes, cudaMemcpyHostToDevice, h.stream), "H2D b");
  rc = pab_mul(da, a_bytes, db, b_bytes, dout, h.ws, h.ws_bytes, h.stream);
  if (rc) return rc;
  if (a_bytes + b_bytes)
    CK(cudaMemcpyAsync(out, dout, a_bytes + b_bytes, cudaMemcpyDeviceToHost, h.stream), "D2H");
  CK(cudaStreamSynchronize(h.stream), "synchronize");
  return PAB_OK;
}

void pab_profile_enable(int enable) { profile_enable(enable != 0); }

int pab_profile_collect(const char** names, int* counts, double* total_ms, int cap) {
  return profile_collect(names, counts, total_ms, cap);
}

}  // extern "C"
