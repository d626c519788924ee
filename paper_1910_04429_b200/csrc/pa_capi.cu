// C ABI (include/pa_b200.h): plans, twiddle tables, workspaces, host paths.
//
// Reference seams replaced (pkg/src/modpa): compress pa.py:175-190,
// pa_round pa.py:193-217 (validation stays in Python), mul bignum.py:194-231,
// fused_mul_add bignum.py:234-238, import/export layout pa.py:111-132.
// The reference's SSA plan (ntt.py:69-108) chooses a Fermat-ring geometry;
// here the plan is the coefficient width (64-bit coefficients over five
// primes, or 32-bit over three for the largest blocks), the transform length
// L = m * 2^lg >= 2 K' - 1 (K' coefficients per operand) and its four-step
// split L = R * C.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <climits>
#include <cstring>
#include <atomic>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
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
std::atomic<int> g_force_cw{0};  // test hook (pab_force_coef_words): 0 = automatic
constexpr int kTw4MaxLg = 22;  // full four-step twiddle tables up to L = 2^22 (80 L bytes <= 320 MiB; at 3*2^20 k_row -3%)

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


// w_N = g^((p-1)/N) (dir 1: its inverse): the same roots the device code
// derives at compile time (ntt_core.cuh: croot_n)
u32 root_of(int prime, u64 N, int dir) {
  const u32 p = kPrimes[prime];
  const u64 w = powmod(kGen[prime], (u64)(p - 1) / N, p);
  return dir ? inv_mod((u32)w, p) : (u32)w;
}
u32 root_pow2(int prime, int k, int dir) { return root_of(prime, (u64)1 << k, dir); }

// Transform geometry: L = m * 2^lg, columns of R = m * 2^lgR rows, rows of C = 2^lgC.
// lgR == 0 (m == 1) is the single-CTA path (L <= 4096).
struct Geo {
  int m = 1, lg = 0, lgR = 0, lgC = 0;
  u64 L = 0;
};

// Cheapest length >= need among m * 2^lg (lg <= maxlg), m in {1, 3, 5} (radix-3/5
// column stage costs ~2.5 / ~3.7 radix-2 stages).  Returns false if none fits.
bool choose_geo(u64 need, int maxlg, Geo* out) {
  Geo best;
  double best_cost = 0;
  bool found = false;
  const int ms[3] = {1, 3, 5};
  const double extra[3] = {0.0, 2.5, 3.7};
  for (int i = 0; i < 3; ++i) {
    const int m = ms[i];
    int lg = 0;
    while (((u64)m << lg) < need || ((u64)m << lg) < 64) ++lg;
    if (lg > maxlg) continue;
    Geo g;
    g.m = m;
    g.lg = lg;
    g.L = (u64)m << lg;
    static const int force_lgc = [] {  // development override of the four-step split
      const char* e = getenv("PAB_LGC");
      return e ? atoi(e) : 0;
    }();
    if (m == 1) {
      if (lg <= kTwLg) {
        g.lgR = 0;
        g.lgC = lg;
      } else {
        g.lgC = force_lgc ? force_lgc : lg - lg / 2;
        g.lgR = lg - g.lgC;
      }
    } else {
      if (g.L <= (u64)kTwN) continue;  // small lengths: single-CTA pow2 path
      const double lgm = m == 3 ? 1.585 : 2.322;
      int lgC = (int)std::ceil((lg + lgm) / 2.0);  // rows >= columns: smaller column panels
      // measured exceptions (profiles/README.md, split sweep): the row kernel is
      // most efficient at lgC = 9, and 3 * 2^20 prefers the shorter columns
      if (m == 5 && lg == 16) lgC = 9;
      if (m == 3 && lg == 20) lgC = 12;
      if (force_lgc) lgC = force_lgc;
      if (lgC > kTwLg) lgC = kTwLg;
      if (lgC < 6) lgC = 6;
      g.lgC = lgC;
      g.lgR = lg - lgC;
    }
    if (!conv_supported(g.m, g.lgR, g.lgC)) continue;
    const double cost = (double)g.L * (lg + extra[i]);
    if (!found || cost < best_cost) {
      best = g;
      best_cost = cost;
      found = true;
    }
  }
  if (found) *out = best;
  return found;
}

// ------------------------------------------------------------ device state
struct Plan {
  Geo geo;
  u32* tlo_m = nullptr;
  uint2* thi = nullptr;
  int thi_stride = 0;
  uint2* g = nullptr;
  uint2* trad = nullptr;
  int tstride = 0;
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
  uint8_t* pinned = nullptr;      // pinned, mapped staging of the Python-int digit path
  uint8_t* pinned_dev = nullptr;
  size_t pinned_bytes = 0;
  // pab_hash_seeded_host's pipeline: H2D / hashing / D2H streams and per-slot events
  static constexpr int kSlots = 3;
  cudaStream_t p_in = nullptr, p_comp = nullptr, p_out = nullptr;
  cudaEvent_t ev_in[kSlots] = {}, ev_comp[kSlots] = {}, ev_out[kSlots] = {};
  std::mutex mu;
};

struct SplitSlot {  // one prime share of pab_hash_host_split on this device
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  uint8_t* io = nullptr;
  size_t io_bytes = 0;
};

struct DevState {
  bool ready = false;
  uint2* stw = nullptr;
  std::map<int, Plan> plans;  // keyed by m * 64 + lg
  HostCtx host;
  std::vector<std::unique_ptr<SplitSlot>> split;  // guarded by g_split_mu
};

std::mutex g_split_mu;  // pab_hash_host_split calls run one at a time

std::mutex g_mu;
std::map<int, std::unique_ptr<DevState>> g_dev;

int ensure_device(int dev, DevState** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto& slot = g_dev[dev];
  if (!slot) slot.reset(new DevState());
  DevState* ds = slot.get();
  if (!ds->ready) {
    for (int i = 0; i < kNumPrimes; ++i) {  // compiled-in generators must be primitive roots
      const u32 p = kPrimes[i];
      const u32 q[4] = {2, 3, 5, 0};
      for (int j = 0; q[j]; ++j)
        if ((p - 1) % q[j] != 0 || powmod(kGen[i], (p - 1) / q[j], p) == 1)
          return fail(PAB_ECUDA, "internal: bad prime / generator constants");
      const int need = i < 3 ? kMaxLg : kMaxLg5;
      if (((p - 1) >> need) << need != p - 1)
        return fail(PAB_ECUDA, "internal: prime 2-adicity below kMaxLg");
    }
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

int bitrev(int x, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
  return r;
}

int upload(void** dst, const void* src, size_t bytes) {
  CK(cudaMalloc(dst, bytes), "alloc plan tables");
  CK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "upload plan tables");
  return PAB_OK;
}

int get_plan(DevState* ds, const Geo& geo, const Plan** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  const int key = geo.m * 64 + geo.lg;
  auto it = ds->plans.find(key);
  if (it != ds->plans.end()) {
    *out = &it->second;
    return PAB_OK;
  }
  Plan pl;
  pl.geo = geo;
  const u64 L = geo.L;
  const int R = geo.m << geo.lgR, C = 1 << geo.lgC;
  pl.thi_stride = (int)((L + kTwN - 1) / kTwN);
  pl.tstride = R;
  std::vector<u32> tlo((size_t)kNumPrimes * 2 * kTwN, 0);
  std::vector<uint2> thi((size_t)kNumPrimes * 2 * pl.thi_stride, make_uint2(0, 0));
  std::vector<uint2> gt((size_t)kNumPrimes * 2 * R, make_uint2(0, 0));
  std::vector<uint2> trad((size_t)kNumPrimes * 2 * R, make_uint2(0, 0));
  // row-pass twiddle step: w_L^(k1 * 2^slo0), slo0 = lowest stage of the row's top pass
  const int slo0 = pass_plan(geo.lgC).slo[0];
  for (int i = 0; i < kNumPrimes; ++i) {
    const u32 p = kPrimes[i];
    pl.scale[i] = pl.scale_sh[i] = 0;
    if ((p - 1) % L != 0) continue;  // a cw = 1 length beyond this prime's 2-adicity
    const u64 r32 = ((u64)1 << 32) % p;
    // L^-1 * 2^32: undoes the length and the Montgomery factor of the pointwise
    // product.  The four-step path folds it into the inverse four-step twiddles
    // (thi and tw4, dir 1), so the inverse column pass only canonicalises; the
    // single-CTA path (R == 1) applies pl.scale itself.
    const u64 linv = inv_mod((u32)(L % p), p);
    const u64 sc = linv * r32 % p;
    pl.scale[i] = (u32)sc;
    pl.scale_sh[i] = shoup_of(pl.scale[i], p);
    for (int dir = 0; dir < 2; ++dir) {
      const size_t pd = (size_t)i * 2 + dir;
      const u32 wL = root_of(i, L, dir);
      if (R > 1) {
        const u64 gstep = powmod(wL, (u64)1 << slo0, p);
        const u64 wR = root_of(i, (u64)R, dir);
        u64 y = 1, z = 1;
        for (int k = 0; k < R; ++k) {
          gt[pd * R + k] = make_uint2((u32)y, shoup_of((u32)y, p));
          trad[pd * R + k] = make_uint2((u32)z, shoup_of((u32)z, p));
          y = y * gstep % p;
          z = z * wR % p;
        }
      }
      u64 x = 1;
      for (int e = 0; e < kTwN; ++e) {
        tlo[pd * kTwN + e] = (u32)(x * r32 % p);
        x = x * wL % p;
      }
      const u64 step = powmod(wL, kTwN, p);
      x = (dir == 1 && R > 1) ? sc : 1;
      for (int j = 0; j < pl.thi_stride; ++j) {
        thi[pd * pl.thi_stride + j] = make_uint2((u32)x, shoup_of((u32)x, p));
        x = x * step % p;
      }
    }
  }
  int rc;
  if ((rc = upload((void**)&pl.tlo_m, tlo.data(), tlo.size() * sizeof(u32)))) return rc;
  if ((rc = upload((void**)&pl.thi, thi.data(), thi.size() * sizeof(uint2)))) return rc;
  if ((rc = upload((void**)&pl.g, gt.data(), gt.size() * sizeof(uint2)))) return rc;
  if ((rc = upload((void**)&pl.trad, trad.data(), trad.size() * sizeof(uint2)))) return rc;
  // full four-step twiddle tables (L <= 2^kTw4MaxLg): 80 L bytes, read once per launch
  if (R > 1 && L <= ((u64)1 << kTw4MaxLg)) {
    std::vector<uint2> t4((size_t)kNumPrimes * 2 * L);
    // one host thread per (prime, direction): 10 x L entries (0.3 s serial at 3 * 2^20)
    std::vector<std::thread> workers;
    for (int i = 0; i < kNumPrimes; ++i) {
      const u32 p = kPrimes[i];
      if ((p - 1) % L != 0) continue;
      for (int dir = 0; dir < 2; ++dir) {
        workers.emplace_back([&, i, p, dir] {
          const u32 wL = root_of(i, L, dir);
          uint2* t = &t4[((size_t)i * 2 + dir) * L];
          for (int q = 0; q < R; ++q) {
            // column frequency of storage row q (conv_kernels.cuh: row_k1)
            const int k1 = (q >> geo.lgR) + geo.m * bitrev(q & ((1 << geo.lgR) - 1), geo.lgR);
            const u64 step = powmod(wL, (u64)k1, p);
            u64 x = dir == 1 ? pl.scale[i] : 1;  // the inverse carries L^-1 * 2^32
            for (int c = 0; c < C; ++c) {
              t[(size_t)q * C + c] = make_uint2((u32)x, shoup_of((u32)x, p));
              x = x * step % p;
            }
          }
        });
      }
    }
    for (auto& w : workers) w.join();
    if ((rc = upload((void**)&pl.tw4, t4.data(), t4.size() * sizeof(uint2)))) return rc;
  }
  auto res = ds->plans.emplace(key, pl);
  *out = &res.first->second;
  return PAB_OK;
}

PlanTables tables_of(const DevState* ds, const Plan* pl) {
  PlanTables t;
  t.stw = ds->stw;
  t.tlo_m = pl->tlo_m;
  t.thi = pl->thi;
  t.thi_stride = pl->thi_stride;
  t.g = pl->g;
  t.trad = pl->trad;
  t.tstride = pl->tstride;
  t.tw4 = pl->tw4;
  for (int i = 0; i < kNumPrimes; ++i) {
    t.scale[i] = pl->scale[i];
    t.scale_sh[i] = pl->scale_sh[i];
  }
  return t;
}

// Exact convolution bound: k coefficients of cw words each give coefficient
// sums below k * (2^(32 cw) - 1)^2, which must stay below P = p_0 ... p_(np-1).
// Multiword (3 x 64-bit limbs, P < 2^150).
void limbs_mul(u64 a[3], u64 m) {
  unsigned __int128 c = 0;
  for (int i = 0; i < 3; ++i) {
    c += (unsigned __int128)a[i] * m;
    a[i] = (u64)c;
    c >>= 64;
  }
}
bool limbs_lt(const u64 a[3], const u64 b[3]) {
  for (int i = 2; i >= 0; --i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}
bool crt_bound_ok(u64 k, int cw) {
  const int np = cw == 2 ? 5 : 3;
  u64 P[3] = {1, 0, 0};
  for (int i = 0; i < np; ++i) limbs_mul(P, kPrimes[i]);
  // (2^(32 cw) - 1)^2 as limbs
  u64 X[3];
  if (cw == 2) {  // 2^128 - 2^65 + 1
    X[0] = 1;
    X[1] = 0xFFFFFFFFFFFFFFFEull;
    X[2] = 0;
  } else {
    X[0] = 0xFFFFFFFE00000001ull;
    X[1] = X[2] = 0;
  }
  limbs_mul(X, k);
  return limbs_lt(X, P);
}

// Convolution mode: coefficient words (2: five primes, 1: three primes).
struct Mode {
  int cw = 1, np = 3;
  Geo geo;
};

// product of two operands of ka and kb words: prefer 64-bit coefficients
bool choose_mode(u64 ka, u64 kb, Mode* md) {
  const int force = g_force_cw.load();
  const u64 ca = (ka + 1) / 2, cb = (kb + 1) / 2;
  if (force != 1 && crt_bound_ok(ca < cb ? ca : cb, 2) && choose_geo(ca + cb - 1, kMaxLg5, &md->geo)) {
    md->cw = 2;
    md->np = 5;
    return true;
  }
  if (force != 2 && crt_bound_ok(ka < kb ? ka : kb, 1) && choose_geo(ka + kb - 1, kMaxLg, &md->geo)) {
    md->cw = 1;
    md->np = 3;
    return true;
  }
  return false;
}

constexpr u64 kMaxChunk = 16384;  // blocks per launch (grid.y/z <= 65535)

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

Layout layout_for(u64 kmax, u64 L, u64 nT, u64 mw, u64 batch, int np) {
  Layout ly;
  ly.in_stride = round_up(kmax > 0 ? kmax : 1, 64);
  ly.L = L;
  ly.tiles = ceil_div(nT, kCarryTileMin);  // look-back states for the smallest tile of any carry kernel
  ly.mw = mw;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += round_up(bytes, 256);
    return o;
  };
  ly.off_words = take(batch * 3 * ly.in_stride * 4);
  ly.off_buf = take(batch * 2 * np * ly.L * 4);
  ly.off_out = take(batch * mw * 4);
  ly.off_state = take(batch * ly.tiles * 8);
  ly.off_ctr = take(batch * 4);
  ly.total = off;
  return ly;
}

struct HashGeo {
  u64 K;    // words per operand
  Mode md;
  u64 KC;   // coefficients per operand (K / cw rounded up)
  u64 mw;
};

int hash_geo(u64 n, u64 r, HashGeo* g) {
  if (n < 1) return fail(PAB_EINVAL, "block length must be >= 1");
  if (r < 1 || r > n) return fail(PAB_EINVAL, "output length r must satisfy 1 <= r <= n");
  if (n > pab_max_bits()) return fail(PAB_ERANGE, "block length exceeds pab_max_bits()");
  g->K = ceil_div(n, 32);
  if (!choose_mode(g->K, g->K, &g->md))
    return fail(PAB_ERANGE, "no transform geometry for this block length");
  g->KC = ceil_div(g->K, (u64)g->md.cw);
  g->mw = ceil_div(r, 32);
  return PAB_OK;
}

ConvJob make_job(const Layout& ly, void* ws, const Mode& md, int batch) {
  const Geo& geo = md.geo;
  ConvJob j;
  std::memset(&j, 0, sizeof(j));
  char* base = (char*)ws;
  j.batch = batch;
  j.cw = md.cw;
  j.np = md.np;
  j.p0 = 0;
  j.pn = md.np;
  j.m = geo.m;
  j.lg = geo.lg;
  j.lgR = geo.lgR;
  j.lgC = geo.lgC;
  j.L = (long long)geo.L;
  j.buf = (u32*)(base + ly.off_buf);
  j.out_words = (u32*)(base + ly.off_out);
  j.mw = (long long)ly.mw;
  j.tile_state = (unsigned long long*)(base + ly.off_state);
  j.tile_ctr = (u32*)(base + ly.off_ctr);
  j.tiles = (int)ly.tiles;
  j.maskA = j.maskX = j.maskD = 0xFFFFFFFFu;
  return j;
}

bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p & (a - 1)) == 0; }

}  // namespace

// The hash over a workspace.  mode kFull: convolution over every prime + carry;
// kConvOnly: convolution over primes [p0, p0 + pn) into the workspace's residue
// slots (one chunk: the batch must fit); kCarryOnly: carry from residues
// already in the workspace (all primes).  The split modes serve
// pab_hash_host_split (primes over GPUs).
enum HashMode { kFull = 0, kConvOnly = 1, kCarryOnly = 2 };
static int hash_batch_impl(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t in_stride,
                           uint64_t n_bits, uint64_t r_bits, uint32_t batch, int byte_order,
                           uint8_t* out, uint64_t out_stride, void* workspace,
                           size_t workspace_bytes, void* stream, int p0, int pn, int mode) {
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
  if ((rc = get_plan(ds, g.md.geo, &pl))) return rc;
  const PlanTables tab = tables_of(ds, pl);
  cudaStream_t st = (cudaStream_t)stream;
  // blocks per chunk that fit the workspace
  u64 chunk = batch < kMaxChunk ? batch : kMaxChunk;  // grid y/z limits
  while (chunk > 0 && layout_for(g.K, g.md.geo.L, g.K, g.mw, chunk, g.md.np).total > workspace_bytes)
    chunk /= 2;
  if (chunk == 0) return fail(PAB_EINVAL, "workspace too small for one block");
  if (mode != kFull && chunk < batch)
    return fail(PAB_EINVAL, "split hashing needs the whole batch in one workspace");
  const int msf = byte_order == PAB_ORDER_MSF;
  // LSF blocks whose words can be read in place (the common case): no pack kernel
  // (64-bit coefficients are read as one 8-byte load where the row is 8-byte
  // aligned, as two 4-byte loads elsewhere)
  const u64 al = 4;
  const bool direct_in = !msf && nbytes % al == 0 && in_stride % al == 0 && aligned(x, al) &&
                         aligned(c, al) && aligned(d, al);
  const bool direct_out = !msf && out_stride % 4 == 0 && aligned(out, 4);
  const u32 mask = (n_bits & 31) ? ((1u << (n_bits & 31)) - 1u) : 0xFFFFFFFFu;
  for (u64 b0 = 0; b0 < batch; b0 += chunk) {
    const int nb = (int)((batch - b0) < chunk ? (batch - b0) : chunk);
    const Layout ly = layout_for(g.K, g.md.geo.L, g.K, g.mw, nb, g.md.np);
    ConvJob job = make_job(ly, workspace, g.md, nb);
    job.p0 = p0;
    job.pn = pn;
    job.kA = job.kX = job.kD = (long long)g.K;
    job.maskA = job.maskX = job.maskD = mask;
    job.nT = (long long)g.K;
    job.nRes = (long long)g.KC;
    job.n_mod_bits = (long long)n_bits;
    job.shift = (long long)(n_bits - r_bits);
    job.mw = (long long)g.mw;
    if (mode != kConvOnly)
      CK(cudaMemsetAsync((char*)workspace + ly.off_state, 0, ly.total - ly.off_state, st), "memset");
    if (direct_in) {
      job.srcA = (const u32*)(c + b0 * in_stride);
      job.srcX = (const u32*)(x + b0 * in_stride);
      job.srcD = (const u32*)(d + b0 * in_stride);
      job.src_stride = (long long)(in_stride / 4);
    } else {
      u32* words = (u32*)((char*)workspace + ly.off_words);
      const long long ws = (long long)ly.in_stride;
      if (mode != kCarryOnly) {
        launch_pack(c + b0 * in_stride, (long long)in_stride, (long long)n_bits, msf, nb, words,
                    3 * ws, (long long)g.K, st);
        launch_pack(x + b0 * in_stride, (long long)in_stride, (long long)n_bits, msf, nb,
                    words + ws, 3 * ws, (long long)g.K, st);
      }
      if (mode != kConvOnly)
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
    if (mode != kCarryOnly) launch_conv(job, tab, st);
    if (mode == kConvOnly) {
      CK(cudaGetLastError(), "kernel launch");
      continue;
    }
    launch_carry(job, st);
    if (!direct_out)
      launch_unpack(job.out_words, job.mw, (long long)r_bits, msf, nb, out + b0 * out_stride,
                    (long long)out_stride, st);
    CK(cudaGetLastError(), "kernel launch");
  }
  return PAB_OK;
}

// ================================================================== C ABI
extern "C" {

int pab_version(void) { return 102; }

const char* pab_last_error(void) { return g_err.c_str(); }

// 2K - 1 <= 5 * 2^22 (largest radix-5 length), K < 2^25 (CRT bound)
uint64_t pab_max_bits(void) { return (uint64_t)32 * ((((uint64_t)5 << kMaxLg) + 1) / 2); }

int pab_plan_info(uint64_t n_bits, int* radix, int* lg, int* lg_rows, int* lg_cols) {
  HashGeo g;
  int rc = hash_geo(n_bits, 1, &g);
  if (rc) return rc;
  if (radix) *radix = g.md.geo.m;
  if (lg) *lg = g.md.geo.lg;
  if (lg_rows) *lg_rows = g.md.geo.lgR;
  if (lg_cols) *lg_cols = g.md.geo.lgC;
  return PAB_OK;
}

int pab_plan_width(uint64_t n_bits, int* coef_bits, int* primes) {
  HashGeo g;
  int rc = hash_geo(n_bits, 1, &g);
  if (rc) return rc;
  if (coef_bits) *coef_bits = 32 * g.md.cw;
  if (primes) *primes = g.md.np;
  return PAB_OK;
}

void pab_force_coef_words(int cw) { g_force_cw.store(cw == 1 || cw == 2 ? cw : 0); }

size_t pab_hash_workspace_bytes(uint64_t n_bits, uint32_t batch) {
  HashGeo g;
  if (hash_geo(n_bits, 1, &g)) return 0;
  // output words are bounded by K; size for the largest r
  return layout_for(g.K, g.md.geo.L, g.K, g.K, batch ? batch : 1, g.md.np).total;
}

int pab_hash_batch(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t in_stride,
                   uint64_t n_bits, uint64_t r_bits, uint32_t batch, int byte_order,
                   uint8_t* out, uint64_t out_stride, void* workspace, size_t workspace_bytes,
                   void* stream) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  return hash_batch_impl(x, c, d, in_stride, n_bits, r_bits, batch, byte_order, out, out_stride,
                         workspace, workspace_bytes, stream, 0, g.md.np, kFull);
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

static int host_pipeline(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                         uint64_t r_bits, uint32_t batch, int byte_order, const uint8_t* master,
                         uint64_t master_len, uint64_t first_index, long long bench_index,
                         uint8_t* out, HostCtx& h);

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
  if (!x || !c || !d || !out) return fail(PAB_EINVAL, "null pointer argument");
  // chunks of blocks H2D / hashed / D2H on three streams over three device slots
  return host_pipeline(x, c, d, n_bits, r_bits, batch, byte_order, nullptr, 0, 0, -1, out, h);
}

// Host copies of a few large buffers (the digit path at n ~ 1e8: 40 MB in, 7 MB
// out): one thread moves ~10 GB/s, so split copies above 8 MB over threads (thread start-up costs more below).
static void par_copy(std::initializer_list<std::pair<void*, std::pair<const void*, size_t>>> jobs) {
  size_t total = 0;
  for (const auto& j : jobs) total += j.second.second;
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = total < ((size_t)8 << 20) ? 1u : (hw < 2 ? 1u : (hw > 8 ? 8u : hw));
  if (nt == 1) {
    for (const auto& j : jobs)
      if (j.second.second) std::memcpy(j.first, j.second.first, j.second.second);
    return;
  }
  const size_t per = (total + nt - 1) / nt;
  std::vector<std::thread> th;
  // thread k copies bytes [k * per, (k + 1) * per) of the concatenated jobs
  for (unsigned k = 0; k < nt; ++k) {
    th.emplace_back([&, k] {
      const size_t lo = k * per, hi = lo + per < total ? lo + per : total;
      size_t base = 0;
      for (const auto& j : jobs) {
        const size_t jlo = base, jhi = base + j.second.second;
        const size_t a = lo > jlo ? lo : jlo, b = hi < jhi ? hi : jhi;
        if (a < b)
          std::memcpy((char*)j.first + (a - jlo), (const char*)j.second.first + (a - jlo), b - a);
        base = jhi;
      }
    });
  }
  for (auto& t : th) t.join();
}

int pab_hash_digits(const uint32_t* x, uint64_t x_nd, const uint32_t* c, uint64_t c_nd,
                    const uint32_t* d, uint64_t d_nd, uint64_t n_bits, uint64_t r_bits,
                    uint32_t* out, uint64_t out_nd, int device) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  if ((x_nd && !x) || (c_nd && !c) || (d_nd && !d) || (out_nd && !out))
    return fail(PAB_EINVAL, "null digit array");
  const u64 ndn = ceil_div(n_bits, 30);
  if (out_nd < ceil_div(r_bits, 30)) return fail(PAB_EINVAL, "out_nd must be >= ceil(r/30)");
  // digits >= ceil(n/30) only carry bits >= n, which the hash ignores
  const u64 xn = x_nd < ndn ? x_nd : ndn, cn = c_nd < ndn ? c_nd : ndn,
            dn = d_nd < ndn ? d_nd : ndn;
  CK(cudaSetDevice(device), "cudaSetDevice");
  DevState* ds;
  if ((rc = ensure_device(device, &ds))) return rc;
  HostCtx& h = ds->host;
  std::lock_guard<std::mutex> lk(h.mu);
  const u64 K = ceil_div(n_bits, 32);
  const u64 in_stride = round_up(4 * K, 16);  // bytes per operand row (words)
  const u64 rbytes = ceil_div(r_bits, 8), out_stride = round_up(rbytes, 16);
  const u64 dig_in = 4 * (xn + cn + dn), dig_out = 4 * out_nd;
  const size_t ws_bytes = pab_hash_workspace_bytes(n_bits, 1);
  const size_t io_bytes = 3 * in_stride + round_up(dig_in, 256) + out_stride;
  if ((rc = host_ensure(h, ws_bytes, io_bytes))) return rc;
  const size_t pin_bytes = round_up(dig_in, 256) + round_up(dig_out, 256);
  if (h.pinned_bytes < pin_bytes) {
    if (h.pinned) cudaFreeHost(h.pinned);
    h.pinned = nullptr;
    h.pinned_bytes = 0;
    CK(cudaHostAlloc((void**)&h.pinned, pin_bytes, cudaHostAllocMapped), "pinned alloc");
    CK(cudaHostGetDevicePointer((void**)&h.pinned_dev, h.pinned, 0), "mapped pointer");
    h.pinned_bytes = pin_bytes;
  }
  uint8_t* words = h.dev_io;                        // x, c, d rows
  uint8_t* ddig = words + 3 * in_stride;            // input digits
  uint8_t* dout = ddig + round_up(dig_in, 256);     // key bytes (LSF, 16-byte padded)
  uint8_t* pin_out = h.pinned + round_up(dig_in, 256);
  par_copy({{h.pinned, {x, 4 * xn}},
            {h.pinned + 4 * xn, {c, 4 * cn}},
            {h.pinned + 4 * (xn + cn), {d, 4 * dn}}});
  if (dig_in) CK(cudaMemcpyAsync(ddig, h.pinned, dig_in, cudaMemcpyHostToDevice, h.stream), "H2D");
  DigitOperands ops;
  ops.d[0] = (const u32*)ddig;
  ops.d[1] = ops.d[0] + xn;
  ops.d[2] = ops.d[1] + cn;
  ops.nd[0] = (long long)xn;
  ops.nd[1] = (long long)cn;
  ops.nd[2] = (long long)dn;
  launch_digits_pack(ops, 3, (long long)n_bits, (u32*)words, (long long)(in_stride / 4),
                     (long long)K, h.stream);
  rc = pab_hash_batch(words, words + in_stride, words + 2 * in_stride, in_stride, n_bits, r_bits,
                      1, PAB_ORDER_LSF, dout, out_stride, h.ws, h.ws_bytes, h.stream);
  if (rc) return rc;
  // the key digits go straight to mapped host memory (posted PCIe writes, no D2H copy)
  launch_digits_unpack((const u32*)dout, (long long)r_bits,
                       (u32*)(h.pinned_dev + round_up(dig_in, 256)), (long long)out_nd, h.stream);
  CK(cudaGetLastError(), "kernel launch");
  CK(cudaStreamSynchronize(h.stream), "synchronize");
  par_copy({{out, {pin_out, dig_out}}});
  return PAB_OK;
}

int pab_seed_expand(const uint8_t* master, uint64_t master_len, uint64_t first_index,
                    uint32_t batch, uint64_t n_bits, int byte_order, uint8_t* c, uint8_t* d,
                    uint64_t stride, void* stream) {
  if (n_bits < 1) return fail(PAB_EINVAL, "alpha must be >= 1, got 0");
  if (n_bits > ((u64)1 << 40)) return fail(PAB_ERANGE, "block size beyond the seed expander");
  if (master_len > (u64)kMaxSeedMaster)
    return fail(PAB_EINVAL, "seed material longer than " + std::to_string(kMaxSeedMaster) +
                                " bytes");
  if (master_len && !master) return fail(PAB_EINVAL, "null seed material");
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  if (batch == 0) return PAB_OK;
  if (!c || !d) return fail(PAB_EINVAL, "null pointer argument");
  const u64 nbytes = ceil_div(n_bits, 8);
  if (stride < nbytes) return fail(PAB_EINVAL, "stride smaller than the block byte length");
  if (first_index > ~0ull - batch) return fail(PAB_EINVAL, "block index overflows 64 bits");
  SeedMaster sm;
  std::memset(&sm, 0, sizeof(sm));
  if (master_len) std::memcpy(sm.b, master, master_len);
  const int msf = byte_order == PAB_ORDER_MSF;
  const int word_io = !msf && stride % 8 == 0 && aligned(c, 8) && aligned(d, 8);
  launch_seed_expand(sm, (int)master_len, (unsigned long long)first_index, (int)batch,
                     (long long)n_bits, msf, word_io, c, d, (long long)stride,
                     (cudaStream_t)stream);
  CK(cudaGetLastError(), "kernel launch");
  return PAB_OK;
}

int pab_seed_expand_bench(uint64_t first_seed, uint32_t batch, uint64_t index, uint64_t n_bits,
                          int byte_order, uint8_t* c, uint8_t* d, uint64_t stride, void* stream) {
  if (n_bits < 1) return fail(PAB_EINVAL, "alpha must be >= 1, got 0");
  if (n_bits > ((u64)1 << 40)) return fail(PAB_ERANGE, "block size beyond the seed expander");
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  if (batch == 0) return PAB_OK;
  if (!c || !d) return fail(PAB_EINVAL, "null pointer argument");
  const u64 nbytes = ceil_div(n_bits, 8);
  if (stride < nbytes) return fail(PAB_EINVAL, "stride smaller than the block byte length");
  if (first_seed > ~0ull - batch) return fail(PAB_EINVAL, "block seed overflows 64 bits");
  if (index > (u64)LLONG_MAX) return fail(PAB_EINVAL, "label index beyond 2^63");
  SeedMaster sm;
  std::memset(&sm, 0, sizeof(sm));
  const int msf = byte_order == PAB_ORDER_MSF;
  const int word_io = !msf && stride % 8 == 0 && aligned(c, 8) && aligned(d, 8);
  launch_seed_expand(sm, 0, (unsigned long long)first_seed, (int)batch, (long long)n_bits, msf,
                     word_io, c, d, (long long)stride, (cudaStream_t)stream, (long long)index);
  CK(cudaGetLastError(), "kernel launch");
  return PAB_OK;
}

// Seed windows (in hashing chunks) of a call of `nchunks` chunks: as even as possible,
// none above `target` chunks -- a longer expansion starves the copies -- except a call
// of up to 1.5 targets, which is one window; none above `cap` (the seed budget).
// (paper_1910_04429_b200/batch.py: exclusive_windows, the same policy.)
static std::vector<u64> seed_windows(u64 nchunks, u64 target, u64 cap) {
  if (cap < 1) cap = 1;
  if (target < 1) target = 1;
  const u64 one = target + target / 2 < cap ? target + target / 2 : cap;
  if (nchunks <= one) return {nchunks};
  const u64 t = target < cap ? target : cap;
  const u64 k = ceil_div(nchunks, t);
  std::vector<u64> w(k);
  for (u64 i = 0; i < k; ++i) w[i] = nchunks / k + (i < nchunks % k ? 1 : 0);
  return w;
}

// One call = the whole pipeline (the C counterpart of HashEngine.hash_seeded_host's
// exclusive schedule): the key blocks go H2D chunk by chunk on one stream into
// kSlots device slots, each seed window is expanded on the hashing stream right
// before its chunks are hashed (expansion and hashing never share the SMs), keys
// return D2H on a third stream; per-slot events order slot reuse.  With x and out in
// pinned memory the copies overlap the hashing (n = 1e6: x over PCIe is the bound);
// pageable buffers work too, at the speed the driver stages them.
// The host-buffer pipeline (h.mu held, device current).  c != null: the members come
// from the host with the key blocks (pab_hash_host); else they are expanded on the
// device, bench_index >= 0 selecting the reference benchmark protocol's seeds
// (pab_seed_expand_bench: block j's seed is the integer first_index + j, label index
// bench_index) and bench_index < 0 run_pa's (pab_seed_expand).
static int host_pipeline(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                         uint64_t r_bits, uint32_t batch, int byte_order, const uint8_t* master,
                         uint64_t master_len, uint64_t first_index, long long bench_index,
                         uint8_t* out, HostCtx& h) {
  int rc;
  constexpr int kS = HostCtx::kSlots;
  const bool seeded = c == nullptr;
  const u64 nbytes = ceil_div(n_bits, 8), rbytes = ceil_div(r_bits, 8);
  // rows the kernels can read and write in place stay packed (one contiguous copy per chunk)
  const u64 in_stride = nbytes % 8 == 0 ? nbytes : round_up(nbytes, 16);
  const u64 out_stride = rbytes % 4 == 0 ? rbytes : round_up(rbytes, 16);
  // hashing chunks: at most 1024 blocks and ~2 GiB of transform workspace
  u64 chunk = batch < 1024 ? batch : 1024;
  while (chunk > 1 && pab_hash_workspace_bytes(n_bits, (uint32_t)chunk) > ((size_t)2 << 30))
    chunk /= 2;
  const u64 nchunks = ceil_div(batch, chunk);
  // seed windows: 4096 blocks (8192 XOF streams: a throughput-bound launch) where the
  // 4 GiB seed budget holds them, at least one chunk; host members: no windows
  const u64 cap = (((u64)4 << 30) / (2 * in_stride)) / chunk;
  const u64 target = ceil_div(4096, chunk);
  const std::vector<u64> wins = seeded ? seed_windows(nchunks, target, cap)
                                       : std::vector<u64>{nchunks};
  u64 wmax = 0;
  for (u64 w : wins) wmax = w > wmax ? w : wmax;
  const size_t ws_bytes = pab_hash_workspace_bytes(n_bits, (uint32_t)chunk);
  const size_t slot_bytes = round_up(chunk * ((seeded ? 1 : 3) * in_stride + out_stride), 256);
  const size_t seed_bytes = seeded ? round_up(wmax * chunk * in_stride, 256) : 0;
  if ((rc = host_ensure(h, ws_bytes, kS * slot_bytes + 2 * seed_bytes))) return rc;
  if (!h.p_in) {
    CK(cudaStreamCreateWithFlags(&h.p_in, cudaStreamNonBlocking), "stream");
    CK(cudaStreamCreateWithFlags(&h.p_comp, cudaStreamNonBlocking), "stream");
    CK(cudaStreamCreateWithFlags(&h.p_out, cudaStreamNonBlocking), "stream");
    for (int k = 0; k < kS; ++k) {
      CK(cudaEventCreateWithFlags(&h.ev_in[k], cudaEventDisableTiming), "event");
      CK(cudaEventCreateWithFlags(&h.ev_comp[k], cudaEventDisableTiming), "event");
      CK(cudaEventCreateWithFlags(&h.ev_out[k], cudaEventDisableTiming), "event");
    }
  }
  uint8_t* dc = h.dev_io + kS * slot_bytes;
  uint8_t* dd = dc + seed_bytes;
  u64 b0 = 0, slot = 0;
  for (u64 wlen : wins) {
    const u64 w0 = b0;
    const u64 w1 = w0 + wlen * chunk < batch ? w0 + wlen * chunk : batch;
    if (seeded) {
      rc = bench_index >= 0
               ? pab_seed_expand_bench(first_index + w0, (uint32_t)(w1 - w0), (u64)bench_index,
                                       n_bits, byte_order, dc, dd, in_stride, h.p_comp)
               : pab_seed_expand(master, master_len, first_index + w0, (uint32_t)(w1 - w0),
                                 n_bits, byte_order, dc, dd, in_stride, h.p_comp);
      if (rc) return rc;
    }
    for (; b0 < w1; b0 += chunk, ++slot) {
      const int k = (int)(slot % kS);
      const u64 nb = w1 - b0 < chunk ? w1 - b0 : chunk;
      uint8_t* dx = h.dev_io + k * slot_bytes;
      uint8_t* sc = seeded ? dc + (b0 - w0) * in_stride : dx + chunk * in_stride;
      uint8_t* sd = seeded ? dd + (b0 - w0) * in_stride : dx + 2 * chunk * in_stride;
      uint8_t* dout = dx + (seeded ? 1 : 3) * chunk * in_stride;
      CK(cudaStreamWaitEvent(h.p_in, h.ev_comp[k], 0), "wait");  // slot k's inputs consumed
      CK(cudaMemcpy2DAsync(dx, in_stride, x + b0 * nbytes, nbytes, nbytes, nb,
                           cudaMemcpyHostToDevice, h.p_in), "H2D x");
      if (!seeded) {
        CK(cudaMemcpy2DAsync(sc, in_stride, c + b0 * nbytes, nbytes, nbytes, nb,
                             cudaMemcpyHostToDevice, h.p_in), "H2D c");
        CK(cudaMemcpy2DAsync(sd, in_stride, d + b0 * nbytes, nbytes, nbytes, nb,
                             cudaMemcpyHostToDevice, h.p_in), "H2D d");
      }
      CK(cudaEventRecord(h.ev_in[k], h.p_in), "record");
      CK(cudaStreamWaitEvent(h.p_comp, h.ev_in[k], 0), "wait");
      CK(cudaStreamWaitEvent(h.p_comp, h.ev_out[k], 0), "wait");  // slot k's keys drained
      rc = pab_hash_batch(dx, sc, sd, in_stride, n_bits, r_bits, (uint32_t)nb, byte_order, dout,
                          out_stride, h.ws, h.ws_bytes, h.p_comp);
      if (rc) return rc;
      CK(cudaEventRecord(h.ev_comp[k], h.p_comp), "record");
      CK(cudaStreamWaitEvent(h.p_out, h.ev_comp[k], 0), "wait");
      CK(cudaMemcpy2DAsync(out + b0 * rbytes, rbytes, dout, out_stride, rbytes, nb,
                           cudaMemcpyDeviceToHost, h.p_out), "D2H out");
      CK(cudaEventRecord(h.ev_out[k], h.p_out), "record");
    }
  }
  CK(cudaStreamSynchronize(h.p_in), "synchronize");
  CK(cudaStreamSynchronize(h.p_comp), "synchronize");
  CK(cudaStreamSynchronize(h.p_out), "synchronize");
  return PAB_OK;
}

static int seeded_host_impl(const uint8_t* x, uint64_t n_bits, uint64_t r_bits, uint32_t batch,
                            int byte_order, const uint8_t* master, uint64_t master_len,
                            uint64_t first_index, long long bench_index, uint8_t* out,
                            int device) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  if (batch == 0) return PAB_OK;
  if (!x || !out) return fail(PAB_EINVAL, "null pointer argument");
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  if (first_index > ~0ull - batch) return fail(PAB_EINVAL, "block index overflows 64 bits");
  CK(cudaSetDevice(device), "cudaSetDevice");
  DevState* ds;
  if ((rc = ensure_device(device, &ds))) return rc;
  HostCtx& h = ds->host;
  std::lock_guard<std::mutex> lk(h.mu);
  return host_pipeline(x, nullptr, nullptr, n_bits, r_bits, batch, byte_order, master, master_len,
                       first_index, bench_index, out, h);
}

int pab_hash_seeded_host(const uint8_t* x, uint64_t n_bits, uint64_t r_bits, uint32_t batch,
                         int byte_order, const uint8_t* master, uint64_t master_len,
                         uint64_t first_index, uint8_t* out, int device) {
  return seeded_host_impl(x, n_bits, r_bits, batch, byte_order, master, master_len, first_index,
                          -1, out, device);
}

int pab_hash_seeded_host_bench(const uint8_t* x, uint64_t n_bits, uint64_t r_bits,
                               uint32_t batch, int byte_order, uint64_t first_seed,
                               uint64_t index, uint8_t* out, int device) {
  if (index > (u64)LLONG_MAX) return fail(PAB_EINVAL, "label index beyond 2^63");
  return seeded_host_impl(x, n_bits, r_bits, batch, byte_order, nullptr, 0, first_seed,
                          (long long)index, out, device);
}

int pab_hash_host_split(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                        uint64_t r_bits, uint32_t batch, int byte_order, uint8_t* out,
                        const int* devices, int ndev) {
  HashGeo g;
  int rc = hash_geo(n_bits, r_bits, &g);
  if (rc) return rc;
  if (batch == 0) return PAB_OK;
  if (!x || !c || !d || !out) return fail(PAB_EINVAL, "null pointer argument");
  if (!devices || ndev < 1) return fail(PAB_EINVAL, "need at least one device");
  if (byte_order != PAB_ORDER_LSF && byte_order != PAB_ORDER_MSF)
    return fail(PAB_EINVAL, "byte_order must be PAB_ORDER_LSF or PAB_ORDER_MSF");
  const int np = g.md.np;
  const int nsh = ndev < np ? ndev : np;  // shares of the primes
  const u64 nbytes = ceil_div(n_bits, 8), rbytes = ceil_div(r_bits, 8);
  const u64 in_stride = round_up(nbytes, 16), out_stride = round_up(rbytes, 16);
  const size_t ws_bytes = pab_hash_workspace_bytes(n_bits, batch);
  if (ws_bytes == 0) return fail(PAB_EINVAL, "no workspace size for this block");
  const size_t io_bytes = (size_t)batch * (3 * in_stride + out_stride);
  const Layout ly = layout_for(g.K, g.md.geo.L, g.K, g.mw, batch, np);
  std::lock_guard<std::mutex> lk(g_split_mu);
  struct Share {
    int dev, p0, pn;
    SplitSlot* slot;
  };
  std::vector<Share> sh;
  std::map<int, int> used;  // shares already placed on a device
  for (int s = 0; s < nsh; ++s) {
    Share e;
    e.dev = devices[s];
    e.p0 = (int)((long long)s * np / nsh);
    e.pn = (int)((long long)(s + 1) * np / nsh) - e.p0;
    CK(cudaSetDevice(e.dev), "cudaSetDevice");
    DevState* ds;
    if ((rc = ensure_device(e.dev, &ds))) return rc;
    const int k = used[e.dev]++;
    while ((int)ds->split.size() <= k) ds->split.emplace_back(new SplitSlot());
    SplitSlot& sl = *ds->split[k];
    if (!sl.stream) CK(cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking), "stream");
    if (!sl.done) CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming), "event");
    if (sl.ws_bytes < ws_bytes) {
      if (sl.ws) cudaFree(sl.ws);
      sl.ws = nullptr;
      sl.ws_bytes = 0;
      CK(cudaMalloc(&sl.ws, ws_bytes), "split workspace alloc");
      sl.ws_bytes = ws_bytes;
    }
    if (sl.io_bytes < io_bytes) {
      if (sl.io) cudaFree(sl.io);
      sl.io = nullptr;
      sl.io_bytes = 0;
      CK(cudaMalloc(&sl.io, io_bytes), "split io alloc");
      sl.io_bytes = io_bytes;
    }
    if (e.dev != devices[0]) {  // residues go straight over NVLink when the pair allows it
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[0], e.dev);
      if (can) {
        CK(cudaSetDevice(devices[0]), "cudaSetDevice");
        const cudaError_t pe = cudaDeviceEnablePeerAccess(e.dev, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
          return cuda_fail(pe, "enable peer access");
        cudaGetLastError();
      }
    }
    e.slot = &sl;
    sh.push_back(e);
  }
  // each share: its operands host -> its device, the convolution over its primes
  for (int s = 0; s < nsh; ++s) {
    const Share& e = sh[s];
    CK(cudaSetDevice(e.dev), "cudaSetDevice");
    SplitSlot& sl = *e.slot;
    uint8_t* dx = sl.io;
    uint8_t* dc = dx + batch * in_stride;
    uint8_t* dd = dc + batch * in_stride;
    uint8_t* dout = dd + batch * in_stride;
    CK(cudaMemcpy2DAsync(dx, in_stride, x, nbytes, nbytes, batch, cudaMemcpyHostToDevice,
                         sl.stream), "H2D x");
    CK(cudaMemcpy2DAsync(dc, in_stride, c, nbytes, nbytes, batch, cudaMemcpyHostToDevice,
                         sl.stream), "H2D c");
    if (s == 0)
      CK(cudaMemcpy2DAsync(dd, in_stride, d, nbytes, nbytes, batch, cudaMemcpyHostToDevice,
                           sl.stream), "H2D d");
    if ((rc = hash_batch_impl(dx, dc, dd, in_stride, n_bits, r_bits, batch, byte_order, dout,
                              out_stride, sl.ws, sl.ws_bytes, sl.stream, e.p0, e.pn, kConvOnly)))
      return rc;
    CK(cudaEventRecord(sl.done, sl.stream), "event record");
  }
  // home (share 0): gather the other shares' residue slots, then CRT + carry
  const Share& h = sh[0];
  CK(cudaSetDevice(h.dev), "cudaSetDevice");
  SplitSlot& hs = *h.slot;
  const u64 L = g.md.geo.L;
  const size_t slot_bytes = (size_t)g.KC * 4;  // residues below K' are all the carry reads
  for (int s = 1; s < nsh; ++s) {
    const Share& e = sh[s];
    CK(cudaStreamWaitEvent(hs.stream, e.slot->done, 0), "stream wait");
    for (u32 b = 0; b < batch; ++b)
      for (int P = e.p0; P < e.p0 + e.pn; ++P) {
        const size_t off = ly.off_buf + (((size_t)b * 2 + 0) * np + P) * L * 4;
        CK(cudaMemcpyPeerAsync((char*)hs.ws + off, h.dev, (const char*)e.slot->ws + off, e.dev,
                               slot_bytes, hs.stream), "residue gather");
      }
  }
  uint8_t* hx = hs.io;
  uint8_t* hc = hx + batch * in_stride;
  uint8_t* hd = hc + batch * in_stride;
  uint8_t* hout = hd + batch * in_stride;
  if ((rc = hash_batch_impl(hx, hc, hd, in_stride, n_bits, r_bits, batch, byte_order, hout,
                            out_stride, hs.ws, hs.ws_bytes, hs.stream, 0, np, kCarryOnly)))
    return rc;
  CK(cudaMemcpy2DAsync(out, rbytes, hout, out_stride, rbytes, batch, cudaMemcpyDeviceToHost,
                       hs.stream), "D2H out");
  CK(cudaStreamSynchronize(hs.stream), "synchronize");
  return PAB_OK;
}

// out = acc + a*b over LSF byte strings (acc may be absent).  The product's
// convolution is the hash's; the addend enters the carry kernel as its D
// operand (the hash's +d), and nothing is truncated (n_mod_bits = 32 nT).
static u64 mul_add_words(u64 ka, u64 kb, u64 kacc, u64 out_bytes) {
  const u64 need = (ka + kb > kacc ? ka + kb : kacc) + (kacc ? 1 : 0);
  const u64 have = ceil_div(out_bytes, 4);
  return have > need ? have : need;
}

static size_t mul_add_ws(u64 acc_bytes, u64 a_bytes, u64 b_bytes, u64 out_bytes) {
  const u64 ka = ceil_div(a_bytes, 4), kb = ceil_div(b_bytes, 4), kc = ceil_div(acc_bytes, 4);
  if (ka == 0 || kb == 0) return 256;
  Mode md;
  if (!choose_mode(ka, kb, &md)) return 0;
  const u64 nT = mul_add_words(ka, kb, kc, out_bytes);
  u64 kmax = ka > kb ? ka : kb;
  kmax = kmax > kc ? kmax : kc;
  return layout_for(kmax, md.geo.L, nT, nT, 1, md.np).total;
}

static int mul_add_core(const uint8_t* acc, u64 acc_bytes, const uint8_t* a, u64 a_bytes,
                        const uint8_t* b, u64 b_bytes, uint8_t* out, u64 out_bytes,
                        void* workspace, size_t workspace_bytes, cudaStream_t st) {
  const u64 ka = ceil_div(a_bytes, 4), kb = ceil_div(b_bytes, 4);
  const u64 kc = acc ? ceil_div(acc_bytes, 4) : 0;
  if (out_bytes == 0) return PAB_OK;
  if (ka == 0 || kb == 0) {  // zero product: out = acc, zero padded
    CK(cudaMemsetAsync(out, 0, out_bytes, st), "memset");
    if (acc_bytes && acc)
      CK(cudaMemcpyAsync(out, acc, acc_bytes < out_bytes ? acc_bytes : out_bytes,
                         cudaMemcpyDeviceToDevice, st), "copy addend");
    return PAB_OK;
  }
  Mode md;
  if (!choose_mode(ka, kb, &md))
    return fail(PAB_ERANGE, "operands exceed the exact multi-prime convolution range");
  const u64 nT = mul_add_words(ka, kb, kc, out_bytes);
  const Geo& geo = md.geo;
  u64 kmax = ka > kb ? ka : kb;
  kmax = kmax > kc ? kmax : kc;
  const Layout ly = layout_for(kmax, geo.L, nT, nT, 1, md.np);
  if (workspace_bytes < ly.total) return fail(PAB_EINVAL, "workspace too small");
  int rc;
  DevState* ds;
  if ((rc = current_device(&ds))) return rc;
  const Plan* pl;
  if ((rc = get_plan(ds, geo, &pl))) return rc;
  ConvJob job = make_job(ly, workspace, md, 1);
  job.kA = (long long)ka;
  job.kX = (long long)kb;
  job.kD = (long long)kc;
  job.nT = (long long)nT;
  // product coefficients 0 .. ca + cb - 2 (<= L - 1)
  job.nRes = (long long)(ceil_div(ka, (u64)md.cw) + ceil_div(kb, (u64)md.cw) - 1);
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
  if (kc) {
    launch_pack(acc, (long long)acc_bytes, 8ll * (long long)acc_bytes, 0, 1,
                words + 2 * ly.in_stride, 0, (long long)kc, st);
    job.srcD = words + 2 * ly.in_stride;
  }
  job.src_stride = 0;
  launch_conv(job, tables_of(ds, pl), st);
  launch_carry(job, st);
  launch_unpack(job.out_words, job.mw, 8ll * (long long)out_bytes, 0, 1, out,
                (long long)out_bytes, st);
  CK(cudaGetLastError(), "kernel launch");
  return PAB_OK;
}

static int mul_add_host(const uint8_t* acc, u64 acc_bytes, const uint8_t* a, u64 a_bytes,
                        const uint8_t* b, u64 b_bytes, uint8_t* out, u64 out_bytes, int device) {
  CK(cudaSetDevice(device), "cudaSetDevice");
  DevState* ds;
  int rc;
  if ((rc = ensure_device(device, &ds))) return rc;
  HostCtx& h = ds->host;
  std::lock_guard<std::mutex> lk(h.mu);
  const size_t ws = mul_add_ws(acc_bytes, a_bytes, b_bytes, out_bytes);
  if (ws == 0) return fail(PAB_ERANGE, "operands exceed the exact multi-prime convolution range");
  const size_t io = round_up(a_bytes + 1, 256) + round_up(b_bytes + 1, 256) +
                    round_up(acc_bytes + 1, 256) + round_up(out_bytes + 1, 256);
  if ((rc = host_ensure(h, ws, io))) return rc;
  uint8_t* da = h.dev_io;
  uint8_t* db = da + round_up(a_bytes + 1, 256);
  uint8_t* dacc = db + round_up(b_bytes + 1, 256);
  uint8_t* dout = dacc + round_up(acc_bytes + 1, 256);
  if (a_bytes) CK(cudaMemcpyAsync(da, a, a_bytes, cudaMemcpyHostToDevice, h.stream), "H2D a");
  if (b_bytes) CK(cudaMemcpyAsync(db, b, b_bytes, cudaMemcpyHostToDevice, h.stream), "H2D b");
  if (acc_bytes)
    CK(cudaMemcpyAsync(dacc, acc, acc_bytes, cudaMemcpyHostToDevice, h.stream), "H2D acc");
  rc = mul_add_core(acc_bytes ? dacc : nullptr, acc_bytes, da, a_bytes, db, b_bytes, dout,
                    out_bytes, h.ws, h.ws_bytes, h.stream);
  if (rc) return rc;
  if (out_bytes) CK(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, h.stream), "D2H");
  CK(cudaStreamSynchronize(h.stream), "synchronize");
  return PAB_OK;
}

size_t pab_mul_workspace_bytes(uint64_t a_bytes, uint64_t b_bytes) {
  return mul_add_ws(0, a_bytes, b_bytes, a_bytes + b_bytes);
}

int pab_mul(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes, uint8_t* out,
            void* workspace, size_t workspace_bytes, void* stream) {
  return mul_add_core(nullptr, 0, a, a_bytes, b, b_bytes, out, a_bytes + b_bytes, workspace,
                      workspace_bytes, (cudaStream_t)stream);
}

int pab_mul_host(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes,
                 uint8_t* out, int device) {
  return mul_add_host(nullptr, 0, a, a_bytes, b, b_bytes, out, a_bytes + b_bytes, device);
}

size_t pab_mul_add_workspace_bytes(uint64_t acc_bytes, uint64_t a_bytes, uint64_t b_bytes) {
  const u64 ob = (a_bytes + b_bytes > acc_bytes ? a_bytes + b_bytes : acc_bytes) + 1;
  return mul_add_ws(acc_bytes, a_bytes, b_bytes, ob);
}

int pab_mul_add(const uint8_t* acc, uint64_t acc_bytes, const uint8_t* a, uint64_t a_bytes,
                const uint8_t* b, uint64_t b_bytes, uint8_t* out, uint64_t out_bytes,
                void* workspace, size_t workspace_bytes, void* stream) {
  if (out_bytes < (a_bytes + b_bytes > acc_bytes ? a_bytes + b_bytes : acc_bytes) + 1)
    return fail(PAB_EINVAL, "out_bytes must be >= max(a_bytes + b_bytes, acc_bytes) + 1");
  if (acc_bytes && !acc) return fail(PAB_EINVAL, "null addend");
  return mul_add_core(acc, acc_bytes, a, a_bytes, b, b_bytes, out, out_bytes, workspace,
                      workspace_bytes, (cudaStream_t)stream);
}

int pab_mul_add_host(const uint8_t* acc, uint64_t acc_bytes, const uint8_t* a, uint64_t a_bytes,
                     const uint8_t* b, uint64_t b_bytes, uint8_t* out, uint64_t out_bytes,
                     int device) {
  if (out_bytes < (a_bytes + b_bytes > acc_bytes ? a_bytes + b_bytes : acc_bytes) + 1)
    return fail(PAB_EINVAL, "out_bytes must be >= max(a_bytes + b_bytes, acc_bytes) + 1");
  return mul_add_host(acc, acc_bytes, a, a_bytes, b, b_bytes, out, out_bytes, device);
}

void pab_profile_enable(int enable) { profile_enable(enable != 0); }

int pab_profile_collect(const char** names, int* counts, double* total_ms, int cap) {
  return profile_collect(names, counts, total_ms, cap);
}

}  // extern "C"
