/*
 * pa_b200.h -- C ABI of the B200-native modular-arithmetic PA hash.
 *
 * The hash (reference: modpa, arxiv/paper_1910_04429) is
 *     y = floor(((c * x + d) mod 2^n) / 2^(n - r)),   c odd,
 * over n-bit blocks x and a per-block seed (c, d).  Blocks are byte strings
 * of ceil(n/8) bytes in the reference's layout: bit i of the block is bit i
 * of its integer value, bytes least-significant-first (LSF, default) or
 * most-significant-first (MSF), zero padded at the most-significant end
 * (pkg/src/modpa/pa.py:8-11, 111-132).  Outputs are ceil(r/8) bytes per
 * block in the same byte order.
 *
 * The reference has no FFI: its seam is the Python functions listed at each
 * entry point below.  This header is what the Python drop-in
 * (paper_1910_04429_b200/pa.py, bignum.py) binds with ctypes; see
 * INTEGRATION.md for the binding a modpa maintainer would add.
 *
 * Conventions: every function returns PAB_OK (0) or a negative PAB_E* code
 * and never throws; pab_last_error() returns a thread-local message for the
 * last failure on the calling thread.  Device pointers must be CUDA device
 * memory of the current device; `stream` is a cudaStream_t (NULL = legacy
 * default stream).  All entry points are reentrant; tables are built once
 * per (device, transform length) under a mutex and never freed.
 */
#ifndef PA_B200_H
#define PA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAB_OK 0
#define PAB_EINVAL (-1) /* bad argument (message in pab_last_error) */
#define PAB_ENOMEM (-2) /* device allocation failed -> Python MemoryError */
#define PAB_ECUDA (-3)  /* any other CUDA error */
#define PAB_ERANGE (-4) /* size beyond the exact-convolution bound */

#define PAB_ORDER_LSF 0 /* WordOrder.LEAST_SIGNIFICANT_FIRST, pkg/src/modpa/bignum.py:27-31 */
#define PAB_ORDER_MSF 1 /* WordOrder.MOST_SIGNIFICANT_FIRST */

/* ABI version (major*100 + minor). */
int pab_version(void);
/* Thread-local description of the last error on this thread ("" if none). */
const char* pab_last_error(void);
/* Largest block size n (bits) the exact convolution supports (32-bit coefficients, three primes). */
uint64_t pab_max_bits(void);

/*
 * Transform geometry chosen for an n-bit hash: length L = radix * 2^lg (radix
 * 1, 3 or 5), split into columns of R = radix * 2^lg_rows rows and rows of
 * C = 2^lg_cols (lg_rows == 0: one CTA per block and prime).  Any pointer may
 * be NULL.
 */
int pab_plan_info(uint64_t n_bits, int* radix, int* lg, int* lg_rows, int* lg_cols);

/*
 * Convolution mode chosen for an n-bit hash: coefficient width (64: two words
 * per coefficient over five NTT primes, used up to 121,295,104 bits; 32: one
 * word over three primes, beyond) and the number of primes.  Any pointer may
 * be NULL.
 */
int pab_plan_width(uint64_t n_bits, int* coef_bits, int* primes);

/*
 * Test hook: force the coefficient width (1 or 2 words) wherever it is valid,
 * 0 restores the automatic choice.  Process-wide; results are identical in
 * every mode, only the work differs.
 */
void pab_force_coef_words(int words);

/*
 * Device workspace needed to hash `batch` n-bit blocks in one pass.
 * pab_hash_batch processes larger batches in chunks that fit the workspace
 * it is given (at least one block must fit).
 */
size_t pab_hash_workspace_bytes(uint64_t n_bits, uint32_t batch);

/*
 * Batched, device-resident hash.  Replaces, per block i,
 *   export_block(compress(import_block(x_i), HashSeed(c_i, d_i, n), r))
 * i.e. pkg/src/modpa/pa.py:175-190 (compress) with the byte layout of
 * import_block/export_block (pa.py:111-132).
 *   x, c, d : device, block i at offset i*in_stride, ceil(n/8) bytes each
 *   out     : device, block i at offset i*out_stride, ceil(r/8) bytes each
 * Requirements (checked in Python by the drop-in, as in the reference):
 * 1 <= r <= n <= pab_max_bits(); c odd; bits >= n of x, c, d are ignored.
 */
int pab_hash_batch(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t in_stride,
                   uint64_t n_bits, uint64_t r_bits, uint32_t batch, int byte_order,
                   uint8_t* out, uint64_t out_stride, void* workspace, size_t workspace_bytes,
                   void* stream);

/*
 * Host-buffer hash on `device` (the drop-in compress / pa_round path,
 * pkg/src/modpa/pa.py:175-217): copies x, c, d (batch*ceil(n/8) bytes each,
 * contiguous) host->device, hashes, copies batch*ceil(r/8) bytes back.
 * Batches run in chunks of up to 1024 blocks over three streams (H2D, hashing,
 * D2H) and three device slots, so with pinned buffers the copies overlap the
 * hashing; blocks of n <= 2048 bits take one kernel over mapped memory.
 * Uses a per-device cached workspace; blocks until done.
 */
int pab_hash_host(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                  uint64_t r_bits, uint32_t batch, int byte_order, uint8_t* out, int device);

/*
 * Host hash over CPython integer digits (the drop-in compress / pa_round path
 * with Python ints, pkg/src/modpa/pa.py:175-217): x, c, d are magnitudes as
 * 30-bit digits in 32-bit slots, least significant first (CPython's own int
 * layout, sys.int_info.bits_per_digit == 30), x_nd / c_nd / d_nd digits each
 * (missing high digits are zero, bits >= n ignored).  out receives out_nd >=
 * ceil(r/30) digits of the key (not normalized: high digits may be zero).
 * The digit <-> word conversion runs on the GPU.  Blocks until done.
 */
int pab_hash_digits(const uint32_t* x, uint64_t x_nd, const uint32_t* c, uint64_t c_nd,
                    const uint32_t* d, uint64_t d_nd, uint64_t n_bits, uint64_t r_bits,
                    uint32_t* out, uint64_t out_nd, int device);

/*
 * Host layout conversions of the drop-in boundary (import_block /
 * export_block, pkg/src/modpa/pa.py:111-132): CPython int digits (30-bit
 * payload in 32-bit slots, least significant first) <-> nbytes serialized
 * bytes in byte_order.  pab_digits_to_bytes writes exactly nbytes bytes (bits
 * beyond them are dropped, missing digits are zero); pab_bytes_to_digits fills
 * nd digits (zero beyond the input).  Pure host code, no device involved.
 */
int pab_digits_to_bytes(const uint32_t* dig, uint64_t nd, uint8_t* out, uint64_t nbytes,
                        int byte_order);
int pab_bytes_to_digits(const uint8_t* in, uint64_t nbytes, int byte_order, uint32_t* dig,
                        uint64_t nd);

/*
 * One batch hashed with its NTT primes split over several GPUs (SURVEY.md
 * §8f: single-block multi-GPU).  The convolution modulo each prime is
 * independent, so share s of `ndev` computes the residues for its contiguous
 * run of primes on devices[s]; the other shares' residue slots are then copied
 * to devices[0] (peer to peer over NVLink where the pair allows it) for the
 * CRT + carry.  Lowers the latency of one large block; throughput stays best
 * with whole blocks per GPU (pab_hash_batch).  Host buffers as pab_hash_host;
 * a device may repeat (its shares run on separate streams).  Blocks until done.
 */
int pab_hash_host_split(const uint8_t* x, const uint8_t* c, const uint8_t* d, uint64_t n_bits,
                        uint64_t r_bits, uint32_t batch, int byte_order, uint8_t* out,
                        const int* devices, int ndev);

/*
 * Seed expansion on the device (SHAKE-256): for j < batch, the hash-family
 * member of block i = first_index + j exactly as run_pa derives it,
 *   gen_seed(n, derive_block_seed(master, i))          pkg/src/modpa/pa.py:156-172
 * with _expand (pa.py:138-153) as the XOF; run_pa's call site is
 * pkg/src/modpa/bench.py:258.  master = the seed material bytes (an int seed s
 * is s.to_bytes(max(1, ceil(bitlen/8)), "little"), pa.py:142-144), at most 1024
 * bytes, host memory.  c and d (device) receive ceil(n/8) bytes per block at
 * offset j*stride in byte_order (c with its low bit set, bits >= n cleared),
 * ready for pab_hash_batch.  Asynchronous on `stream`.
 */
int pab_seed_expand(const uint8_t* master, uint64_t master_len, uint64_t first_index,
                    uint32_t batch, uint64_t n_bits, int byte_order, uint8_t* c, uint8_t* d,
                    uint64_t stride, void* stream);

/*
 * Seed expansion of the reference's benchmark protocol (pkg/src/modpa/bench.py:156,
 * run_bench's inputs; BASELINE configs' per-block seeds): block j gets
 *   gen_seed(n, derive_block_seed(s, index)),   s = first_seed + j,
 * i.e. the integer s itself is the seed material and the label index is fixed
 * (the reference passes index = n).  Outputs and layout as pab_seed_expand.
 */
int pab_seed_expand_bench(uint64_t first_seed, uint32_t batch, uint64_t index, uint64_t n_bits,
                          int byte_order, uint8_t* c, uint8_t* d, uint64_t stride, void* stream);

/*
 * Host-buffer run_pa step on `device` (pkg/src/modpa/bench.py:256-262 for a
 * contiguous run of blocks): x = batch*ceil(n/8) host bytes (blocks first_index
 * .. first_index+batch-1 of the key file), seeds derived on the device by
 * pab_seed_expand, out = batch*ceil(r/8) host bytes.  Blocks until done.
 * One call is the whole pipeline: the key blocks go host -> device in chunks of up
 * to 1024 blocks on one stream, each seed window (4096 blocks where 4 GiB hold it)
 * is expanded on the hashing stream right before its chunks, keys return on a
 * third stream; three device slots.  Hand it a whole shard.  With x and out in
 * pinned (page-locked) memory the copies overlap the hashing and x over PCIe is
 * the bound (n = 1e6: 2.6 ms per 1024 blocks); pageable buffers are staged by the
 * driver (about 7x slower there).
 */
int pab_hash_seeded_host(const uint8_t* x, uint64_t n_bits, uint64_t r_bits, uint32_t batch,
                         int byte_order, const uint8_t* master, uint64_t master_len,
                         uint64_t first_index, uint8_t* out, int device);

/*
 * The same call on the reference benchmark protocol's seeds (pab_seed_expand_bench,
 * pkg/src/modpa/bench.py:156): block j is hashed with
 * gen_seed(n, derive_block_seed(first_seed + j, index)).
 */
int pab_hash_seeded_host_bench(const uint8_t* x, uint64_t n_bits, uint64_t r_bits,
                               uint32_t batch, int byte_order, uint64_t first_seed,
                               uint64_t index, uint8_t* out, int device);

/*
 * Exact product of two naturals given as LSF byte strings (bignum.mul,
 * pkg/src/modpa/bignum.py:194-231): out receives a_bytes + b_bytes LSF bytes.
 */
size_t pab_mul_workspace_bytes(uint64_t a_bytes, uint64_t b_bytes);
int pab_mul(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes, uint8_t* out,
            void* workspace, size_t workspace_bytes, void* stream);
int pab_mul_host(const uint8_t* a, uint64_t a_bytes, const uint8_t* b, uint64_t b_bytes,
                 uint8_t* out, int device);

/*
 * Fused multiply-add (bignum.fused_mul_add, pkg/src/modpa/bignum.py:234-238):
 * out = acc + a*b over LSF byte strings, out_bytes >= max(a_bytes + b_bytes,
 * acc_bytes) + 1 (zero padded).  The addend rides in the carry kernel (the
 * hash's +d); no truncation.  Device variant asynchronous on `stream`; the
 * host variant blocks, like pab_mul_host.
 */
size_t pab_mul_add_workspace_bytes(uint64_t acc_bytes, uint64_t a_bytes, uint64_t b_bytes);
int pab_mul_add(const uint8_t* acc, uint64_t acc_bytes, const uint8_t* a, uint64_t a_bytes,
                const uint8_t* b, uint64_t b_bytes, uint8_t* out, uint64_t out_bytes,
                void* workspace, size_t workspace_bytes, void* stream);
int pab_mul_add_host(const uint8_t* acc, uint64_t acc_bytes, const uint8_t* a, uint64_t a_bytes,
                     const uint8_t* b, uint64_t b_bytes, uint8_t* out, uint64_t out_bytes,
                     int device);

/*
 * Optional per-kernel timing: while enabled, CUDA events are recorded on the
 * launching stream around every kernel.  pab_profile_collect synchronizes on
 * them, aggregates by kernel name (static strings) into the caller's arrays
 * (at most `cap` names) and clears the record; returns the number of names.
 */
void pab_profile_enable(int enable);
int pab_profile_collect(const char** names, int* counts, double* total_ms, int cap);

#ifdef __cplusplus
}
#endif

#endif /* PA_B200_H */
