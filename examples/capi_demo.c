/*
 * Plain-C consumer of the C ABI (include/pa_b200.h): what a non-Python caller of
 * the reference's hash path (pkg/src/modpa/pa.py:175-190, compress) links against.
 *
 *   gcc -O2 -I include examples/capi_demo.c -L paper_1910_04429_b200/_lib -lpa_b200 \
 *       -Wl,-rpath,$PWD/paper_1910_04429_b200/_lib -o capi_demo
 *   ./capi_demo <n_bits> <r_bits> <x.bin> <c.bin> <d.bin> <out.bin>
 *
 * Reads three serialized n-bit blocks (ceil(n/8) bytes, LSF), hashes them on
 * device 0 with pab_hash_host, and writes the ceil(r/8)-byte key.  Without
 * arguments it only prints the ABI version and the largest block size (no GPU
 * needed), which is how the CPU test suite checks that the library links.
 *
 *   ./capi_demo keyfile <n_bits> <r_bits> <blocks> <seed byte> <key.bin> <out.bin>
 *
 * hashes a key file of <blocks> n-bit blocks the way the reference's run_pa does
 * (pkg/src/modpa/bench.py:256-262): block i with gen_seed(n, derive_block_seed(seed, i)),
 * the seeds expanded on the GPU -- one pab_hash_seeded_host call, host buffers in,
 * keys out.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pa_b200.h"

static unsigned char* slurp(const char* path, size_t want) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  unsigned char* buf = (unsigned char*)malloc(want ? want : 1);
  size_t got = buf ? fread(buf, 1, want, f) : 0;
  fclose(f);
  if (got != want) {
    free(buf);
    return NULL;
  }
  return buf;
}

int main(int argc, char** argv) {
  printf("pa_b200 ABI %d, max block %llu bits\n", pab_version(),
         (unsigned long long)pab_max_bits());
  if (argc >= 8 && strcmp(argv[1], "keyfile") == 0) {
    const unsigned long long kn = strtoull(argv[2], NULL, 10), kr = strtoull(argv[3], NULL, 10);
    const unsigned long blocks = strtoul(argv[4], NULL, 10);
    const unsigned char seed = (unsigned char)strtoul(argv[5], NULL, 10);  /* rng_seed < 256 */
    const size_t knb = (size_t)((kn + 7) / 8), krb = (size_t)((kr + 7) / 8);
    unsigned char* key = slurp(argv[6], knb * blocks);
    unsigned char* keys = (unsigned char*)malloc(krb * blocks + 1);
    if (!key || !keys) {
      fprintf(stderr, "cannot read %lu blocks of %zu bytes\n", blocks, knb);
      return 2;
    }
    const int rc = pab_hash_seeded_host(key, kn, kr, (uint32_t)blocks, PAB_ORDER_LSF, &seed, 1, 0,
                                        keys, 0);
    if (rc != PAB_OK) {
      fprintf(stderr, "pab_hash_seeded_host: %d (%s)\n", rc, pab_last_error());
      return 1;
    }
    FILE* kf = fopen(argv[7], "wb");
    if (!kf || fwrite(keys, 1, krb * blocks, kf) != krb * blocks) return 3;
    fclose(kf);
    free(key), free(keys);
    return 0;
  }
  if (argc < 7) return 0;
  const unsigned long long n = strtoull(argv[1], NULL, 10), r = strtoull(argv[2], NULL, 10);
  const size_t nb = (size_t)((n + 7) / 8), rb = (size_t)((r + 7) / 8);
  unsigned char *x = slurp(argv[3], nb), *c = slurp(argv[4], nb), *d = slurp(argv[5], nb);
  unsigned char* out = (unsigned char*)malloc(rb ? rb : 1);
  if (!x || !c || !d || !out) {
    fprintf(stderr, "cannot read the %zu-byte input blocks\n", nb);
    return 2;
  }
  const int rc = pab_hash_host(x, c, d, n, r, 1, PAB_ORDER_LSF, out, 0);
  if (rc != PAB_OK) {
    fprintf(stderr, "pab_hash_host: %d (%s)\n", rc, pab_last_error());
    return 1;
  }
  FILE* f = fopen(argv[6], "wb");
  if (!f || fwrite(out, 1, rb, f) != rb) return 3;
  fclose(f);
  free(x), free(c), free(d), free(out);
  return 0;
}
