/* sma_c_demo.c -- drive libsma through its C ABI alone (no Python, no torch).
 *
 * Build:  gcc -O2 -I include examples/sma_c_demo.c -L paper_1901_02244_b200 -lsma \
 *             -Wl,-rpath,$PWD/paper_1901_02244_b200 -o sma_c_demo
 * Run:    ./sma_c_demo [d] [k] [rounds] [z_out.bin]
 * Creates an SMA handle (Alg. 1, arXiv 1901.02244) with w0 = 0, registers the
 * handle's synthetic gradients each round, runs `rounds` rounds on the legacy
 * stream and prints z[0..3] and the replica-kernel time; with a fourth
 * argument it also writes all d floats of z (raw little-endian fp32) there.
 * Exit code 0 on success; on any error it prints sma_last_error() and exits 1.
 */
#include <stdio.h>
#include <stdlib.h>

#include "sma.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    sma_status _s = (call);                                                      \
    if (_s != SMA_OK) {                                                          \
      fprintf(stderr, "%s -> %d: %s\n", #call, (int)_s, sma_last_error());      \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(int argc, char** argv) {
  const int64_t d = argc > 1 ? atoll(argv[1]) : 1000003;
  const int32_t k = argc > 2 ? atoi(argv[2]) : 4;
  const int rounds = argc > 3 ? atoi(argv[3]) : 10;
  float* w0 = (float*)calloc((size_t)d, sizeof(float));
  float* z = (float*)malloc(sizeof(float) * (size_t)d);
  sma_config cfg = {d, k, 1.0f / (float)k, 0.1f, 0.9f, 0, 1, 0, NULL, SMA_FLAG_TIMING};
  sma_handle* h = NULL;
  CHECK(sma_create(&cfg, w0, &h));
  for (int i = 0; i < rounds; ++i) {
    CHECK(sma_synth_grads(h, i, 2244, NULL));
    CHECK(sma_step(h, NULL));
  }
  CHECK(sma_get_central(h, z, 0));
  double ms = 0;
  int64_t n = 0;
  CHECK(sma_kernel_time(h, SMA_PHASE_REPLICA, &ms, &n, 0));
  printf("abi=%d d=%lld k=%d rounds=%d z[0..3]=%.9g %.9g %.9g %.9g replica_kernel_ms=%.4f launches=%lld\n",
         sma_abi_version(), (long long)d, k, rounds, z[0], z[1], z[2], z[3], n ? ms / n : 0.0,
         (long long)sma_launch_count(h));
  if (argc > 4) {
    FILE* f = fopen(argv[4], "wb");
    if (!f || fwrite(z, sizeof(float), (size_t)d, f) != (size_t)d) {
      fprintf(stderr, "cannot write %s\n", argv[4]);
      return 1;
    }
    fclose(f);
  }
  sma_destroy(h);
  free(w0);
  free(z);
  return 0;
}
