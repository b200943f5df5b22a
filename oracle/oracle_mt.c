/*
 * oracle_mt.c — a multi-threaded form of the u16 oracle, for TIMING ONLY (the
 * cpu_baseline of bench.py on the host cores of the GPU box).  TEST / BENCH
 * INFRASTRUCTURE ONLY, like oracle.c; shares no code with the CUDA path.
 *
 * It is the paper's own CPU scheme (§III.A-B, Local Thread
 * Update then Global Histogram Update): every thread counts its contiguous
 * share of the keys into a private histogram; the private histograms are summed
 * into the global one; one exclusive scan (Alg. 3); then every thread
 * reconstructs its own range of output positions (Alg. 5 with t = 0) with the
 * single-threaded oracle's oracle_reconstruct_counts_u16.  POSIX threads, two
 * joins (no barrier objects).  Pinned against oracle_sort_u16 by
 * tests/test_oracle_pins.py.
 */
#include <pthread.h>
#include <stdlib.h>

#include "oracle.h"

typedef struct {
  const uint16_t* keys;
  uint16_t* out;
  uint64_t a, b;  /* this thread's share of the keys, then of the output */
  uint64_t* H;    /* private histogram (step 1) */
  uint64_t* C;    /* merged histogram (steps 2, 3) */
} mt_arg;

static void* count_part(void* p) { /* local thread update */
  mt_arg* x = (mt_arg*)p;
  oracle_histogram_u16(x->keys + x->a, x->b - x->a, x->H);
  return NULL;
}

static void* expand_part(void* p) { /* ReconstructAll of this thread's output range */
  mt_arg* x = (mt_arg*)p;
  oracle_reconstruct_counts_u16(x->C, 65536, x->a, x->b, x->out + x->a);
  return NULL;
}

int oracle_sort_u16_mt(const uint16_t* keys, uint64_t n, uint16_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 1024) nthreads = 1024;
  const int T = nthreads;
  uint64_t* H = (uint64_t*)calloc((size_t)T * 65536, sizeof(uint64_t));
  uint64_t* C = (uint64_t*)calloc(65536, sizeof(uint64_t));
  mt_arg* arg = (mt_arg*)calloc((size_t)T, sizeof(mt_arg));
  pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
  if (!H || !C || !arg || !th) {
    free(H); free(C); free(arg); free(th);
    return 1;
  }
  for (int t = 0; t < T; ++t) {
    arg[t].keys = keys;
    arg[t].out = out;
    arg[t].a = n * (uint64_t)t / (uint64_t)T;
    arg[t].b = n * (uint64_t)(t + 1) / (uint64_t)T;
    arg[t].H = H + (size_t)t * 65536;
    arg[t].C = C;
  }
  int rc = 0;
  for (int t = 1; t < T; ++t) rc |= pthread_create(&th[t], NULL, count_part, &arg[t]);
  count_part(&arg[0]);
  for (int t = 1; t < T; ++t) rc |= pthread_join(th[t], NULL);
  for (int v = 0; v < 65536; ++v) { /* global histogram update: sum of the private ones */
    uint64_t s = 0;
    for (int r = 0; r < T; ++r) s += H[(size_t)r * 65536 + v];
    C[v] = s;
  }
  for (int t = 1; t < T; ++t) rc |= pthread_create(&th[t], NULL, expand_part, &arg[t]);
  expand_part(&arg[0]);
  for (int t = 1; t < T; ++t) rc |= pthread_join(th[t], NULL);
  free(H); free(C); free(arg); free(th);
  return rc ? 2 : 0;
}
