/*
 * streams.c — host twin of the device's uniform candidate stream.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): bench.py's parity block
 * and its reference arm regenerate, on the host, exactly the candidates the
 * GPU arm generated with ls_generate(LS_GEN_UNIFORM, seed, start, n) so both
 * arms and the checker see identical inputs. It restates
 * paper_2509_00217_b200/generator.py (GEN_UNIFORM) in C for speed; the CPU
 * test tests/test_streams_cpu.py pins the two against each other.
 *
 * Stream position i -> two splitmix64 draws -> a uniform coarse rank over the
 * tp/ep/pp/batch domains and a uniform axis rank over 3^(A-4), each split
 * mixed-radix (last head fastest) into the index vector
 * (baselines.uniform_vector semantics, reference baselines.py:50-54).
 */
#include <pthread.h>
#include <stdint.h>

#include "../include/ls_eval.h"

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t mulhi64(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

typedef struct {
  const ls_workload_desc* m;
  uint64_t seed;
  int64_t start, lo, hi, stride;
  uint8_t* planes;
} gen_job_t;

static void gen_range(const gen_job_t* j) {
  const ls_workload_desc* m = j->m;
  const int A = m->vector_length;
  uint64_t coarse_size = 1, axis_size = 1;
  int h;
  for (h = 0; h < 4; ++h) coarse_size *= (uint64_t)m->domain_len[h];
  for (h = 4; h < A; ++h) axis_size *= 3u;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    const uint64_t g = (uint64_t)(j->start + i);
    uint64_t coarse = mulhi64(splitmix64(j->seed ^ (2u * g)), coarse_size);
    uint64_t axis = mulhi64(splitmix64(j->seed ^ (2u * g + 1u)), axis_size);
    for (h = 3; h >= 0; --h) {
      const uint64_t k = (uint64_t)m->domain_len[h];
      j->planes[(int64_t)h * j->stride + i] = (uint8_t)(coarse % k);
      coarse /= k;
    }
    for (h = A - 1; h >= 4; --h) {
      j->planes[(int64_t)h * j->stride + i] = (uint8_t)(axis % 3u);
      axis /= 3u;
    }
  }
}

static void* gen_run(void* arg) {
  gen_range((const gen_job_t*)arg);
  return NULL;
}

/* Stream positions [start, start + n) of the uniform stream as [A, stride]
 * uint8 SoA planes, over `threads` pthreads. A <= 16 (as on the device). */
int or_gen_uniform(const ls_workload_desc* m, uint64_t seed, int64_t start, int64_t n, uint8_t* planes,
                   int64_t stride, int threads) {
  pthread_t tid[256];
  gen_job_t jobs[256];
  int t;
  if (m->vector_length > 16 || n < 0 || stride < n) return -1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  for (t = 0; t < threads; ++t) {
    jobs[t].m = m;
    jobs[t].seed = seed;
    jobs[t].start = start;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    jobs[t].stride = stride;
    jobs[t].planes = planes;
    if (threads == 1) gen_run(&jobs[t]);
    else pthread_create(&tid[t], NULL, gen_run, &jobs[t]);
  }
  if (threads > 1)
    for (t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}
