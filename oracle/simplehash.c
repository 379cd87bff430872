/* Plain-C restatement of the reference simplehash -- TEST INFRASTRUCTURE ONLY.
 *
 * Follows /root/reference/pkg/src/churncomm/sharedstate.py:
 *   constants            :24-28  (FNV offset/prime, 256 lanes, depth 8, rotl 27)
 *   _word_array          :45-54  (little-endian u32 words, tail zero-padded)
 *   _lane_slice          :57-72  (lane i mod 256 runs h = (h ^ w) * P)
 *   _tree_fold           :75-84  (pairs (2j, 2j+1): (a ^ rotl(b, 27)) * P, x8)
 *   simplehash_reference :108-128 (root ^ byte length)
 * and SPEC.md:278-295.
 *
 * Used by tests/ as the checker and by bench.py as the timed CPU baseline
 * (`oracle_simplehash_many` hashes entries on up to `threads` pthreads, each
 * entry single-threaded like the reference's workers=1 path). Never linked by
 * the product.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FNV_OFFSET 0xcbf29ce484222325ULL
#define FNV_PRIME 0x100000001b3ULL
#define LANES 256
#define DEPTH 8
#define ROT 27

static inline uint64_t rotl64(uint64_t v, unsigned r) { return (v << r) | (v >> (64 - r)); }

uint64_t oracle_simplehash(const uint8_t *data, uint64_t nbytes) {
  uint64_t lanes[LANES];
  for (int i = 0; i < LANES; ++i) lanes[i] = FNV_OFFSET;
  uint64_t full = nbytes / 4;
  uint64_t rounds = full / LANES;
  const uint8_t *p = data;
  for (uint64_t r = 0; r < rounds; ++r) {
    for (int l = 0; l < LANES; ++l) {
      uint32_t w;
      memcpy(&w, p + 4 * l, 4); /* host is little-endian (x86/arm64) */
      lanes[l] = (lanes[l] ^ (uint64_t)w) * FNV_PRIME;
    }
    p += 4 * LANES;
  }
  uint64_t words_left = full - rounds * LANES;
  uint64_t i = 0;
  for (; i < words_left; ++i) {
    uint32_t w;
    memcpy(&w, p + 4 * i, 4);
    lanes[i] = (lanes[i] ^ (uint64_t)w) * FNV_PRIME;
  }
  uint64_t tail = nbytes % 4;
  if (tail) {
    uint32_t w = 0;
    for (uint64_t b = 0; b < tail; ++b) w |= (uint32_t)p[4 * i + b] << (8 * b);
    lanes[i] = (lanes[i] ^ (uint64_t)w) * FNV_PRIME;
  }
  int width = LANES;
  for (int d = 0; d < DEPTH; ++d) {
    width /= 2;
    for (int j = 0; j < width; ++j)
      lanes[j] = (lanes[2 * j] ^ rotl64(lanes[2 * j + 1], ROT)) * FNV_PRIME;
  }
  return lanes[0] ^ nbytes;
}

struct job {
  const uint8_t *const *ptrs;
  const uint64_t *nbytes;
  uint64_t *out;
  uint32_t count;
  uint32_t *next;
  pthread_mutex_t *mu;
};

static void *worker(void *arg) {
  struct job *j = (struct job *)arg;
  for (;;) {
    pthread_mutex_lock(j->mu);
    uint32_t k = (*j->next)++;
    pthread_mutex_unlock(j->mu);
    if (k >= j->count) return NULL;
    j->out[k] = oracle_simplehash(j->ptrs[k], j->nbytes[k]);
  }
}

/* Hash `count` entries; entries are dealt to `threads` workers in order
 * (callers pass them largest-first for balance). */
int oracle_simplehash_many(const uint8_t *const *ptrs, const uint64_t *nbytes, uint32_t count,
                           uint64_t *out, int threads) {
  if (threads < 1) threads = 1;
  if ((uint32_t)threads > count) threads = (int)(count ? count : 1);
  uint32_t next = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  struct job j = {ptrs, nbytes, out, count, &next, &mu};
  pthread_t *t = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  if (!t) return -1;
  for (int i = 0; i < threads; ++i) pthread_create(&t[i], NULL, worker, &j);
  for (int i = 0; i < threads; ++i) pthread_join(t[i], NULL);
  free(t);
  return 0;
}
