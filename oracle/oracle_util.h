/* oracle_util.h -- TEST INFRASTRUCTURE ONLY: helpers shared by the oracle's
 * single-threaded (aiwc_oracle.c) and multi-threaded (aiwc_oracle_mt.c) drivers. */
#ifndef ORACLE_UTIL_H
#define ORACLE_UTIL_H
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "aiwc_oracle.h"

/* ---- kind codes (include/aiwc_b200.h) ---------------------------------- */
enum {
  K_INSTR = 0x01, K_LOAD = 0x02, K_ATOMIC_LOAD = 0x82, K_STORE = 0x04, K_ATOMIC_STORE = 0x84,
  K_BRANCH = 0x08, K_WI_END = 0x10, K_BARRIER = 0x90, K_WI_BEGIN = 0x30, K_WI_RESUME = 0xB0,
  K_WG_BEGIN = 0x40, K_WG_END = 0xC0, K_KERNEL_BEGIN = 0x20, K_KERNEL_END = 0xA0
};

/* ---- u64 -> u64 open-addressing map (stands in for Python's Counter/dict) -- */
typedef struct {
  uint64_t *keys, *vals;
  uint8_t *used;
  uint64_t cap, size;
} map64;

static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27; x *= 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static inline int map_init(map64 *m, uint64_t cap) {
  m->cap = 16;
  while (m->cap < cap * 2) m->cap <<= 1;
  m->size = 0;
  m->keys = (uint64_t *)malloc(m->cap * 8);
  m->vals = (uint64_t *)malloc(m->cap * 8);
  m->used = (uint8_t *)calloc(m->cap, 1);
  return (m->keys && m->vals && m->used) ? 0 : -1;
}

static inline void map_free(map64 *m) { free(m->keys); free(m->vals); free(m->used); memset(m, 0, sizeof *m); }

/* returns slot; *fresh = 1 when the key was inserted (value zeroed) */
static inline uint64_t map_slot(map64 *m, uint64_t key, int *fresh);

static inline int map_grow(map64 *m) {
  map64 n;
  if (map_init(&n, m->cap) != 0) return -1; /* doubles capacity */
  for (uint64_t i = 0; i < m->cap; i++)
    if (m->used[i]) {
      int f;
      uint64_t s = map_slot(&n, m->keys[i], &f);
      n.vals[s] = m->vals[i];
    }
  map_free(m);
  *m = n;
  return 0;
}

static inline uint64_t map_slot(map64 *m, uint64_t key, int *fresh) {
  if ((m->size + 1) * 2 > m->cap) map_grow(m);
  uint64_t mask = m->cap - 1, i = mix64(key) & mask;
  while (m->used[i]) {
    if (m->keys[i] == key) { *fresh = 0; return i; }
    i = (i + 1) & mask;
  }
  m->used[i] = 1; m->keys[i] = key; m->vals[i] = 0; m->size++;
  *fresh = 1;
  return i;
}

static inline int map_find(const map64 *m, uint64_t key, uint64_t *slot) {
  uint64_t mask = m->cap - 1, i = mix64(key) & mask;
  while (m->used[i]) {
    if (m->keys[i] == key) { *slot = i; return 1; }
    i = (i + 1) & mask;
  }
  return 0;
}

/* ---- growable u64 vector (Python list) ---------------------------------- */
typedef struct { uint64_t *v; uint64_t n, cap; } vec64;
static inline int vec_push(vec64 *a, uint64_t x) {
  if (a->n == a->cap) {
    uint64_t nc = a->cap ? a->cap * 2 : 1024;
    uint64_t *nv = (uint64_t *)realloc(a->v, nc * 8);
    if (!nv) return -1;
    a->v = nv; a->cap = nc;
  }
  a->v[a->n++] = x;
  return 0;
}

static inline int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}
static inline int cmp_u64_desc(const void *a, const void *b) { return cmp_u64(b, a); }

/* Neumaier-compensated sum: numpy's pairwise sum is ~eps accurate, a naive
 * running sum over 10^8 terms is not. */
typedef struct { double s, c; } ksum;
static inline void kadd(ksum *k, double x) {
  double t = k->s + x;
  if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x; else k->c += (x - t) + k->s;
  k->s = t;
}
static inline double kval(const ksum *k) { return k->s + k->c; }

/* coverage_count (entropy.py:49-66): smallest k of the most frequent keys with
 * cumulative >= 9/10 of the total; the Fraction compare is the exact integer
 * test 10*cum >= 9*total (reference.py:57). Sorts `counts` in place. */
static inline uint64_t coverage90(uint64_t *counts, uint64_t n) {
  if (n == 0) return 0;
  qsort(counts, n, 8, cmp_u64_desc);
  unsigned __int128 total = 0, cum = 0;
  for (uint64_t i = 0; i < n; i++) total += counts[i];
  for (uint64_t i = 0; i < n; i++) {
    cum += counts[i];
    if (cum * 10 >= total * 9) return i + 1;
  }
  return n;
}

/* shannon_entropy (entropy.py:20-29): p = c/total; -(sum p*log2 p).
 * A single key gives -(0.0) = -0.0, as in the reference. */
static inline double shannon(const uint64_t *counts, uint64_t n, uint64_t total) {
  ksum k = {0.0, 0.0};
  double t = (double)total;
  for (uint64_t i = 0; i < n; i++) {
    double p = (double)counts[i] / t;
    kadd(&k, p * log2(p));
  }
  return -kval(&k);
}


typedef struct { uint64_t addr, count; } addr_count;
static inline int cmp_addr(const void *a, const void *b) {
  uint64_t x = ((const addr_count *)a)->addr, y = ((const addr_count *)b)->addr;
  return (x > y) - (x < y);
}

typedef struct {
  uint64_t last_group; /* group of this site's current stream */
  uint64_t executions; /* branch_executions() (metrics.py:91-95) */
  uint32_t hist;       /* last history_len outcomes of the current stream, oldest = MSB */
  uint64_t len;        /* length of the current stream */
} site_rec;

typedef struct { uint64_t segment, total; } tally;

/* consume()'s accumulator state (metrics.py:110-124) over one stream or one
 * work-group shard of it */
typedef struct {
  uint32_t H;
  uint64_t table, cap, n_opcodes;
  map64 rd, wr, sites, tal, wmap;
  vec64 itb, ipt, site_ids, wvals, wcnts, wfirst;
  site_rec *srec; uint64_t n_srec, cap_srec;
  tally *tl; uint64_t n_tl, cap_tl;
  uint64_t *opc, *taken_tab, *total_tab;
  uint64_t entries, barriers, work_items, total_instr, excluded, entries_at_fail;
  int64_t current;
  uint64_t open_group;
} acc_state;

/* internal to liboracle.so (hidden: never interposed by, or interposing on, other libraries) */
#define ORACLE_INTERNAL __attribute__((visibility("hidden")))
ORACLE_INTERNAL int oacc_init(acc_state *a, const oracle_params *prm);
ORACLE_INTERNAL int oacc_feed(acc_state *a, const uint8_t *kind, const uint64_t *payload, uint64_t lo, uint64_t hi);
ORACLE_INTERNAL void oacc_close_streams(acc_state *a);
ORACLE_INTERNAL void oacc_free(acc_state *a);
#endif
