/*
 * aiwc_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the
 * reference metric path, used as the parity checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  Nothing in the product path links or calls this file.
 *
 * It restates, event by event, the reference's
 *   consume   pkg/src/aiwc/metrics.py:98-196
 *   finalize  pkg/src/aiwc/metrics.py:273-386
 *   shannon_entropy / local_entropy / coverage_count / branch_entropy
 *             pkg/src/aiwc/entropy.py:20-133
 * over the columnar layout of include/aiwc_b200.h (kind u8 + payload u64).
 * Parity is pinned by tests/test_oracle_golden.py against reports produced by
 * the reference itself (tests/golden/make_golden.py).
 *
 * Real-valued finishing that the reference does in Python on exact integers
 * (median midpoint, means, SIMD mean/sd, ratios, round12) is left to the
 * Python wrapper oracle/oracle.py, which receives the exact integers.
 */
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

static uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27; x *= 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static int map_init(map64 *m, uint64_t cap) {
  m->cap = 16;
  while (m->cap < cap * 2) m->cap <<= 1;
  m->size = 0;
  m->keys = (uint64_t *)malloc(m->cap * 8);
  m->vals = (uint64_t *)malloc(m->cap * 8);
  m->used = (uint8_t *)calloc(m->cap, 1);
  return (m->keys && m->vals && m->used) ? 0 : -1;
}

static void map_free(map64 *m) { free(m->keys); free(m->vals); free(m->used); memset(m, 0, sizeof *m); }

/* returns slot; *fresh = 1 when the key was inserted (value zeroed) */
static uint64_t map_slot(map64 *m, uint64_t key, int *fresh);

static int map_grow(map64 *m) {
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

static uint64_t map_slot(map64 *m, uint64_t key, int *fresh) {
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

static int map_find(const map64 *m, uint64_t key, uint64_t *slot) {
  uint64_t mask = m->cap - 1, i = mix64(key) & mask;
  while (m->used[i]) {
    if (m->keys[i] == key) { *slot = i; return 1; }
    i = (i + 1) & mask;
  }
  return 0;
}

/* ---- growable u64 vector (Python list) ---------------------------------- */
typedef struct { uint64_t *v; uint64_t n, cap; } vec64;
static int vec_push(vec64 *a, uint64_t x) {
  if (a->n == a->cap) {
    uint64_t nc = a->cap ? a->cap * 2 : 1024;
    uint64_t *nv = (uint64_t *)realloc(a->v, nc * 8);
    if (!nv) return -1;
    a->v = nv; a->cap = nc;
  }
  a->v[a->n++] = x;
  return 0;
}

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}
static int cmp_u64_desc(const void *a, const void *b) { return cmp_u64(b, a); }

/* Neumaier-compensated sum: numpy's pairwise sum is ~eps accurate, a naive
 * running sum over 10^8 terms is not. */
typedef struct { double s, c; } ksum;
static void kadd(ksum *k, double x) {
  double t = k->s + x;
  if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x; else k->c += (x - t) + k->s;
  k->s = t;
}
static double kval(const ksum *k) { return k->s + k->c; }

/* coverage_count (entropy.py:49-66): smallest k of the most frequent keys with
 * cumulative >= 9/10 of the total; the Fraction compare is the exact integer
 * test 10*cum >= 9*total (reference.py:57). Sorts `counts` in place. */
static uint64_t coverage90(uint64_t *counts, uint64_t n) {
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
static double shannon(const uint64_t *counts, uint64_t n, uint64_t total) {
  ksum k = {0.0, 0.0};
  double t = (double)total;
  for (uint64_t i = 0; i < n; i++) {
    double p = (double)counts[i] / t;
    kadd(&k, p * log2(p));
  }
  return -kval(&k);
}

typedef struct { uint64_t addr, count; } addr_count;
static int cmp_addr(const void *a, const void *b) {
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

int oracle_run(const uint8_t *kind, const uint64_t *payload, uint64_t n,
               const oracle_params *prm, oracle_result *r) {
  memset(r, 0, sizeof *r);
  const uint32_t H = prm->history_len ? prm->history_len : 16;
  const uint64_t cap = prm->entry_cap;
  const uint64_t table = 1ULL << H;

  map64 rd, wr, sites, tal;
  if (map_init(&rd, 1024) || map_init(&wr, 1024) || map_init(&sites, 64) || map_init(&tal, 1024)) return -1;
  vec64 itb = {0}, ipt = {0}, site_ids = {0};
  site_rec *srec = NULL; uint64_t n_srec = 0, cap_srec = 0;
  tally *tl = NULL; uint64_t n_tl = 0, cap_tl = 0;
  uint64_t *opc = (uint64_t *)calloc(prm->n_opcodes ? prm->n_opcodes : 1, 8);
  /* width Counter in insertion order (metrics.py:136, order drives the sd sum) */
  map64 wmap; map_init(&wmap, 64);
  vec64 wvals = {0}, wcnts = {0}, wfirst = {0};
  uint64_t *taken_tab = (uint64_t *)calloc(table, 8), *total_tab = (uint64_t *)calloc(table, 8);
  if (!opc || !taken_tab || !total_tab) return -1;

  uint64_t entries = 0, barriers = 0, work_items = 0, total_instr = 0;
  uint64_t excluded = 0;
  int64_t current = -1;          /* index into tl; -1 = None */
  uint64_t open_group = 0;       /* checker.open_group (metrics.py:149) */
  int status = 0;

  for (uint64_t i = 0; i < n && status == 0; i++) {
    const uint8_t k = kind[i];
    const uint64_t p = payload[i];
    switch (k) {
      case K_INSTR: { /* metrics.py:131-136 */
        tl[current].segment++; tl[current].total++;
        total_instr++;
        uint32_t op = (uint32_t)(p >> 32), w = (uint32_t)p;
        if (op < prm->n_opcodes) opc[op]++; else { status = 2; break; }
        int fresh; uint64_t s = map_slot(&wmap, w, &fresh);
        if (fresh) { wmap.vals[s] = wvals.n; vec_push(&wvals, w); vec_push(&wcnts, 0); vec_push(&wfirst, i); }
        wcnts.v[wmap.vals[s]]++;
        break;
      }
      case K_LOAD: case K_ATOMIC_LOAD: case K_STORE: case K_ATOMIC_STORE: { /* metrics.py:137-144 */
        map64 *h = (k & 0x02) ? &rd : &wr;
        int fresh; uint64_t s = map_slot(h, p, &fresh);
        if (fresh) {
          entries++;
          if (cap && entries > cap) { status = 1; r->entries_at_fail = entries; break; }
        }
        h->vals[s]++;
        break;
      }
      case K_BRANCH: { /* metrics.py:145-155; histories per (site, group) stream */
        uint64_t site = p >> 1, bit = p & 1;
        int fresh; uint64_t s = map_slot(&sites, site, &fresh);
        if (fresh) {
          if (n_srec == cap_srec) { cap_srec = cap_srec ? cap_srec * 2 : 64; srec = (site_rec *)realloc(srec, cap_srec * sizeof *srec); }
          sites.vals[s] = n_srec;
          srec[n_srec].executions = 0; srec[n_srec].len = 0; srec[n_srec].hist = 0;
          srec[n_srec].last_group = open_group;
          n_srec++;
          vec_push(&site_ids, site);
        }
        site_rec *sr = &srec[sites.vals[s]];
        if (!fresh && sr->last_group != open_group) { /* streams[-1][0] != group -> new stream */
          excluded += sr->len < H ? sr->len : H;
          sr->len = 0; sr->hist = 0; sr->last_group = open_group;
        }
        /* branch_entropy (entropy.py:102-117): execution t >= H of a stream is an
         * observation keyed by the previous H outcomes, oldest as MSB */
        if (sr->len >= H) { total_tab[sr->hist]++; taken_tab[sr->hist] += bit; }
        sr->hist = (uint32_t)(((sr->hist << 1) | bit) & (table - 1));
        sr->len++;
        sr->executions++;
        entries++;
        if (cap && entries > cap) { status = 1; r->entries_at_fail = entries; }
        break;
      }
      case K_BARRIER: /* metrics.py:156-161: always sampled, even 0 */
        barriers++;
        vec_push(&itb, tl[current].segment);
        tl[current].segment = 0;
        current = -1;
        break;
      case K_WI_BEGIN: { /* metrics.py:162-165: fresh tally keyed by global id */
        work_items++;
        if (n_tl == cap_tl) { cap_tl = cap_tl ? cap_tl * 2 : 1024; tl = (tally *)realloc(tl, cap_tl * sizeof *tl); }
        tl[n_tl].segment = 0; tl[n_tl].total = 0;
        int fresh; uint64_t s = map_slot(&tal, (open_group << 32) | (uint32_t)p, &fresh);
        tal.vals[s] = n_tl;
        current = (int64_t)n_tl++;
        break;
      }
      case K_WI_RESUME: { /* metrics.py:166-168 */
        uint64_t s;
        if (!map_find(&tal, (open_group << 32) | (uint32_t)p, &s)) { status = 2; break; }
        current = (int64_t)tal.vals[s];
        break;
      }
      case K_WI_END: /* metrics.py:169-174: trailing segment only when non-empty */
        if (tl[current].segment > 0) vec_push(&itb, tl[current].segment);
        vec_push(&ipt, tl[current].total);
        current = -1;
        break;
      case K_WG_BEGIN: open_group = p; break;
      case K_WG_END: case K_KERNEL_BEGIN: case K_KERNEL_END: break;
      default: status = 2; break;
    }
  }
  r->status = status;
  if (status != 0) goto done;

  /* ---------------- finalize (metrics.py:273-386) ---------------- */
  r->total_instructions = total_instr;
  r->work_items = work_items;
  r->barriers = barriers;
  {
    uint64_t *oc = (uint64_t *)malloc((prm->n_opcodes + 1) * 8), m = 0;
    for (uint32_t o = 0; o < prm->n_opcodes; o++) if (opc[o]) oc[m++] = opc[o];
    r->opcode_cov = coverage90(oc, m);
    free(oc);
  }
  /* ITB / IPT order statistics (summarize_distribution, metrics.py:207-223) */
  vec64 *samp[2] = {&itb, &ipt};
  for (int s = 0; s < 2; s++) {
    vec64 *v = samp[s];
    oracle_dist *d = s ? &r->ipt : &r->itb;
    d->n = v->n;
    if (!v->n) continue;
    qsort(v->v, v->n, 8, cmp_u64);
    d->min = v->v[0]; d->max = v->v[v->n - 1];
    d->mid_lo = v->v[(v->n - 1) / 2]; d->mid_hi = v->v[v->n / 2];
    for (uint64_t i = 0; i < v->n; i++) d->sum += v->v[i];
  }
  /* SIMD width Counter, insertion order */
  r->n_widths = wvals.n;
  r->width_vals = wvals.v; r->width_counts = wcnts.v;
  wvals.v = NULL; wcnts.v = NULL;

  /* memory: merged = Counter(read) + write (metrics.py:308-321) */
  {
    r->unique_reads = rd.size; r->unique_writes = wr.size;
    uint64_t U = 0;
    addr_count *mg = (addr_count *)malloc((rd.size + wr.size + 1) * sizeof *mg);
    map64 merged; map_init(&merged, rd.size + wr.size + 1);
    for (int pass = 0; pass < 2; pass++) {
      map64 *h = pass ? &wr : &rd;
      for (uint64_t i = 0; i < h->cap; i++) {
        if (!h->used[i]) continue;
        if (pass) r->total_writes += h->vals[i]; else r->total_reads += h->vals[i];
        int fresh; uint64_t s = map_slot(&merged, h->keys[i], &fresh);
        if (fresh) { merged.vals[s] = U; mg[U].addr = h->keys[i]; mg[U].count = 0; U++; }
        mg[merged.vals[s]].count += h->vals[i];
      }
    }
    map_free(&merged);
    r->footprint = U;
    uint64_t M = r->total_reads + r->total_writes;
    if (U) {
      uint64_t *cnt = (uint64_t *)malloc(U * 8);
      for (uint64_t i = 0; i < U; i++) cnt[i] = mg[i].count;
      r->gmae = shannon(cnt, U, M);
      /* local_entropy (entropy.py:32-46): re-key by addr >> n, merge, Shannon.
       * Sorting by address makes each re-keyed bin a contiguous run. */
      qsort(mg, U, sizeof *mg, cmp_addr);
      for (int lvl = 1; lvl <= 10; lvl++) {
        uint64_t m = 0;
        for (uint64_t i = 0; i < U; i++) {
          if (i == 0 || (mg[i].addr >> lvl) != (mg[i - 1].addr >> lvl)) cnt[m++] = 0;
          cnt[m - 1] += mg[i].count;
        }
        r->lmae[lvl - 1] = shannon(cnt, m, M);
      }
      for (uint64_t i = 0; i < U; i++) cnt[i] = mg[i].count;
      r->footprint90 = coverage90(cnt, U);
      free(cnt);
    }
    free(mg);
  }

  /* branches (metrics.py:323-341, entropy.py:76-133) */
  {
    for (uint64_t s = 0; s < n_srec; s++) excluded += srec[s].len < H ? srec[s].len : H;
    r->n_sites = n_srec;
    uint64_t *ex = (uint64_t *)malloc((n_srec + 1) * 8);
    for (uint64_t s = 0; s < n_srec; s++) { ex[s] = srec[s].executions; r->executions += ex[s]; }
    r->branch90 = coverage90(ex, n_srec);
    free(ex);
    r->excluded = excluded;
    uint64_t obs = 0;
    for (uint64_t t = 0; t < table; t++) obs += total_tab[t];
    r->observations = obs;
    ksum y = {0, 0}, l = {0, 0};
    for (uint64_t t = 0; t < table && obs; t++) {
      if (!total_tab[t]) continue;
      double tot = (double)total_tab[t];
      double pp = (double)taken_tab[t] / tot, q = 1.0 - pp;
      double h = -((pp > 0 ? pp * log2(pp) : 0.0) + (q > 0 ? q * log2(q) : 0.0));
      double w = tot / (double)obs;
      kadd(&y, w * h);
      kadd(&l, w * (pp < q ? pp : q));
    }
    r->yokota = kval(&y);
    r->linear = kval(&l);
  }

  if (prm->keep_raw) {  /* hand the accumulator over (ownership moves to r->raw) */
    oracle_raw *w = &r->raw;
    w->n_itb = itb.n; w->itb = itb.v; itb.v = NULL;
    w->n_ipt = ipt.n; w->ipt = ipt.v; ipt.v = NULL;
    w->n_opc = prm->n_opcodes; w->opc = opc; opc = NULL;
    w->width_first = wfirst.v; wfirst.v = NULL;
    w->n_sites = n_srec;
    w->site_ids = site_ids.v; site_ids.v = NULL;
    w->site_exec = (uint64_t *)malloc((n_srec + 1) * 8);
    for (uint64_t s = 0; s < n_srec; s++) w->site_exec[s] = srec[s].executions;
    w->table_size = table;
    w->taken_tab = taken_tab; taken_tab = NULL;
    w->total_tab = total_tab; total_tab = NULL;
    map64 *hs[2] = {&rd, &wr};
    for (int q = 0; q < 2; q++) {
      uint64_t *a = (uint64_t *)malloc((hs[q]->size + 1) * 8), *c = (uint64_t *)malloc((hs[q]->size + 1) * 8), m = 0;
      for (uint64_t i = 0; i < hs[q]->cap; i++)
        if (hs[q]->used[i]) { a[m] = hs[q]->keys[i]; c[m] = hs[q]->vals[i]; m++; }
      if (q) { w->n_wr = m; w->wr_addr = a; w->wr_cnt = c; } else { w->n_rd = m; w->rd_addr = a; w->rd_cnt = c; }
    }
  }

done:
  free(wfirst.v);
  map_free(&rd); map_free(&wr); map_free(&sites); map_free(&tal); map_free(&wmap);
  free(itb.v); free(ipt.v); free(site_ids.v); free(srec); free(tl); free(opc);
  free(wvals.v); free(wcnts.v); free(taken_tab); free(total_tab);
  return 0;
}

void oracle_free(oracle_result *r) {
  free(r->width_vals); free(r->width_counts);
  r->width_vals = r->width_counts = NULL;
  oracle_raw *w = &r->raw;
  free(w->itb); free(w->ipt); free(w->opc); free(w->width_first); free(w->site_ids); free(w->site_exec);
  free(w->taken_tab); free(w->total_tab); free(w->rd_addr); free(w->rd_cnt); free(w->wr_addr); free(w->wr_cnt);
  memset(w, 0, sizeof *w);
}
