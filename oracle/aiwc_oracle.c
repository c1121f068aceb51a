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

#include "oracle_util.h"




int oacc_init(acc_state *a, const oracle_params *prm) {
  memset(a, 0, sizeof *a);
  a->H = prm->history_len ? prm->history_len : 16;
  a->cap = prm->entry_cap;
  a->table = 1ULL << a->H;
  a->n_opcodes = prm->n_opcodes;
  if (map_init(&a->rd, 1024) || map_init(&a->wr, 1024) || map_init(&a->sites, 64) || map_init(&a->tal, 1024) ||
      map_init(&a->wmap, 64))
    return -1;
  a->opc = (uint64_t *)calloc(prm->n_opcodes ? prm->n_opcodes : 1, 8);
  a->taken_tab = (uint64_t *)calloc(a->table, 8);
  a->total_tab = (uint64_t *)calloc(a->table, 8);
  a->current = -1;     /* index into tl; -1 = None */
  a->open_group = 0;   /* checker.open_group (metrics.py:149) */
  return (a->opc && a->taken_tab && a->total_tab) ? 0 : -1;
}

void oacc_free(acc_state *a) {
  map_free(&a->rd); map_free(&a->wr); map_free(&a->sites); map_free(&a->tal); map_free(&a->wmap);
  free(a->itb.v); free(a->ipt.v); free(a->site_ids.v); free(a->wvals.v); free(a->wcnts.v); free(a->wfirst.v);
  free(a->srec); free(a->tl); free(a->opc); free(a->taken_tab); free(a->total_tab);
  memset(a, 0, sizeof *a);
}

/* consume()'s loop (metrics.py:125-180) over events [lo, hi); returns 0, or
 * 1 = TraceTooLarge, 2 = malformed columnar input */
int oacc_feed(acc_state *a, const uint8_t *kind, const uint64_t *payload, uint64_t lo, uint64_t hi) {
  const uint32_t H = a->H;
  const uint64_t cap = a->cap, table = a->table;
  tally *tl = a->tl;
  int64_t current = a->current;
  uint64_t open_group = a->open_group;
  int status = 0;
  for (uint64_t i = lo; i < hi && status == 0; i++) {
    const uint8_t k = kind[i];
    const uint64_t p = payload[i];
    switch (k) {
      case K_INSTR: { /* metrics.py:131-136 */
        if (current < 0) { status = 2; break; }
        tl[current].segment++; tl[current].total++;
        a->total_instr++;
        uint32_t op = (uint32_t)(p >> 32), w = (uint32_t)p;
        if (op < a->n_opcodes) a->opc[op]++; else { status = 2; break; }
        int fresh; uint64_t s = map_slot(&a->wmap, w, &fresh);
        if (fresh) { a->wmap.vals[s] = a->wvals.n; vec_push(&a->wvals, w); vec_push(&a->wcnts, 0); vec_push(&a->wfirst, i); }
        a->wcnts.v[a->wmap.vals[s]]++;
        break;
      }
      case K_LOAD: case K_ATOMIC_LOAD: case K_STORE: case K_ATOMIC_STORE: { /* metrics.py:137-144 */
        map64 *h = (k & 0x02) ? &a->rd : &a->wr;
        int fresh; uint64_t s = map_slot(h, p, &fresh);
        if (fresh) {
          a->entries++;
          if (cap && a->entries > cap) { status = 1; a->entries_at_fail = a->entries; break; }
        }
        h->vals[s]++;
        break;
      }
      case K_BRANCH: { /* metrics.py:145-155; histories per (site, group) stream */
        uint64_t site = p >> 1, bit = p & 1;
        int fresh; uint64_t s = map_slot(&a->sites, site, &fresh);
        if (fresh) {
          if (a->n_srec == a->cap_srec) {
            a->cap_srec = a->cap_srec ? a->cap_srec * 2 : 64;
            a->srec = (site_rec *)realloc(a->srec, a->cap_srec * sizeof *a->srec);
          }
          a->sites.vals[s] = a->n_srec;
          site_rec *nr = &a->srec[a->n_srec];
          nr->executions = 0; nr->len = 0; nr->hist = 0; nr->last_group = open_group;
          a->n_srec++;
          vec_push(&a->site_ids, site);
        }
        site_rec *sr = &a->srec[a->sites.vals[s]];
        if (!fresh && sr->last_group != open_group) { /* streams[-1][0] != group -> new stream */
          a->excluded += sr->len < H ? sr->len : H;
          sr->len = 0; sr->hist = 0; sr->last_group = open_group;
        }
        /* branch_entropy (entropy.py:102-117): execution t >= H of a stream is an
         * observation keyed by the previous H outcomes, oldest as MSB */
        if (sr->len >= H) { a->total_tab[sr->hist]++; a->taken_tab[sr->hist] += bit; }
        sr->hist = (uint32_t)(((sr->hist << 1) | bit) & (table - 1));
        sr->len++;
        sr->executions++;
        a->entries++;
        if (cap && a->entries > cap) { status = 1; a->entries_at_fail = a->entries; }
        break;
      }
      case K_BARRIER: /* metrics.py:156-161: always sampled, even 0 */
        if (current < 0) { status = 2; break; }
        a->barriers++;
        vec_push(&a->itb, tl[current].segment);
        tl[current].segment = 0;
        current = -1;
        break;
      case K_WI_BEGIN: { /* metrics.py:162-165: fresh tally keyed by global id */
        a->work_items++;
        if (a->n_tl == a->cap_tl) {
          a->cap_tl = a->cap_tl ? a->cap_tl * 2 : 1024;
          a->tl = (tally *)realloc(a->tl, a->cap_tl * sizeof *a->tl);
          tl = a->tl;
        }
        tl[a->n_tl].segment = 0; tl[a->n_tl].total = 0;
        int fresh; uint64_t s = map_slot(&a->tal, (open_group << 32) | (uint32_t)p, &fresh);
        a->tal.vals[s] = a->n_tl;
        current = (int64_t)a->n_tl++;
        break;
      }
      case K_WI_RESUME: { /* metrics.py:166-168 */
        uint64_t s;
        if (!map_find(&a->tal, (open_group << 32) | (uint32_t)p, &s)) { status = 2; break; }
        current = (int64_t)a->tal.vals[s];
        break;
      }
      case K_WI_END: /* metrics.py:169-174: trailing segment only when non-empty */
        if (current < 0) { status = 2; break; }
        if (tl[current].segment > 0) vec_push(&a->itb, tl[current].segment);
        vec_push(&a->ipt, tl[current].total);
        current = -1;
        break;
      case K_WG_BEGIN: open_group = p; break;
      case K_WG_END: case K_KERNEL_BEGIN: case K_KERNEL_END: break;
      default: status = 2; break;
    }
  }
  a->current = current;
  a->open_group = open_group;
  return status;
}

/* the streams still open at the end are whole: their first H executions are warm-up */
void oacc_close_streams(acc_state *a) {
  for (uint64_t s = 0; s < a->n_srec; s++) a->excluded += a->srec[s].len < a->H ? a->srec[s].len : a->H;
}

int oracle_run(const uint8_t *kind, const uint64_t *payload, uint64_t n,
               const oracle_params *prm, oracle_result *r) {
  memset(r, 0, sizeof *r);
  acc_state A;
  if (oacc_init(&A, prm)) return -1;
  const uint64_t table = A.table;
  int status = oacc_feed(&A, kind, payload, 0, n);
  r->entries_at_fail = A.entries_at_fail;
  oacc_close_streams(&A);
  /* finalize's view of the accumulator */
  vec64 itb = A.itb, ipt = A.ipt, wvals = A.wvals, wcnts = A.wcnts;
  map64 rd = A.rd, wr = A.wr;
  site_rec *srec = A.srec;
  const uint64_t n_srec = A.n_srec;
  uint64_t *opc = A.opc, *taken_tab = A.taken_tab, *total_tab = A.total_tab;
  const uint64_t total_instr = A.total_instr, work_items = A.work_items, barriers = A.barriers;
  uint64_t excluded = A.excluded;
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
    w->width_first = A.wfirst.v; A.wfirst.v = NULL;
    w->n_sites = n_srec;
    w->site_ids = A.site_ids.v; A.site_ids.v = NULL;
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
  /* ownership of what was handed to r went with it; the rest is freed */
  A.itb = itb; A.ipt = ipt; A.wvals = wvals; A.wcnts = wcnts;
  A.opc = opc; A.taken_tab = taken_tab; A.total_tab = total_tab;
  oacc_free(&A);
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
