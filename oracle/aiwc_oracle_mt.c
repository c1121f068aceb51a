/*
 * aiwc_oracle_mt.c -- TEST INFRASTRUCTURE ONLY (CPU baseline).  The oracle's
 * consume + finalize restatement (aiwc_oracle.c) run on every host core, by
 * the reference's own multi-process recipe: contiguous
 * work-group shards are consumed independently (streams, segments and
 * work-items never cross a group, so the shard accumulators merge exactly:
 * pkg/src/aiwc/metrics.py:235-270), then the merged address histogram is
 * finished by owner threads, each owning the addresses with one value of
 * hash(addr >> 10) so every LSB-skip level <= 10 is whole inside one owner
 * (entropy.py:32-46).  Only bench.py's reference / cpu_baseline leg uses it;
 * tests/test_oracle_mt.py pins it to the single-threaded oracle.
 */
#include <pthread.h>

#include "oracle_util.h"

#define CBINS 1024u

typedef struct {
  /* shard phase */
  const uint8_t *kind;
  const uint64_t *payload;
  uint64_t lo, hi;
  const oracle_params *prm;
  uint32_t T;
  acc_state A;
  int status;
  vec64 bucket_addr[2], bucket_cnt[2]; /* [read/write] entries of every owner, owner-major */
  uint64_t *bucket_off[2];             /* [T + 1] offsets of each owner's run            */
  /* owner phase */
  void *all;                           /* the job array (owner phase reads every shard) */
  uint32_t self;
  uint64_t ur, uw, fp, m_r, m_w;
  ksum lev[11];
  uint64_t hist[CBINS];
  vec64 big;
} mt_job;

static uint32_t owner_of(uint64_t addr, uint32_t T) { return (uint32_t)(mix64(addr >> 10) % T); }

/* per shard: consume, then bucket the address Counters by owner */
static void *shard_main(void *arg) {
  mt_job *j = (mt_job *)arg;
  if (oacc_init(&j->A, j->prm)) { j->status = -1; return NULL; }
  j->status = oacc_feed(&j->A, j->kind, j->payload, j->lo, j->hi);
  if (j->status) return NULL;
  oacc_close_streams(&j->A);
  map64 *hs[2] = {&j->A.rd, &j->A.wr};
  for (int q = 0; q < 2; q++) {
    const map64 *h = hs[q];
    uint64_t *cnt = (uint64_t *)calloc(j->T + 1, 8);
    for (uint64_t i = 0; i < h->cap; i++)
      if (h->used[i]) cnt[owner_of(h->keys[i], j->T) + 1]++;
    for (uint32_t t = 0; t < j->T; t++) cnt[t + 1] += cnt[t];
    uint64_t *cur = (uint64_t *)malloc((j->T + 1) * 8);
    memcpy(cur, cnt, (j->T + 1) * 8);
    vec64 *a = &j->bucket_addr[q], *c = &j->bucket_cnt[q];
    a->n = c->n = a->cap = c->cap = h->size;
    a->v = (uint64_t *)malloc((h->size + 1) * 8);
    c->v = (uint64_t *)malloc((h->size + 1) * 8);
    for (uint64_t i = 0; i < h->cap; i++)
      if (h->used[i]) {
        const uint64_t o = cur[owner_of(h->keys[i], j->T)]++;
        a->v[o] = h->keys[i];
        c->v[o] = h->vals[i];
      }
    free(cur);
    j->bucket_off[q] = cnt;
  }
  /* the maps are no longer needed */
  map_free(&j->A.rd); map_free(&j->A.wr);
  return NULL;
}

static double g_m; /* total accesses M (read-only during the owner phase) */

/* per owner: merge its addresses from every shard and finish them
 * (metrics.py:308-321): unique reads / writes, footprint, the level-n sums of
 * p log2 p over addr >> n, and the count-of-counts for footprint_90 */
static void *owner_main(void *arg) {
  mt_job *me = (mt_job *)arg;
  mt_job *all = (mt_job *)me->all;
  const uint32_t T = me->T, t = me->self;
  map64 rd, wr, mg;
  uint64_t nr = 0, nw = 0;
  for (uint32_t s = 0; s < T; s++) {
    nr += all[s].bucket_off[0][t + 1] - all[s].bucket_off[0][t];
    nw += all[s].bucket_off[1][t + 1] - all[s].bucket_off[1][t];
  }
  map_init(&rd, nr + 1); map_init(&wr, nw + 1); map_init(&mg, nr + nw + 1);
  addr_count *v = (addr_count *)malloc((nr + nw + 1) * sizeof *v);
  uint64_t U = 0;
  for (int q = 0; q < 2; q++)
    for (uint32_t s = 0; s < T; s++) {
      const uint64_t *off = all[s].bucket_off[q];
      for (uint64_t i = off[t]; i < off[t + 1]; i++) {
        const uint64_t a = all[s].bucket_addr[q].v[i], c = all[s].bucket_cnt[q].v[i];
        int fresh;
        map_slot(q ? &wr : &rd, a, &fresh);
        if (q) me->m_w += c; else me->m_r += c;
        uint64_t sl = map_slot(&mg, a, &fresh);
        if (fresh) { mg.vals[sl] = U; v[U].addr = a; v[U].count = 0; U++; }
        v[mg.vals[sl]].count += c;
      }
    }
  me->ur = rd.size; me->uw = wr.size; me->fp = U;
  map_free(&rd); map_free(&wr); map_free(&mg);
  qsort(v, U, sizeof *v, cmp_addr);
  for (int lvl = 0; lvl <= 10; lvl++) {
    uint64_t run = 0;
    for (uint64_t i = 0; i < U; i++) {
      if (i && (v[i].addr >> lvl) != (v[i - 1].addr >> lvl)) {
        const double p = (double)run / g_m;
        kadd(&me->lev[lvl], p * log2(p));
        run = 0;
      }
      run += v[i].count;
    }
    if (U) { const double p = (double)run / g_m; kadd(&me->lev[lvl], p * log2(p)); }
  }
  for (uint64_t i = 0; i < U; i++) {
    if (v[i].count < CBINS) me->hist[v[i].count]++;
    else vec_push(&me->big, v[i].count);
  }
  free(v);
  return NULL;
}

/* coverage_count (entropy.py:49-66) from big counts + a count-of-counts histogram */
static uint64_t coverage_hist(uint64_t *big, uint64_t n_big, const uint64_t *hist, unsigned __int128 total) {
  if (!total) return 0;
  qsort(big, n_big, 8, cmp_u64_desc);
  unsigned __int128 cum = 0;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n_big; i++) {
    cum += big[i]; k++;
    if (cum * 10 >= total * 9) return k;
  }
  for (int64_t c = CBINS - 1; c >= 1; c--) {
    if (!hist[c]) continue;
    const unsigned __int128 need = total * 9 - cum * 10, per = (unsigned __int128)c * 10;
    const unsigned __int128 take = (need + per - 1) / per;
    if (take <= hist[c]) return k + (uint64_t)take;
    cum += (unsigned __int128)hist[c] * c;
    k += hist[c];
  }
  return k;
}

int oracle_run_mt(const uint8_t *kind, const uint64_t *payload, uint64_t n, const oracle_params *prm,
                  uint32_t threads, oracle_result *r) {
  memset(r, 0, sizeof *r);
  if (prm->entry_cap || prm->keep_raw) { r->status = 3; return 0; } /* the baseline runs uncapped */
  uint32_t T = threads ? threads : 1;
  /* shard cuts at work-group begins near k * n / T */
  uint64_t *cut = (uint64_t *)malloc((T + 1) * 8);
  cut[0] = 0;
  for (uint32_t k = 1; k < T; k++) {
    uint64_t c = n * (uint64_t)k / T;
    if (c < cut[k - 1]) c = cut[k - 1];
    while (c < n && kind[c] != K_WG_BEGIN) c++;
    cut[k] = c;
  }
  cut[T] = n;
  mt_job *jobs = (mt_job *)calloc(T, sizeof *jobs);
  pthread_t *th = (pthread_t *)malloc(T * sizeof *th);
  for (uint32_t t = 0; t < T; t++) {
    jobs[t].kind = kind; jobs[t].payload = payload; jobs[t].lo = cut[t]; jobs[t].hi = cut[t + 1];
    jobs[t].prm = prm; jobs[t].T = T; jobs[t].all = jobs; jobs[t].self = t;
    pthread_create(&th[t], NULL, shard_main, &jobs[t]);
  }
  for (uint32_t t = 0; t < T; t++) pthread_join(th[t], NULL);
  int status = 0;
  for (uint32_t t = 0; t < T; t++) if (jobs[t].status) status = jobs[t].status < 0 ? 2 : jobs[t].status;
  r->status = status;
  if (status) goto done;

  /* ---- merge (metrics.py:252-262) ---- */
  {
    const uint64_t table = jobs[0].A.table;
    vec64 itb = {0}, ipt = {0};
    uint64_t *opc = (uint64_t *)calloc(prm->n_opcodes + 1, 8);
    uint64_t *taken = (uint64_t *)calloc(table, 8), *total = (uint64_t *)calloc(table, 8);
    map64 wm, sm;
    map_init(&wm, 64); map_init(&sm, 64);
    vec64 wv = {0}, wc = {0}, wf = {0}, sx = {0};
    for (uint32_t t = 0; t < T; t++) {
      acc_state *A = &jobs[t].A;
      r->total_instructions += A->total_instr; r->work_items += A->work_items; r->barriers += A->barriers;
      r->excluded += A->excluded;
      for (uint64_t i = 0; i < A->itb.n; i++) vec_push(&itb, A->itb.v[i]);
      for (uint64_t i = 0; i < A->ipt.n; i++) vec_push(&ipt, A->ipt.v[i]);
      for (uint32_t o = 0; o < prm->n_opcodes; o++) opc[o] += A->opc[o];
      for (uint64_t i = 0; i < table; i++) { taken[i] += A->taken_tab[i]; total[i] += A->total_tab[i]; }
      for (uint64_t i = 0; i < A->wvals.n; i++) {  /* width Counter: first appearance over the whole trace */
        int fresh; uint64_t s = map_slot(&wm, A->wvals.v[i], &fresh);
        if (fresh) { wm.vals[s] = wv.n; vec_push(&wv, A->wvals.v[i]); vec_push(&wc, 0); vec_push(&wf, A->wfirst.v[i]); }
        wc.v[wm.vals[s]] += A->wcnts.v[i];
        if (A->wfirst.v[i] < wf.v[wm.vals[s]]) wf.v[wm.vals[s]] = A->wfirst.v[i];
      }
      for (uint64_t i = 0; i < A->n_srec; i++) {
        int fresh; uint64_t s = map_slot(&sm, A->site_ids.v[i], &fresh);
        if (fresh) { sm.vals[s] = sx.n; vec_push(&sx, 0); }
        sx.v[sm.vals[s]] += A->srec[i].executions;
      }
    }
    /* opcode coverage */
    {
      uint64_t *oc = (uint64_t *)malloc((prm->n_opcodes + 1) * 8), m = 0;
      for (uint32_t o = 0; o < prm->n_opcodes; o++) if (opc[o]) oc[m++] = opc[o];
      r->opcode_cov = coverage90(oc, m);
      free(oc);
    }
    /* ITB / IPT order statistics */
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
    /* widths ordered by first appearance (Counter insertion order) */
    {
      uint64_t *ord = (uint64_t *)malloc((wv.n + 1) * 8);
      for (uint64_t i = 0; i < wv.n; i++) ord[i] = i;
      for (uint64_t i = 1; i < wv.n; i++) {  /* few widths: insertion sort by first index */
        const uint64_t x = ord[i];
        uint64_t k = i;
        while (k && wf.v[ord[k - 1]] > wf.v[x]) { ord[k] = ord[k - 1]; k--; }
        ord[k] = x;
      }
      r->n_widths = wv.n;
      r->width_vals = (uint64_t *)malloc((wv.n + 1) * 8);
      r->width_counts = (uint64_t *)malloc((wv.n + 1) * 8);
      for (uint64_t i = 0; i < wv.n; i++) { r->width_vals[i] = wv.v[ord[i]]; r->width_counts[i] = wc.v[ord[i]]; }
      free(ord);
    }
    /* branches */
    r->n_sites = sx.n;
    for (uint64_t i = 0; i < sx.n; i++) r->executions += sx.v[i];
    r->branch90 = coverage90(sx.v, sx.n);
    {
      uint64_t obs = 0;
      for (uint64_t i = 0; i < table; i++) obs += total[i];
      r->observations = obs;
      ksum y = {0, 0}, l = {0, 0};
      for (uint64_t i = 0; i < table && obs; i++) {
        if (!total[i]) continue;
        const double tot = (double)total[i], pp = (double)taken[i] / tot, q = 1.0 - pp;
        const double h = -((pp > 0 ? pp * log2(pp) : 0.0) + (q > 0 ? q * log2(q) : 0.0));
        const double w = tot / (double)obs;
        kadd(&y, w * h);
        kadd(&l, w * (pp < q ? pp : q));
      }
      r->yokota = kval(&y);
      r->linear = kval(&l);
    }
    free(itb.v); free(ipt.v); free(opc); free(taken); free(total);
    map_free(&wm); map_free(&sm); free(wv.v); free(wc.v); free(wf.v); free(sx.v);
  }

  /* ---- memory: owner threads ---- */
  {
    uint64_t M = 0;
    for (uint32_t s = 0; s < T; s++)
      for (int q = 0; q < 2; q++)
        for (uint64_t i = 0; i < jobs[s].bucket_cnt[q].n; i++) M += jobs[s].bucket_cnt[q].v[i];
    g_m = (double)M;
    for (uint32_t t = 0; t < T; t++) pthread_create(&th[t], NULL, owner_main, &jobs[t]);
    for (uint32_t t = 0; t < T; t++) pthread_join(th[t], NULL);
    ksum lev[11];
    memset(lev, 0, sizeof lev);
    uint64_t hist[CBINS];
    memset(hist, 0, sizeof hist);
    vec64 big = {0};
    for (uint32_t t = 0; t < T; t++) {
      r->unique_reads += jobs[t].ur; r->unique_writes += jobs[t].uw; r->footprint += jobs[t].fp;
      r->total_reads += jobs[t].m_r; r->total_writes += jobs[t].m_w;
      for (int l = 0; l <= 10; l++) kadd(&lev[l], kval(&jobs[t].lev[l]));
      for (uint32_t c = 0; c < CBINS; c++) hist[c] += jobs[t].hist[c];
      for (uint64_t i = 0; i < jobs[t].big.n; i++) vec_push(&big, jobs[t].big.v[i]);
    }
    if (r->footprint) {
      r->gmae = -kval(&lev[0]);
      for (int l = 1; l <= 10; l++) r->lmae[l - 1] = -kval(&lev[l]);
      r->footprint90 = coverage_hist(big.v, big.n, hist, (unsigned __int128)M);
    }
    free(big.v);
  }

done:
  for (uint32_t t = 0; t < T; t++) {
    oacc_free(&jobs[t].A);
    for (int q = 0; q < 2; q++) {
      free(jobs[t].bucket_addr[q].v); free(jobs[t].bucket_cnt[q].v); free(jobs[t].bucket_off[q]);
    }
    free(jobs[t].big.v);
  }
  free(jobs); free(th); free(cut);
  return 0;
}
