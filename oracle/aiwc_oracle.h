/* aiwc_oracle.h -- TEST INFRASTRUCTURE ONLY (see aiwc_oracle.c). */
#ifndef AIWC_ORACLE_H
#define AIWC_ORACLE_H
#include <stdint.h>

typedef struct {
  uint32_t n_opcodes;    /* opcode dictionary size */
  uint32_t history_len;  /* branch history bits, 0 -> 16 (entropy.py:16) */
  uint64_t entry_cap;    /* TraceTooLarge cap (metrics.py:54-57); 0 = unlimited */
  uint32_t keep_raw;     /* 1: also return the accumulator tables (oracle_raw) */
  uint32_t pad;
} oracle_params;

/* The accumulator behind a result (metrics.py:71-95), for shard tests. */
typedef struct {
  uint64_t n_itb, n_ipt, n_opc, n_sites, table_size, n_rd, n_wr;
  uint64_t *itb, *ipt, *opc, *width_first;  /* width_first parallels width_vals   */
  uint64_t *site_ids, *site_exec;
  uint64_t *taken_tab, *total_tab;
  uint64_t *rd_addr, *rd_cnt, *wr_addr, *wr_cnt;
} oracle_raw;

typedef struct {
  uint64_t n, min, max, sum, mid_lo, mid_hi; /* mid_lo/hi: ranks (n-1)/2 and n/2 */
} oracle_dist;

typedef struct {
  int status;               /* 0 ok, 1 TraceTooLarge, 2 malformed columnar input */
  uint64_t entries_at_fail;
  uint64_t total_instructions, work_items, barriers, opcode_cov;
  oracle_dist itb, ipt;
  uint64_t n_widths;        /* width Counter in insertion order */
  uint64_t *width_vals, *width_counts;
  uint64_t footprint, footprint90, unique_reads, unique_writes, total_reads, total_writes;
  double gmae, lmae[10];
  uint64_t n_sites, branch90, executions, excluded, observations;
  double yokota, linear;
  oracle_raw raw;
} oracle_result;

int oracle_run(const uint8_t *kind, const uint64_t *payload, uint64_t n,
               const oracle_params *p, oracle_result *r);
void oracle_free(oracle_result *r);
/* the same on `threads` host threads (work-group shards + owner merge; aiwc_oracle_mt.c).
 * Uncapped only (entry_cap = 0, keep_raw = 0), else status 3. */
int oracle_run_mt(const uint8_t *kind, const uint64_t *payload, uint64_t n,
                  const oracle_params *p, uint32_t threads, oracle_result *r);
#endif
