/*
 * aiwc_b200.h -- C ABI of the B200-native AIWC metric engine.
 *
 * Replaces the reference's metric hot path (pure Python):
 *   aiwc.metrics.consume   pkg/src/aiwc/metrics.py:98-196   -> aiwc_reset + aiwc_ingest
 *   aiwc.metrics.finalize  pkg/src/aiwc/metrics.py:273-386  -> aiwc_finalize
 *   aiwc.entropy.*         pkg/src/aiwc/entropy.py:20-133   (inside aiwc_finalize)
 *   aiwc.errors.InvalidStream / TraceTooLarge / AiwcError    -> AIWC_ERR_* codes + aiwc_last_error
 * The Python mirror (paper_1805_04207_b200.metrics) binds these with ctypes;
 * INTEGRATION.md shows the binding a maintainer of the reference would add.
 *
 * Plain C types only.  Device pointers are CUDA global-memory addresses on the
 * ctx's device; `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  One ctx per trace stream: a ctx is not thread-safe,
 * distinct ctxs are.  The ctx owns all scratch memory; trace buffers passed to
 * aiwc_ingest must stay valid until the work that call queued on `stream` has
 * completed (stream order; aiwc_finalize on the same stream implies it).
 */
#ifndef AIWC_B200_H
#define AIWC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIWC_ABI_VERSION 2

/* ---- columnar trace layout: one kind byte + one payload u64 per event ----
 * bit0 instr, bit1 read, bit2 write, bit3 branch, bit4 work-item boundary,
 * bit5 segment open (with bit4), bit6 work-group, bit7 variant.            */
enum {
  AIWC_K_PAD = 0x00,          /* no event (padding); never produced by encoders */
  AIWC_K_INSTR = 0x01,        /* payload = opcode_id << 32 | width             */
  AIWC_K_LOAD = 0x02,         /* payload = address                             */
  AIWC_K_ATOMIC_LOAD = 0x82,
  AIWC_K_STORE = 0x04,
  AIWC_K_ATOMIC_STORE = 0x84,
  AIWC_K_BRANCH = 0x08,       /* payload = site << 1 | taken, site < 2^32       */
  AIWC_K_WI_END = 0x10,       /* payload = local linear id                     */
  AIWC_K_BARRIER = 0x90,
  AIWC_K_WI_BEGIN = 0x30,     /* payload = local linear id                     */
  AIWC_K_WI_RESUME = 0xB0,    /* payload = local linear id                     */
  AIWC_K_WG_BEGIN = 0x40,     /* payload = group key (< 2^31, injective)       */
  AIWC_K_WG_END = 0xC0,
  AIWC_K_KERNEL_BEGIN = 0x20,
  AIWC_K_KERNEL_END = 0xA0
};

/* ---- return codes (0 = success) ---- */
enum {
  AIWC_OK = 0,
  AIWC_ERR_INVALID_STREAM = 1, /* aiwc.errors.InvalidStream  (errors.py:70-79)  */
  AIWC_ERR_TOO_LARGE = 2,      /* aiwc.errors.TraceTooLarge  (errors.py:82-89)  */
  AIWC_ERR_INCONSISTENT = 3,   /* aiwc.errors.AiwcError      (metrics.py:276-285) */
  AIWC_ERR_UNSUPPORTED = 4,    /* value outside the columnar format's range      */
  AIWC_ERR_ARGUMENT = 5,       /* bad argument / misaligned buffer / wrong state */
  AIWC_ERR_CUDA = 6,           /* CUDA runtime / driver failure                  */
  AIWC_ERR_NCCL = 7
};

typedef struct aiwc_ctx aiwc_ctx;

/* aiwc_opts.flags */
#define AIWC_OPT_NO_CONSERVATION 1u /* skip finalize's conservation checks (caller does them) */
#define AIWC_OPT_TIMING 2u          /* record CUDA events around each phase (aiwc_result.phase_ms) */
#define AIWC_OPT_VALIDATE_REPLAY 8u /* aiwc_validate: always use the per-work-group replay checker (testing) */

/* aiwc_result.phase_ms indices */
enum { AIWC_PH_PASS1 = 0, AIWC_PH_INGEST = 1, AIWC_PH_MEMORY = 2, AIWC_PH_BRANCH = 3, AIWC_PH_INGEST_TOTAL = 4,
       AIWC_PH_FINALIZE_TOTAL = 5, AIWC_N_PHASES = 8 };

typedef struct {
  uint32_t history_len;       /* branch history bits, 1..16; 0 -> 16 (entropy.py:16)   */
  uint32_t flags;             /* AIWC_OPT_*                                            */
  uint64_t entry_cap;         /* TraceTooLarge cap in entries; 0 = unlimited           */
  uint64_t dense_budget_bytes;/* max bytes for the dense address table; 0 = default    */
} aiwc_opts;

/* Per-trace description passed with the columns. */
typedef struct {
  uint64_t n_events;
  uint32_t local_volume;      /* product of the launch's local size                   */
  uint32_t n_opcodes;         /* opcode dictionary size                               */
  uint32_t has_addr_stats;    /* 1 when addr_* below describe every memory address    */
  uint32_t has_counts;        /* 1 when the class totals below are declared           */
  uint64_t addr_min, addr_max, addr_and, addr_or;
  /* Declared class totals (producers that know them: walkers, generators, the
   * device NDRange producer).  With them aiwc_ingest makes every host decision
   * up front and queues pass 1 and the ingest with no device->host round trip;
   * pass 1's totals are checked against them at finalize (AIWC_ERR_ARGUMENT
   * when they differ). */
  uint64_t n_instr, n_reads, n_writes, n_branches, n_groups;
  uint32_t any_barrier_or_resume;
  /* 1: the columns come from an untrusted producer -- check StreamChecker's
   * invariants (trace.py:289-424) inside the pass.  A violation makes
   * aiwc_finalize return AIWC_ERR_INVALID_STREAM (aiwc_validate locates the
   * first one); aiwc_result.stream_checked says the pass certified the stream
   * (barrier / resume traces included: per-work-item order words, +24 B per
   * (group, local id) slot of device scratch).                              */
  uint32_t check_stream;
  /* Event index of this trace's first event in the whole job (a work-group shard
   * of a multi-GPU job: first-appearance order of widths spans the ranks); 0 else. */
  uint64_t first_event;
  /* 1: keep the accumulator's state for aiwc_state_export (a later merge). */
  uint32_t export_state, reserved2;
} aiwc_trace_info;

typedef struct {
  uint64_t n, min, max, sum;  /* sample count, extremes, exact sum                    */
  uint64_t mid_lo, mid_hi;    /* order statistics at ranks (n-1)/2 and n/2            */
} aiwc_dist;

/* Exact integers plus unrounded fp64 entropies; the host finishes reals with
 * the reference's expressions and round12 (metrics.py:287-386).  Array
 * pointers reference ctx-owned host memory valid until the next call on ctx. */
typedef struct {
  uint64_t n_events;
  uint64_t total_instructions, work_items, barriers_hit;
  uint64_t opcode_coverage;                 /* coverage_count(opcodes, 0.9)              */
  aiwc_dist itb, ipt;
  uint64_t total_reads, total_writes, unique_reads, unique_writes;
  uint64_t footprint, footprint_90;
  double gmae, lmae[10];                    /* -sum p log2 p, levels 0 and 1..10         */
  uint64_t branch_executions, branch_observations, branch_excluded;
  uint64_t n_sites, branch_90;
  double yokota, linear;
  uint64_t entries;                         /* unique reads + unique writes + branches  */
  uint32_t n_opcodes;  const uint64_t *opcode_counts;                 /* by opcode id   */
  uint32_t n_widths;   const uint64_t *width_values, *width_counts;   /* first-seen order */
  uint32_t n_site_list; const uint64_t *site_ids, *site_counts;      /* ascending site  */
  uint32_t used_dense_table;                /* memory path taken (diagnostics)          */
  uint32_t kernels_launched;                /* engine kernels launched for this trace   */
  uint64_t d2h_bytes;                       /* device->host bytes read for this trace   */
  double phase_ms[AIWC_N_PHASES];           /* with AIWC_OPT_TIMING: CUDA-event times   */
  uint64_t binned_accesses;                 /* accesses counted through key-block bins  */
  uint32_t stream_checked;                  /* check_stream: the pass certified the stream */
  uint32_t reserved;
} aiwc_result;

typedef struct {
  int32_t code;
  int64_t event_index;        /* InvalidStream: first offending event              */
  char rule[48];              /* InvalidStream rule id (trace.py:278-286)           */
  uint64_t entries, cap;      /* TraceTooLarge                                      */
  char message[256];
} aiwc_error;

int  aiwc_abi_version(void);
int  aiwc_ctx_create(aiwc_ctx **out, int device, const aiwc_opts *opts);
void aiwc_ctx_destroy(aiwc_ctx *ctx);

/* Start a new accumulator (one kernel invocation) in ctx. */
int  aiwc_reset(aiwc_ctx *ctx);

/* consume(): fold one trace resident in device memory (16-byte aligned
 * columns) into the ctx accumulator.  Asynchronous w.r.t. the host except for
 * one small device->host read of the column counts. */
int  aiwc_ingest(aiwc_ctx *ctx, const uint8_t *kind_dev, const uint64_t *payload_dev,
                 const aiwc_trace_info *info, void *stream);

/* Same as aiwc_ingest from HOST columns (pinned or pageable): copies to the
 * ctx's device staging buffers on `stream` first. */
int  aiwc_ingest_host(aiwc_ctx *ctx, const uint8_t *kind_host, const uint64_t *payload_host,
                      const aiwc_trace_info *info, void *stream);

/* finalize(): every metric of the accumulator; synchronizes `stream`. */
int  aiwc_finalize(aiwc_ctx *ctx, aiwc_result *out, void *stream);

/* Details of the last non-zero return on ctx. */
int  aiwc_last_error(const aiwc_ctx *ctx, aiwc_error *err);

/* ---- multi-GPU job mode: NCCL inside the engine -------------
 * Rank 0 makes an id with aiwc_nccl_unique_id (ncclUniqueId, 128 bytes), the
 * caller broadcasts it, and every rank's ctx joins the job's communicator with
 * aiwc_ctx_set_comm.  From then on aiwc_ingest takes this rank's work-group shard
 * (info->first_event = its first event's index in the job) and aiwc_finalize
 * returns the WHOLE job's result, identical on every rank: the address
 * statistics all-gather, the dense chunk exchange (aiwc_shard_* below, NCCL
 * send / recv) and the combine (one all-reduce of a packed u64 buffer, one
 * all-gather of the variable lists) all run in the engine on `stream`.        */
int  aiwc_nccl_unique_id(void *id_out);
int  aiwc_ctx_set_comm(aiwc_ctx *ctx, const void *nccl_unique_id, int rank, int nranks);

/* ---- multi-GPU (work-group shards) ----------------------------
 * A ctx created with AIWC_OPT_SHARD ingests one rank's work-group shard:
 * memory addresses stay compacted on the device and aiwc_finalize fills every
 * non-memory field.  The caller exchanges addresses between ranks (owner of a
 * key = key / keys_per_rank over the global key map) and each owner computes
 * the memory partials of its key range with aiwc_memory_partial. */
#define AIWC_OPT_SHARD 4u

typedef struct {
  const uint64_t *itb_hist, *ipt_hist;          /* 1024 bins each                      */
  uint64_t n_itb_ovf, n_ipt_ovf;
  const uint64_t *itb_ovf, *ipt_ovf;            /* ascending values >= 1024            */
  uint32_t branch_table_size;                   /* 2^history_len                       */
  const uint64_t *branch_table;                 /* total << 32 | taken per pattern     */
  const uint64_t *width_first;                  /* first event index, per aiwc_result width */
  uint64_t addr_stats[4];                       /* min, max, and, or of shard addresses */
  const uint64_t *rd_dev, *wr_dev;              /* compacted addresses (device)        */
} aiwc_shard_tables;

typedef struct {
  uint64_t unique_reads, unique_writes, footprint;
  double level_sum[11];       /* sum of p log2 p over the owned keys, p = c / total_m  */
  const uint64_t *cnt_hist0;  /* 1024 bins: level-0 count-of-counts                    */
  uint64_t n_big;             /* level-0 counts >= 1024                                 */
  const uint64_t *big;        /* their values                                           */
  uint32_t kernels_launched;  /* engine kernels this call queued                        */
} aiwc_memory_part;

/* after aiwc_finalize on a shard ctx */
int  aiwc_shard_tables_get(aiwc_ctx *ctx, aiwc_shard_tables *out);

/* Group this shard's read and write addresses by owner, owner = min(nranks-1,
 * ((addr - base) >> k) / keys_per_rank).  *reads_dev / *writes_dev hold the
 * owner-grouped addresses (valid until the next call on ctx); counts[0..nranks)
 * are read counts per owner, counts[nranks..2*nranks) write counts. */
int  aiwc_partition_addresses(aiwc_ctx *ctx, uint64_t base, uint32_t k, uint64_t keys_per_rank,
                              uint32_t nranks, uint64_t **reads_dev, uint64_t **writes_dev, uint64_t *counts,
                              void *stream);

/* Memory statistics of the owned keys [key_lo, key_lo + n_keys) of the global
 * key map (base, k) from the received addresses (device).  key_lo must be a
 * multiple of 1024.  Dense table or sort path, as in aiwc_finalize. */
int  aiwc_memory_partial(aiwc_ctx *ctx, const uint64_t *reads_dev, uint64_t n_rd, const uint64_t *writes_dev,
                         uint64_t n_wr, uint64_t base, uint32_t k, uint64_t key_lo, uint64_t n_keys,
                         uint64_t total_m, aiwc_memory_part *out, void *stream);

/* Run-length form of this shard's addresses for the owners (pre-aggregation):
 * maximal stretches of consecutive keys with one owner (<= 65536 keys each),
 * two words per run -- global key, length | is_write << 63 -- grouped by owner;
 * counts[0..nranks) are runs per owner.  Valid until the next call on ctx.
 * Streaming shards become a handful of runs; the caller compares the run count
 * with the access count to choose between this and aiwc_partition_addresses. */
int  aiwc_partition_runs(aiwc_ctx *ctx, uint64_t base, uint32_t k, uint64_t keys_per_rank, uint32_t nranks,
                         uint64_t **runs_dev, uint64_t *counts, void *stream);

/* Owner side of the run exchange: memory statistics of the owned keys
 * [key_lo, key_lo + n_keys) (dense table) from the received runs. */
int  aiwc_memory_partial_runs(aiwc_ctx *ctx, const uint64_t *runs_dev, uint64_t n_runs, uint32_t k,
                              uint64_t key_lo, uint64_t n_keys, uint64_t total_m, aiwc_memory_part *out,
                              void *stream);

/* ---- multi-GPU dense exchange (aiwc_exchange.cu) ---------------------
 * The per-rank work is the single-GPU ingest: every rank fills a dense table over
 * the WHOLE job's key map, then only the 1024-key chunks several ranks touched
 * travel, as runs of equal table entries, to one owner each.  On a shard ctx:
 *   1. aiwc_shard_prepare  -- pass 1 of the shard; its address statistics and access count;
 *   2. (caller) combine every rank's aiwc_shard_stats: min / max / and / or / sum,
 *      budget = the smallest dense_budget_bytes;
 *   3. aiwc_shard_ingest   -- ingest with the job's key map; *dense = 1 when the job's
 *      span fits a dense table (every rank decides alike from the same inputs),
 *      else the addresses stay compacted for aiwc_partition_* / aiwc_memory_partial*;
 *   4. aiwc_finalize       -- every non-memory field of the shard;
 *   5. aiwc_shard_chunks   -- device bitmap of the touched chunks (n_words u32);
 *      (caller) all-gather the bitmaps into [nranks][n_words];
 *   6. aiwc_shard_pack     -- runs of the touched chunks other ranks own, grouped by owner
 *      (two u64 per run: key | length << 32, table entry); counts[o] = runs for owner o;
 *      (caller) all-to-all of the runs;
 *   7. aiwc_shard_owned    -- add the received runs, memory statistics of the owned chunks
 *      with the job's access count; clears every chunk this rank wrote.
 * Owner of a chunk: the only rank that touched it, else a hash of its index.       */
typedef struct {
  uint64_t addr_min, addr_max, addr_and, addr_or;  /* no accesses: ~0, 0, ~0, 0         */
  uint64_t n_accesses;                             /* reads + writes                    */
  uint64_t dense_budget_bytes;                     /* dense-table budget of the ctx     */
  uint64_t n_branches;                             /* branch events of the shard        */
} aiwc_shard_stats;

int  aiwc_shard_prepare(aiwc_ctx *ctx, const uint8_t *kind_dev, const uint64_t *payload_dev,
                        const aiwc_trace_info *info, aiwc_shard_stats *local, void *stream);
int  aiwc_shard_ingest(aiwc_ctx *ctx, const aiwc_shard_stats *job, uint32_t *dense, void *stream);
int  aiwc_shard_chunks(aiwc_ctx *ctx, uint32_t **bits_dev, uint64_t *n_words);
int  aiwc_shard_pack(aiwc_ctx *ctx, const uint32_t *all_bits_dev, uint32_t rank, uint32_t nranks,
                     uint64_t **runs_dev, uint64_t *counts, void *stream);
int  aiwc_shard_owned(aiwc_ctx *ctx, const uint64_t *runs_dev, uint64_t n_runs, const uint32_t *all_bits_dev,
                      uint32_t rank, uint32_t nranks, uint64_t total_m, aiwc_memory_part *out, void *stream);

/* ---- accumulator state and state merges (merge_accumulators, metrics.py:235-270) ----
 * With info->export_state, aiwc_finalize keeps the trace's per-key memory state
 * as runs of equal dense-table entries (two u64 per run: key | length << 32,
 * count | read seen << 62 | write seen << 63) over its key map (address =
 * base + (key << k) + low_const), plus the histograms finalize consumed.  A merge
 * adds the parts' histograms on the host and rebuilds the memory statistics of
 * the union from the parts' runs (aiwc_memory_merge): no re-ingest.        */
typedef struct {
  uint32_t exported;                        /* 0: the trace took the sort path (no table) */
  uint32_t branch_table_size;
  uint64_t n_runs;
  const uint64_t *runs_dev;                 /* ctx-owned device memory, valid until the next ingest */
  uint64_t base, low_const;
  uint32_t k, pad;
  uint64_t addr_stats[4];                   /* min, max, and, or of the addresses                   */
  const uint64_t *itb_hist, *ipt_hist;      /* host, 1024 bins each                                 */
  uint64_t n_itb_ovf, n_ipt_ovf;
  const uint64_t *itb_ovf, *ipt_ovf;        /* ascending                                            */
  const uint64_t *branch_table;             /* host: total << 32 | taken per pattern                */
  const uint64_t *width_first;              /* per aiwc_result width: first event index             */
} aiwc_state;

typedef struct {
  const uint64_t *runs_dev;
  uint64_t n_runs, base, low_const;
  uint32_t k, pad;
} aiwc_runs_part;

int  aiwc_state_export(aiwc_ctx *ctx, aiwc_state *out);
/* memory statistics of the union of the parts' runs (counts add, flags OR) over the
 * key map of the merged address statistics (min, max, and, or); AIWC_ERR_UNSUPPORTED
 * when that span does not fit a dense table (the caller re-ingests instead). */
int  aiwc_memory_merge(aiwc_ctx *ctx, const aiwc_runs_part *parts, uint32_t n_parts, const uint64_t stats[4],
                       uint64_t total_m, aiwc_memory_part *out, void *stream);

/* ---- stream validation (StreamChecker, trace.py:289-424) -------------------------
 * First violation of a columnar trace, decoded as ColumnarTrace.iter_events
 * would (group from the last wg_begin, work-item ids from the local linear id).
 * Returns AIWC_OK (valid: out->event_index = -1), AIWC_ERR_INVALID_STREAM
 * (out filled, also readable through aiwc_last_error), or AIWC_ERR_UNSUPPORTED
 * (a kind byte outside the alphabet, or a local volume above 1024, which the
 * device checker's per-work-item tables do not hold).  `detail` is the
 * reference's text; groups outside the launch grid (dictionary keys) print as
 * "key K" -- detail_code / group_key / local_id / counts let a caller that
 * holds the dictionary format them itself. */
enum { AIWC_V_NONE = 0, AIWC_V_KB_NOT_FIRST, AIWC_V_KB_DUP, AIWC_V_AFTER_KE, AIWC_V_KE_OPEN_GROUP,
       AIWC_V_OUTSIDE_SEG, AIWC_V_BAR_OUTSIDE, AIWC_V_WGB_OPEN, AIWC_V_WGE_MISMATCH, AIWC_V_WGE_OPEN_SEG,
       AIWC_V_UNFINISHED, AIWC_V_DIVERGENCE, AIWC_V_WI_OUTSIDE_GROUP, AIWC_V_WI_ID, AIWC_V_OPEN_WHILE_OPEN,
       AIWC_V_WIB_STARTED, AIWC_V_WIR_NOT_BARRIER, AIWC_V_WIE_NO_SEG, AIWC_V_NO_KE, AIWC_V_EMPTY };

typedef struct {
  int64_t event_index;         /* -1: valid stream                                  */
  char rule[48];
  char detail[256];
  uint32_t detail_code;        /* AIWC_V_*                                          */
  uint32_t metric_kind;        /* kind byte of an event outside a segment           */
  uint64_t group_key;          /* never ended / divergence: the group               */
  uint64_t local_id;           /* never ended: the work-item's local linear id      */
  uint32_t n_counts, pad;      /* divergence: distinct barrier counts, ascending    */
  uint64_t counts[64];
} aiwc_violation;

int  aiwc_validate(aiwc_ctx *ctx, const uint8_t *kind_dev, const uint64_t *payload_dev, const aiwc_trace_info *info,
                   const int64_t global_size[3], const int64_t local_size[3], aiwc_violation *out, void *stream);

/* Device-side synthetic trace generators.
 * Writes n events starting at event index `first` of config `cfg` into the
 * device columns; aiwc_synth_size returns the config's total event count and
 * fills info (opcode count, local volume, exact address statistics). */
uint64_t aiwc_synth_size(int cfg, uint64_t work_items, aiwc_trace_info *info);
int  aiwc_synth_fill(int cfg, uint64_t work_items, uint64_t seed, uint8_t *kind_dev,
                     uint64_t *payload_dev, uint64_t first, uint64_t n, void *stream);

/* ---- .aiwck NDRange producer (aiwc.sim.simulate_events, pkg/src/aiwc/sim.py:171-372) ----
 * The reference's in-process trace producer, on the device.  The kernel source
 * is parsed on the host (paper_1805_04207_b200/ir.py, ir.py:300-374) and
 * lowered to records of AIWC_SIM_WORDS int32:
 *   [kind, sem|atomic, width, dst, src0, src1, src2, buffer, target0, target1, opcode id, line]
 * kind: 0 compute, 1 load, 2 store, 3 br, 4 jmp, 5 barrier, 6 ret; an operand
 * word is mode << 30 | index (0 register, 1 constant-pool slot, 2 built-in
 * gid0..lsz2); targets are instruction indices.  aiwc_sim_plan interprets the
 * launch (counts, faults, layout; synchronizes `stream`), aiwc_sim_emit writes
 * the events in exactly the order sim.py yields them (sim.py:244-344). */
#define AIWC_SIM_WORDS 12
#define AIWC_SIM_MAX_WIDTH (1u << 20)   /* widest register value the device path holds  */
#define AIWC_SIM_FORCE_SEQUENTIAL 1u    /* run the whole launch in the sequential schedule  */
#define AIWC_SIM_FORCE_GROUP 2u         /* start in the group schedule (tests)              */

enum {
  AIWC_SIM_OK = 0,
  AIWC_SIM_OUT_OF_BOUNDS = 1,   /* OutOfBoundsAccess(buffer, index, line)      sim.py:305-306 */
  AIWC_SIM_WIDTH = 2,           /* SimulationError: register lanes != width     sim.py:216-221 */
  AIWC_SIM_NONE_LEN = 3,        /* TypeError: register never written (len)      sim.py:211     */
  AIWC_SIM_NONE_INDEX = 4,      /* TypeError: register never written ([0])      sim.py:230     */
  AIWC_SIM_DIVERGENCE = 5,      /* BarrierDivergence                            sim.py:262-275 */
  AIWC_SIM_STEP_LIMIT = 6,      /* StepLimitExceeded                            sim.py:235-238 */
  AIWC_SIM_UNSUPPORTED = 7      /* width above AIWC_SIM_MAX_WIDTH, > 2^32 work-items        */
};

typedef struct aiwc_sim aiwc_sim;

typedef struct {
  const int32_t *code;        /* host: n_instr records                                   */
  const uint64_t *imm;        /* host: constant pool (values mod 2^64)                   */
  const uint64_t *buf_base;   /* host: byte address of each buffer (sim.py:132-141)      */
  const uint64_t *buf_len;    /* host: elements of each buffer                           */
  const uint64_t *mem_dev;    /* device: initial values, buffers concatenated in order   */
  uint32_t n_instr, n_imm, n_regs, max_width, n_buffers, flags;
  uint64_t global_size[3], local_size[3];
  uint64_t step_limit;        /* sim.py DEFAULT_STEP_LIMIT = 10^8                        */
} aiwc_sim_launch;

typedef struct {
  uint64_t n_events;          /* columns aiwc_sim_emit writes                            */
  uint64_t prefix_events;     /* fault: events sim.py yields before raising (step limit:
                                 UINT64_MAX, find the (limit+1)-th instruction event)    */
  uint64_t n_instr, n_reads, n_writes, n_branches, n_groups, n_barriers;
  int32_t error;              /* AIWC_SIM_*                                              */
  int32_t line;               /* faulting line; divergence: culprit's last branch (-1)   */
  uint64_t wi, wi2;           /* fault / divergence culprit, waiting work-item (stream order) */
  int64_t index;              /* out-of-bounds index                                     */
  uint32_t buffer, reg, lanes, width;
  uint32_t sequential;        /* schedule used: 0 speculative per work-item, 2 per work-group
                                 (a work-item read another's store), 1 whole launch sequential */
  uint32_t n_round;           /* divergence: the barrier round                           */
} aiwc_sim_result;

aiwc_sim   *aiwc_sim_create(void);
void        aiwc_sim_destroy(aiwc_sim *sim);
const char *aiwc_sim_last_error(const aiwc_sim *sim);
int  aiwc_sim_plan(aiwc_sim *sim, const aiwc_sim_launch *launch, aiwc_sim_result *out, void *stream);
int  aiwc_sim_emit(aiwc_sim *sim, uint8_t *kind_dev, uint64_t *payload_dev, uint64_t n_events, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AIWC_B200_H */
