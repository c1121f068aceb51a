// aiwc_internal.cuh -- shared definitions of the sm_100a AIWC engine.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/aiwc_b200.h"

namespace aiwc {

// ---- ingest geometry -------------------------------------------------------
constexpr int TPB = 256;              // threads per ingest CTA
constexpr int EPT = 16;               // events per thread per tile (one 16 B kind row)
constexpr int TILE = TPB * EPT;       // 4096 events per tile
constexpr int STAGES = 2;             // TMA ring depth (two CTAs per SM -> four tiles in flight)
constexpr int P1_SUB = 8;             // pass-1 sub-ranges per ingest range (= warp ranges per ingest CTA)
constexpr int WARP_TILE = 32 * EPT;   // events per ingest warp tile (512)
constexpr int CTAS_PER_SM = 2;        // ingest CTAs per SM (non-staging variant)
constexpr int OBINS = 16;             // lane-private opcode bins (ids 0..15)
constexpr int WBINS = 16;             // lane-private width bins (widths 1..16)
constexpr int HBINS = 1024;           // ITB / IPT value histogram bins (values 0..1023)
constexpr int CBINS = 1024;           // count-of-counts bins (counts 1..1023)
constexpr int NLEVELS = 11;           // address entropy at LSB-skip 0..10
constexpr uint32_t WIDTH_TABLE = 65536;
constexpr int MAX_SMALL_LIST = 256;   // widths / sites returned inline in DevState
constexpr uint64_t IPT_END_FLAG = 1ull << 63;
// dense-table entries: u32 = access count (bits 0..29) | read seen (bit 30) | write seen (bit 31)
// when the trace has fewer than 2^30 accesses, else u64 = reads | writes << 32
constexpr uint32_t E32_COUNT = 0x3FFFFFFFu, E32_READ = 1u << 30, E32_WRITE = 1u << 31;
constexpr uint64_t E32_MAX_ACCESSES = 1ull << 30;
// dense-table keys travel as 31-bit list entries in the ingest; key n_keys is the
// sentinel slot that addresses outside the declared statistics are counted into
constexpr uint64_t DENSE_MAX_KEYS = (1ull << 31) - 1;
// table entries allocated for n_keys keys: + the sentinel slot, rounded up to whole
// 1024-key chunks (the exchange unit of the multi-GPU dense path)
__host__ __device__ constexpr uint64_t dense_alloc_keys(uint64_t n_keys) { return (n_keys + 1 + 1023) & ~1023ull; }

// Multi-GPU dense exchange (aiwc_exchange.cu): all_bits holds every rank's bitmap of
// touched 1024-key chunks ([nranks][words]).  A chunk touched by exactly one rank is
// owned by it; any other chunk by a hash of its index.
__device__ __forceinline__ uint32_t chunk_owner(const uint32_t* all_bits, uint64_t words, uint64_t c,
                                                uint32_t nranks) {
  const uint64_t w = c >> 5;
  const uint32_t b = 1u << (c & 31);
  uint32_t cnt = 0, who = 0;
  for (uint32_t r = 0; r < nranks; ++r)
    if (all_bits[(uint64_t)r * words + w] & b) { ++cnt; who = r; }
  if (cnt == 1) return who;
  uint32_t h = (uint32_t)c * 0x9E3779B1u ^ (uint32_t)(c >> 32);
  h ^= h >> 15; h *= 0x85EBCA77u; h ^= h >> 13;
  return h % nranks;
}
// owned by `rank` and touched by some rank (the chunks rank's statistics sweep)
__device__ __forceinline__ bool chunk_is_owned(const uint32_t* all_bits, uint64_t words, uint64_t c, uint32_t rank,
                                               uint32_t nranks) {
  uint32_t any = 0;
  for (uint32_t r = 0; r < nranks; ++r) any |= all_bits[(uint64_t)r * words + (c >> 5)];
  return ((any >> (c & 31)) & 1u) && chunk_owner(all_bits, words, c, nranks) == rank;
}

// ---- kind-byte classes (include/aiwc_b200.h) -------------------------------
__host__ __device__ constexpr bool is_instr(uint32_t k) { return k & 0x01; }
__host__ __device__ constexpr bool is_mem(uint32_t k) { return k & 0x06; }

// error flags raised by kernels (DevState::flags)
enum : uint64_t {
  F_BAD_OPCODE = 1, F_BAD_WIDTH = 2, F_BAD_SITE = 4, F_ADDR_HINT = 8, F_BAD_GROUP = 16,
  F_SLOT_RANGE = 32, F_BAD_KIND = 64,
  F_STREAM = 128  // a StreamChecker invariant is violated (in-pass check; aiwc_validate locates it)
};

// Per-range summary computed from kind bytes alone (pass 1): what the ingest
// carry-in and the host's buffer sizing need.  Work-items and barriers are
// counted by the ingest itself.
struct RangeSum {
  uint32_t n_instr, n_rd, n_wr, n_br, n_wgb, instr_after;
  uint32_t any_bres, pad;       // a barrier or resume occurs (work-item lifetime slots needed)
  int64_t last_bnd, last_wgb;   // global event index, -1 when absent
  int64_t last_wge;             // last wg_end, -1 when absent (in-pass stream checks)
};

// Device-resident accumulator scalars and small tables. The prefix up to
// `host_end` is what finalize copies back in one transfer.
struct DevState {
  // counters
  unsigned long long itb_sum, ipt_sum, ipt_tab_n, ipt_tab_sum;
  unsigned long long itb_ovf_n, ipt_ovf_n, lvl0_ovf_n;
  unsigned long long unique_r, unique_w, footprint;
  unsigned long long flags, max_site, max_width;
  unsigned long long addr_min, addr_max, addr_and, addr_or;
  unsigned long long p1_tot[6];                    // pass-1 totals: instr, rd, wr, br, wgb, ranges with bres
  unsigned long long n_obs, n_sites, n_uniq;      // branch observations, #sites, #unique keys (sparse)
  unsigned long long n_wib, n_bar;                 // work-items begun, barriers hit (ingest)
  unsigned long long dup_set;                      // in-pass stream check: set bits of the begin map
  unsigned long long state_runs_n;                 // state export: runs claimed (kept when <= capacity)
  unsigned long long bw_overflow;                  // branch walk: more sites than its table (sort path instead)
  unsigned long long n_widths_listed, n_sites_listed;
  double entropy[NLEVELS];
  double yokota, linear;
  unsigned long long itb_hist[HBINS];
  unsigned long long ipt_hist[HBINS];
  unsigned long long cnt_hist0[CBINS];              // level-0 count-of-counts (footprint_90)
  unsigned long long width_list[3 * MAX_SMALL_LIST]; // (value, count, first) first-seen order
  unsigned long long site_list[2 * MAX_SMALL_LIST];  // (site, count) ascending
  unsigned long long opc_small[MAX_SMALL_LIST];      // opcode counts when the dictionary has <= 256 ids
  // ---- not copied back ----
  unsigned long long host_end;
  unsigned long long cnt_hist[NLEVELS][CBINS];      // count-of-counts per level (entropy)
  unsigned long long hot_key;                       // hot_sample_kernel: first key of the hot window, ~0 none
  unsigned long long bin_zones, bin_total;          // random key zones (bit z: zone z is binned), entries binned
  unsigned int zone_counts[128];                    // zone sampler: (near, far) per zone
  unsigned long long width_unit[WBINS];             // first presence unit of widths 1..16 (launch_width_first)
};

// Memory-path description shared by the ingest and the dense-table kernels.
struct AddrMap {
  uint64_t base;       // min address rounded down to 1024
  uint64_t hi;         // max address
  uint64_t low_mask;   // (1 << k) - 1
  uint64_t low_const;  // (addr - base) & low_mask for every address
  uint32_t k;          // constant low bits dropped from keys
  uint64_t n_keys;     // dense table length
  uint64_t off_max;    // largest valid addr - base: ((n_keys - 1) << k) | low_mask
};

constexpr int ZONES = 64;                   // key zones of the random-access sampler (aiwc_bins.cu)
constexpr uint32_t SMEM_TABLE_KEYS = 1024;  // small dense tables / the hot window live in shared memory per CTA
constexpr uint64_t HOT_MIN_ACCESSES = 1ull << 20;  // traces with fewer accesses skip the hot-window sampler
constexpr int PRES_TILES = 16;         // width presence granularity (tile iterations per mask)

struct IngestArgs {
  const uint8_t* kind;
  const uint64_t* payload;
  uint64_t n;
  uint64_t tma_rows;          // rows of 16 events covered by the tensor maps
  uint32_t tiles_per_cta;
  uint32_t n_opcodes;
  uint32_t local_volume;
  const RangeSum* ranges;
  DevState* st;
  unsigned long long* opc_counts;   // [n_opcodes]
  unsigned long long* width_count;  // [WIDTH_TABLE]
  unsigned long long* width_first;  // [WIDTH_TABLE] (widths > 16; 1..16 found by width_first_kernel)
  uint32_t* width_presence;         // [n_ctas * P1_SUB * pres_blocks]: widths 1..16 present per warp range (bit w - 1)
  uint32_t* itb_ovf;                // [n_bar + n_wie]
  uint32_t* ipt_ovf;                // [n_wie]
  unsigned long long* ipt_tab;      // [n_wgb * local_volume] or null
  uint64_t ipt_tab_len;
  // memory
  AddrMap am;
  void* dense;                      // dense mode: [am.n_keys] u32 (dense32) or u64 entries
  uint32_t dense32;
  uint32_t pres_blocks;
  uint32_t smem_keys;               // > 0: keys [hot_lo, hot_lo + smem_keys) of the dense table are
                                    // accumulated per CTA in shared memory (read / write u32 counters)
                                    // and added to the table once at the end
  uint64_t hot_lo;                  // window base when hot_dev is null (small tables: 0)
  const unsigned long long* hot_dev;  // device-chosen window base (hot_sample_kernel), ~0 = no window
  uint64_t* rd_out;                 // compact mode
  uint64_t* wr_out;
  uint64_t* br_out;                 // branch records site << 32 | gkey << 1 | taken
  uint32_t* chunk_bits;             // shard dense exchange: bit c = this rank touched keys [1024 c, 1024 c + 1024)
  // key-block bins (aiwc_bins.cu): accesses into random zones are appended, not REDed
  uint32_t* bin_seg;                // [accesses]: warp range w appends at bin_base[w]
  unsigned long long* bin_base;     // [warp ranges]: accesses before the range (written by the ingest)
  uint32_t* bin_fill;               // [warp ranges]: entries the range appended
  const unsigned long long* bin_zones;  // device zone mask (null / 0: no bins)
  uint32_t zone_shift;
  // in-pass StreamChecker (trace.py:289-424) of an untrusted trace without barriers /
  // resumes: sequence rules per lane with carried state, duplicate wi_begin per group
  uint32_t check;
  uint32_t* dup_bits;               // [(groups) * local_volume] bits: wi_begin seen
  uint64_t dup_len;
  // traces with barriers / resumes: three words per (group, lid) slot, updated at
  // each segment close (null otherwise): ~min(pos << 1 | opened by resume),
  // max((pos + 1) << 1 | closed by end), barriers | ends << 32
  unsigned long long* wi_rules;
};

// ---- stream validation (aiwc_validate.cu) ---------------------------------------
struct ValidateState {
  unsigned long long first_ke;   // first kernel_end index (~0: none)
  unsigned long long winner;     // min(index << 32 | range) over flagged ranges (~0: none)
  uint32_t n_struct, n_groups;   // structural events, work-group begins
  uint32_t bad_kind, counts_used;
  uint32_t kb0, dp;              // event 0 is the kernel_begin; the data-parallel checker ran
};
struct ValidateRecord {
  uint64_t index;
  uint32_t code, cls;            // violation code (aiwc_validate.cu), metric kind byte
  uint64_t group_key, local_id;
  uint32_t n_counts, counts_off; // distinct barrier counts (barrier.divergence)
};
struct ValidateBufs {
  uint32_t *tile_s, *tile_g, *scan_scratch;
  uint64_t *spos, *spay, *sgap;
  uint32_t* gstart;
  uint32_t *srange, *first_wge;   // per entry: its range; per range: first wg_end entry
  uint64_t *keys, *keys_tmp;      // (range, local id, entry) sort keys
  uint32_t* sort_hist;
  uint8_t* prevk;
  unsigned long long* unf;
  uint32_t *bmin, *bmax;
  ValidateRecord* recs;           // [0, NG]: replay ranges; NG + 1: data-parallel winner; NG + 2: index-0 event
  uint32_t* counts;
  uint32_t counts_cap;
};
constexpr uint32_t VALIDATE_LV_MAX = 1024;   // larger work-groups are validated on the host
constexpr int VALIDATE_TILE = 4096;
void validate_phase1(const uint8_t* kind, uint64_t n, ValidateState* vs, const ValidateBufs& b, cudaStream_t s,
                     int* kernels);
void validate_phase2(const uint8_t* kind, const uint64_t* payload, uint64_t n, uint32_t lv, ValidateState* vs,
                     const ValidateBufs& b, uint64_t S, uint64_t NG, uint32_t n_ctas, bool force_replay,
                     cudaStream_t s, int* kernels);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
cudaError_t set_smem_attr(const void* kernel, int bytes);
template <typename K>
inline cudaError_t set_smem_once(K kernel, int bytes) {
  return set_smem_attr(reinterpret_cast<const void*>(kernel), bytes);
}

// ---- small device helpers ----------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_incl_max(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, u);
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- host-side launchers (defined in the .cu files) -------------------------
void launch_pass1(const uint8_t* kind, const uint64_t* payload, uint64_t n, uint32_t n_ranges,
                  uint32_t tiles_per_cta, bool with_stats, RangeSum* out, DevState* st, cudaStream_t s,
                  bool light = false);
cudaError_t launch_ingest(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap, uint32_t n_ctas,
                          bool dense, bool stage, cudaStream_t s);  // smem grows by 8 * a.smem_keys
// hot-key window: samples memory events, writes the most frequent 1024-key block of the
// dense table (when it holds >= 1/64 of the sampled accesses) to *hot_out, else ~0
void launch_hot_sample(const uint8_t* kind, const uint64_t* payload, uint64_t n, const AddrMap& am,
                       unsigned long long* hot_out, cudaStream_t s);
void launch_ipt_table(const unsigned long long* tab, uint64_t len, DevState* st, uint32_t* ipt_ovf, cudaStream_t s);
void launch_width_first(const uint8_t* kind, const uint64_t* payload, uint64_t n, const uint32_t* presence,
                        uint32_t n_ranges, uint32_t pres_blocks, uint32_t tiles_per_range, uint32_t wt,
                        unsigned long long* width_first, DevState* st, cudaStream_t s);
void launch_width_list(const unsigned long long* count, const unsigned long long* first, DevState* st,
                       cudaStream_t s);
void launch_dense_stats(const void* tab, bool e32, uint64_t n_keys, uint32_t k, uint64_t total_m, DevState* st,
                        double* partials, uint32_t n_ctas, uint64_t* lvl0_ovf, cudaStream_t s,
                        const uint32_t* own_bits = nullptr, uint64_t own_words = 0, uint32_t rank = 0,
                        uint32_t nranks = 1,   // own_bits: only the chunks `rank` owns
                        bool clear = false);   // zero the table while reading it (not with own_bits)
// key-block bins (aiwc_bins.cu)
void launch_zone_sample(const uint8_t* kind, const uint64_t* payload, uint64_t n, const AddrMap& am,
                        uint32_t zone_shift, unsigned int* zone_counts, unsigned long long* zones_out,
                        cudaStream_t s);
size_t bin_scratch_bytes(uint64_t n_bins, uint32_t n_warps, uint64_t n_blocks);
int bin_finish(const uint32_t* seg, const unsigned long long* seg_base, const uint32_t* fill, uint32_t n_warps,
               uint64_t n_bins, void* table, bool e32, uint64_t n_keys, void* scratch, cudaStream_t s);
// multi-GPU dense exchange (aiwc_exchange.cu); return kernel counts
int launch_pack(const void* tab, bool e32, const uint32_t* all_bits, uint64_t words, uint32_t rank, uint32_t nranks,
                int pass, unsigned long long* cursor, uint64_t* out, uint32_t n_sms, cudaStream_t s);
int launch_apply_runs(void* tab, bool e32, const uint64_t* runs, uint64_t n_runs, uint64_t n_keys,
                      const uint32_t* all_bits, uint64_t words, uint32_t rank, uint32_t nranks,
                      unsigned long long* flags, uint32_t n_sms, cudaStream_t s);
uint64_t launch_pack_all(const void* tab, bool e32, uint64_t n_keys, unsigned long long* cursor, uint64_t* out,
                         int pass, uint32_t n_sms, cudaStream_t s, uint64_t cap = ~0ull);
void launch_merge_apply(const uint64_t* runs, uint64_t n_runs, uint64_t base_p, uint64_t low_p, uint32_t k_p,
                        uint64_t base_m, uint32_t k_m, uint64_t n_keys_m, unsigned long long* tab,
                        unsigned long long* flags, uint32_t n_sms, cudaStream_t s);
int launch_clear_chunks(void* tab, bool e32, uint64_t n_keys, const uint32_t* all_bits, uint64_t words, uint32_t rank,
                        uint32_t nranks, uint32_t* my_bits, uint32_t n_sms, cudaStream_t s);
void launch_entropy_finish(DevState* st, const double* partials, uint32_t n_parts, uint64_t total_m, uint32_t k,
                           cudaStream_t s);
// sparse memory path; returns kernel count
int sparse_memory_stats(const uint64_t* rd, uint64_t n_rd, const uint64_t* wr, uint64_t n_wr, AddrMap am,
                        uint64_t total_m, DevState* st, double* partials, uint32_t n_parts, uint64_t* lvl0_ovf,
                        void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t sparse_scratch_bytes(uint64_t m);
// branch path; returns kernel count
int branch_stats(uint64_t* recs, uint64_t n, uint32_t site_bits, uint32_t history_len, bool walk, DevState* st,
                 unsigned long long* tables, void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t branch_scratch_bytes(uint64_t n);
// phase 1 of the sort-free branch walk (launched before finalize's state read-back;
// sets st->bw_overflow when the sites do not fit its table)
int branch_walk_prepare(const uint64_t* recs, uint64_t n, uint32_t history_len, DevState* st, void* scratch,
                        cudaStream_t s);
size_t branch_site_list_offset(uint64_t n);
// utilities
void radix_sort_u64(uint64_t* keys, uint64_t* tmp, uint64_t n, int bit_lo, int bit_hi, uint32_t* hist_scratch,
                    cudaStream_t s, int* kernels);
size_t radix_hist_bytes(uint64_t n);
uint64_t* radix_sort_u64_any(uint64_t* keys, uint64_t* tmp, uint64_t n, int bit_lo, int bit_hi, uint32_t* hist_scratch,
                             cudaStream_t s, int* kernels);
void sort_u32_list(uint32_t* v, uint64_t n, uint64_t* tmp_a, uint64_t* tmp_b, uint32_t* hist, cudaStream_t s,
                   int* kernels);

}  // namespace aiwc
