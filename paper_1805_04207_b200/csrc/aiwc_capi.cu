// aiwc_capi.cu -- the C ABI (include/aiwc_b200.h): context, buffers, the
// ingest / finalize orchestration and the exact-integer host finishing
// (coverage counts, order statistics) of pkg/src/aiwc/metrics.py:273-386.
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "aiwc_util.cuh"

using namespace aiwc;

namespace {

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

cudaError_t grow(Buf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  bytes = std::max<size_t>(bytes, 256);
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e == cudaSuccess) b.cap = bytes;
  return e;
}

template <typename T>
T* P(Buf& b) { return reinterpret_cast<T*>(b.p); }

int bitwidth64(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

__global__ void init_state_kernel(DevState* st) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(st);
  const size_t n = sizeof(DevState) / 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) w[i] = 0;
}
// one launch for every per-trace reset: DevState (with the min / and sentinels),
// the width count / first-index tables and the per-range width presence masks
__global__ void init_trace_kernel(DevState* st, unsigned long long* wcount, unsigned long long* wfirst,
                                  uint32_t* wpres, uint32_t n_ranges) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(st);
  const size_t n = sizeof(DevState) / 8;
  const size_t i_min = offsetof(DevState, addr_min) / 8, i_and = offsetof(DevState, addr_and) / 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    w[i] = (i == i_min || i == i_and) ? ~0ull : 0ull;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < WIDTH_TABLE; i += stride) {
    wcount[i] = 0;
    wfirst[i] = ~0ull;
  }
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ranges; i += stride) wpres[i] = 0;
}

__global__ void widen_u32_kernel(const uint32_t* src, uint64_t n, uint64_t* dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

// ---- region compaction: clustered address spans keep the dense path ----
// The memory statistics only depend on the multiset of accesses per address
// group addr >> n (n <= 10), i.e. inside 1024-byte blocks.  Remapping every
// occupied 1 MB region (addr >> 20) to consecutive 1 MB slots, low 20 bits
// kept, preserves every group, count and entropy exactly; a trace whose
// accesses sit in a few far-apart buffers then spans a few MB instead of the
// distance between its buffers.
constexpr uint32_t REG_SHIFT = 20, REG_SLOTS = 16384, REG_MAX = 4096;
constexpr uint64_t REG_EMPTY = ~0ull, REG_BASE = 1ull << 20;

__device__ __forceinline__ uint32_t reg_hash(uint64_t r) {
  return (uint32_t)((r * 0x9E3779B97F4A7C15ull) >> (64 - 14));  // REG_SLOTS = 2^14
}

// distinct regions of the memory events: misc[0] = count, misc[1] = overflow
__global__ void region_mark_kernel(const uint8_t* __restrict__ kind, const uint64_t* __restrict__ payload, uint64_t n,
                                   unsigned long long* keys, uint32_t* misc) {
  uint64_t last = REG_EMPTY;
  uint32_t since_poll = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    // once the table overflowed the answer is known (the sort path): stop early
    if (++since_poll == 64) {
      since_poll = 0;
      if (*(volatile uint32_t*)&misc[1]) return;
    }
    if (!is_mem(kind[i])) continue;
    const uint64_t r = payload[i] >> REG_SHIFT;
    if (r == last) continue;
    last = r;
    uint32_t h = reg_hash(r);
    for (uint32_t probe = 0;; ++probe, h = (h + 1) & (REG_SLOTS - 1)) {
      if (probe == 64) { atomicOr(&misc[1], 1u); return; }
      // a plain load first: the region is usually present already (no CAS serialisation)
      const unsigned long long cur = *(volatile unsigned long long*)&keys[h];
      if (cur == r) break;
      if (cur != REG_EMPTY) continue;
      const unsigned long long old = atomicCAS(&keys[h], REG_EMPTY, (unsigned long long)r);
      if (old == REG_EMPTY) {
        if (atomicAdd(&misc[0], 1u) >= REG_MAX) { atomicOr(&misc[1], 1u); return; }
        break;
      }
      if (old == r) break;
    }
  }
}

// remapped payload column (memory events only change) + its address statistics
__global__ void region_remap_kernel(const uint8_t* __restrict__ kind, const uint64_t* __restrict__ payload, uint64_t n,
                                    const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                                    uint64_t* __restrict__ out, unsigned long long* stats) {
  unsigned long long mn = ~0ull, mx = 0, an = ~0ull, o = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = payload[i];
    if (is_mem(kind[i])) {
      const uint64_t r = p >> REG_SHIFT;
      uint32_t h = reg_hash(r);
      while (keys[h] != r) h = (h + 1) & (REG_SLOTS - 1);  // every region was inserted
      p = REG_BASE + ((uint64_t)vals[h] << REG_SHIFT) + (p & ((1ull << REG_SHIFT) - 1));
      mn = min(mn, (unsigned long long)p); mx = max(mx, (unsigned long long)p); an &= p; o |= p;
    }
    out[i] = p;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    an &= __shfl_xor_sync(0xffffffffu, an, d);
    o |= __shfl_xor_sync(0xffffffffu, o, d);
  }
  if ((threadIdx.x & 31) == 0 && mn <= mx) {
    atomicMin(&stats[0], mn); atomicMax(&stats[1], mx); atomicAnd(&stats[2], an); atomicOr(&stats[3], o);
  }
}

// set bits of the duplicate-begin bitmap (in-pass stream check): fewer than the
// wi_begin events means some work-item began twice in one group
__global__ void popcount_kernel(const uint32_t* __restrict__ bits, uint64_t words, unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
    c += __popc(bits[i]);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// the per-work-item rules of traces with barriers / resumes (trace.py:355-404), one
// warp per group: every work-item that closed a segment opened its first one with
// wi_begin, closed its last with wi_end, ended once, and all hit the same number of
// barriers (three words per slot, written at each close by the ingest)
__global__ void wi_rules_kernel(const unsigned long long* __restrict__ rules, uint64_t n_groups, uint32_t lv,
                                DevState* st) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  bool bad = false;
  for (uint64_t g = w0; g < n_groups; g += nw) {
    uint32_t bmin = ~0u, bmax = 0;
    for (uint32_t i = lane; i < lv; i += 32) {
      const unsigned long long* w = rules + 3 * (g * lv + i);
      const unsigned long long first = w[0];
      if (first == 0) continue;  // no segment of this work-item in this group
      const unsigned long long last = w[1], k = w[2];
      bad |= (~first & 1ull) || !(last & 1ull) || (k >> 32) != 1ull;
      bmin = min(bmin, (uint32_t)k);
      bmax = max(bmax, (uint32_t)k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
      bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    }
    bad |= bmin != ~0u && bmin != bmax;  // barrier.divergence
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_STREAM);
}

struct aiwc_ctx {
  int device = 0;
  int n_sms = 148;
  aiwc_opts opts{};
  aiwc_error err{};
  int state = 0;  // 0 empty, 1 ingested, 2 finalized
  Buf reg_keys, reg_vals, reg_misc, remap_pay;  // region compaction of clustered address spans
  Buf dev_state, ranges, opc, wcount, wfirst, wpres, itb_ovf, ipt_ovf, ipt_tab, dtab, rd, wr, br, partials, lvl0_ovf,
      sparse_scr, branch_scr, branch_tab, kind_stage, pay_stage, sort_a, sort_b, sort_h;
  DevState* h_state = nullptr;  // pinned
  // per trace
  aiwc_trace_info info{};
  uint64_t n_instr = 0, n_rd = 0, n_wr = 0, n_br = 0, n_wgb = 0, n_bres = 0;
  uint64_t n_events_seen = 0;
  AddrMap am{};
  bool dense = false;
  bool dense32 = false;     // u32 count|flags entries (fewer than 2^30 accesses)
  bool hot_off = false;     // AIWC_HOT_WINDOW=0 disables the shared-memory hot-key window (measurement)
  bool region_off = false;  // AIWC_REGIONS=0 disables region compaction of wide address spans (measurement)
  // key-block bins of random accesses: measured to cost more than the REDs they replace with the
  // current two-pass partition (C3: ingest -1.35 ms, bin processing +6.2 ms), so opt-in:
  // AIWC_BINS=1 enables them for eligible traces, AIWC_BINS=2 for every dense trace (tests)
  bool bins_off = true;
  bool bins_force = false;
  bool bins = false;        // this trace: the zone sampler ran, the ingest may bin
  uint64_t binned = 0;      // this trace: accesses counted through the bins
  bool stream_checked = false;  // this trace: the ingest checked StreamChecker's invariants
  Buf dup_bits, wi_rules;
  uint64_t dup_len = 0;
  bool wi_rules_on = false;
  // exported accumulator state (aiwc_state_export)
  Buf state_runs, state_cur;
  uint64_t state_n_runs = 0;
  bool state_ok = false;
  uint64_t stats4[4] = {};  // address statistics the key map was built from
  uint64_t state_cap = 0;
  Buf bin_seg, bin_base, bin_fill, bin_scr;
  int dense_entry = 0;      // AIWC_DENSE_ENTRY=32|64 forces the entry width (measurement), 0 = rule
  uint64_t ipt_tab_len = 0;
  uint32_t n_ranges = 0, tiles_per_cta = 0;
  uint32_t kernels = 0;
  uint32_t n_parts = 0;
  uint64_t d2h = 0;
  // optional phase timing (AIWC_OPT_TIMING): pairs of events per phase
  cudaEvent_t ev[2 * AIWC_N_PHASES] = {};
  // side stream: the dense table is cleared while pass 1 runs
  cudaStream_t aux = nullptr;
  cudaStream_t aux2 = nullptr;  // hot-key sampler, concurrent with pass 1
  cudaEvent_t p1_ev = nullptr, hot_ev = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  size_t pre_zeroed = 0;
  size_t dtab_clean = 0, dtab_used = 0;  // bytes of the dense table cleared after the last finalize / used now
  bool one_pass = false;  // declared class totals: no round trip between pass 1 and the ingest
  // an ingest between its two halves (ingest_begin -> ingest_finish; the shard path
  // combines the ranks' address statistics in between)
  struct Pending {
    const uint8_t* kind = nullptr;
    const uint64_t* payload = nullptr;
    uint64_t rows = 0;
    CUtensorMap km{}, pm{};
    bool opc_big = false, with_stats = false;
    bool light = false;  // pass 1 ran light (a dense table, no branches predicted from the declaration)
    size_t clean_prev = 0;
    uint32_t G = 0, tpc = 0;
  } pend;
  // multi-GPU dense exchange: 1024-key chunks of the (global) table this rank touched
  Buf chunk_bits, own_list;
  uint64_t n_chunk_words = 0;
  bool shard_dense = false;
  // job mode (aiwc_ctx_set_comm): this ctx ingests one rank's shard and finalize
  // returns the whole job's result; the collectives are NCCL calls on `comm`
  ncclComm_t comm = nullptr;
  uint32_t rank = 0, nranks = 1;
  uint64_t job[7] = {};  // the job's aiwc_shard_stats (combined at ingest)
  Buf nc_bits, nc_small, nc_send, nc_recv, nc_pack, nc_blob;
  std::vector<uint64_t> job_itb_ovf, job_ipt_ovf;
  // last encoded TMA descriptors (re-used while the columns stay the same)
  const void* tm_kind = nullptr;
  const void* tm_payload = nullptr;
  uint64_t tm_rows = 0;
  CUtensorMap tm_k{}, tm_p{};
  bool timing = false;
  uint32_t marked = 0;  // phases whose end event was recorded for the current trace
  void mark(int phase, int end, cudaStream_t s) {
    if (!timing) return;
    cudaEventRecord(ev[2 * phase + end], s);
    if (end) marked |= 1u << phase;
  }
  // host results
  std::vector<uint64_t> opc_counts, width_vals, width_counts, site_ids, site_counts;
  std::vector<uint64_t> itb_ovf_sorted, ipt_ovf_sorted, lvl0_sorted;
  std::vector<uint64_t> width_firsts, branch_tab_host;
  // multi-GPU: owner partition and owned-key memory partials
  Buf part_entries, part_cursor, mp_state, mp_tab, mp_partials, mp_ovf, run_pos, run_blk, run_scan;
  // stream validation
  Buf v_state, v_tiles, v_scan, v_spos, v_spay, v_sgap, v_gstart, v_recs, v_counts;
  Buf v_srange, v_fwge, v_keys, v_keys_tmp, v_hist, v_prevk, v_unf, v_bmm;
  std::vector<uint64_t> mp_hist0, mp_big;
};

static int fail(aiwc_ctx* c, int code, const char* msg) {
  if (c) {
    c->err = aiwc_error{};
    c->err.code = code;
    c->err.event_index = -1;
    snprintf(c->err.message, sizeof c->err.message, "%s", msg);
  }
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      char m_[200];                                                                     \
      snprintf(m_, sizeof m_, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return fail(ctx, AIWC_ERR_CUDA, m_);                                              \
    }                                                                                   \
  } while (0)

extern "C" int aiwc_abi_version(void) { return AIWC_ABI_VERSION; }

extern "C" int aiwc_ctx_create(aiwc_ctx** out, int device, const aiwc_opts* opts) {
  if (!out) return AIWC_ERR_ARGUMENT;
  aiwc_ctx* ctx = new aiwc_ctx();
  ctx->device = device;
  if (opts) ctx->opts = *opts;
  if (ctx->opts.history_len == 0) ctx->opts.history_len = 16;
  if (ctx->opts.history_len > 16) {
    delete ctx;
    return AIWC_ERR_ARGUMENT;
  }
  *out = ctx;
  if (const char* de = getenv("AIWC_DENSE_ENTRY")) ctx->dense_entry = atoi(de);
  if (const char* hw = getenv("AIWC_HOT_WINDOW")) ctx->hot_off = atoi(hw) == 0;
  if (const char* rg = getenv("AIWC_REGIONS")) ctx->region_off = atoi(rg) == 0;
  if (const char* bn = getenv("AIWC_BINS")) { ctx->bins_off = atoi(bn) == 0; ctx->bins_force = atoi(bn) == 2; }
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&ctx->n_sms, cudaDevAttrMultiProcessorCount, device));
  if (ctx->opts.dense_budget_bytes == 0) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    ctx->opts.dense_budget_bytes = std::min<size_t>(fr / 4, 48ull << 30);
  }
  CK(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_state), sizeof(DevState)));
  CK(grow(ctx->dev_state, sizeof(DevState)));
  CK(grow(ctx->wcount, WIDTH_TABLE * 8));
  CK(grow(ctx->wfirst, WIDTH_TABLE * 8));
  ctx->n_parts = (uint32_t)ctx->n_sms * 4;
  CK(grow(ctx->partials, (size_t)NLEVELS * ctx->n_parts * sizeof(double)));
  CK(grow(ctx->branch_tab, (1u << 16) * 8));
  if (ctx->opts.flags & AIWC_OPT_TIMING) {
    ctx->timing = true;
    for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
  }
  CK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->aux2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->p1_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->hot_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  return AIWC_OK;
}

extern "C" void aiwc_ctx_destroy(aiwc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  Buf* bufs[] = {&ctx->dev_state, &ctx->ranges, &ctx->opc, &ctx->wcount, &ctx->wfirst, &ctx->itb_ovf,
                 &ctx->ipt_ovf, &ctx->ipt_tab, &ctx->dtab, &ctx->rd, &ctx->wr, &ctx->br, &ctx->partials,
                 &ctx->lvl0_ovf, &ctx->sparse_scr, &ctx->branch_scr, &ctx->branch_tab, &ctx->kind_stage,
                 &ctx->pay_stage, &ctx->sort_a, &ctx->sort_b, &ctx->sort_h, &ctx->part_entries,
                 &ctx->part_cursor, &ctx->mp_state, &ctx->mp_tab, &ctx->mp_partials, &ctx->mp_ovf, &ctx->wpres,
                 &ctx->run_pos, &ctx->run_blk, &ctx->run_scan, &ctx->reg_keys, &ctx->reg_vals, &ctx->reg_misc,
                 &ctx->remap_pay,
                 &ctx->v_state, &ctx->v_tiles, &ctx->v_scan, &ctx->v_spos, &ctx->v_spay, &ctx->v_sgap,
                 &ctx->v_gstart, &ctx->v_recs, &ctx->v_counts, &ctx->v_srange, &ctx->v_fwge, &ctx->v_keys,
                 &ctx->v_keys_tmp, &ctx->v_hist, &ctx->v_prevk, &ctx->v_unf, &ctx->v_bmm};
  for (Buf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->h_state) cudaFreeHost(ctx->h_state);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->aux2) cudaStreamDestroy(ctx->aux2);
  if (ctx->p1_ev) cudaEventDestroy(ctx->p1_ev);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (Buf* b : {&ctx->chunk_bits, &ctx->own_list, &ctx->nc_bits, &ctx->nc_small, &ctx->nc_send, &ctx->nc_recv,
                 &ctx->nc_pack, &ctx->nc_blob, &ctx->bin_seg, &ctx->bin_base, &ctx->bin_fill, &ctx->bin_scr,
                 &ctx->dup_bits, &ctx->wi_rules, &ctx->state_runs, &ctx->state_cur})
    if (b->p) cudaFree(b->p);
  if (ctx->hot_ev) cudaEventDestroy(ctx->hot_ev);
  delete ctx;
}

extern "C" int aiwc_reset(aiwc_ctx* ctx) {
  if (!ctx) return AIWC_ERR_ARGUMENT;
  if (ctx->remap_pay.p) {  // a region-compacted column is per trace: do not keep ~8 B / event allocated
    cudaSetDevice(ctx->device);
    cudaFree(ctx->remap_pay.p);
    ctx->remap_pay = Buf{};
  }
  ctx->state = 0;
  ctx->err = aiwc_error{};
  return AIWC_OK;
}

extern "C" int aiwc_last_error(const aiwc_ctx* ctx, aiwc_error* e) {
  if (!ctx || !e) return AIWC_ERR_ARGUMENT;
  *e = ctx->err;
  return AIWC_OK;
}

static int encode_maps_uncached(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, uint64_t rows,
                                CUtensorMap* km, CUtensorMap* pm);

static int encode_maps(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, uint64_t rows, CUtensorMap* km,
                       CUtensorMap* pm) {
  if (ctx->tm_kind == kind && ctx->tm_payload == payload && ctx->tm_rows == rows) {
    *km = ctx->tm_k; *pm = ctx->tm_p;
    return AIWC_OK;
  }
  const int rc = encode_maps_uncached(ctx, kind, payload, rows, km, pm);
  if (rc == AIWC_OK) {
    ctx->tm_kind = kind; ctx->tm_payload = payload; ctx->tm_rows = rows;
    ctx->tm_k = *km; ctx->tm_p = *pm;
  } else {
    ctx->tm_kind = ctx->tm_payload = nullptr;
  }
  return rc;
}

static int encode_maps_uncached(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, uint64_t rows,
                                CUtensorMap* km, CUtensorMap* pm) {
  memset(km, 0, sizeof *km);
  memset(pm, 0, sizeof *pm);
  if (rows == 0) return AIWC_OK;
  auto enc = get_encode();
  if (!enc) return fail(ctx, AIWC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {16, rows};
  cuuint32_t box[2] = {16, (cuuint32_t)(WARP_TILE / 16)};  // one ingest warp tile per TMA box
  cuuint32_t estr[2] = {1, 1};
  cuuint64_t kstr[1] = {16};
  CUresult r = enc(km, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(kind), dims, kstr, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, AIWC_ERR_CUDA, "tensor map (kind) encode failed");
  cuuint64_t pstr[1] = {128};
  r = enc(pm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t*>(payload), dims, pstr, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, AIWC_ERR_CUDA, "tensor map (payload) encode failed");
  return AIWC_OK;
}

// Region compaction (see region_mark_kernel): *out = the remapped payload column
// (ctx-owned) and stats[4] its address statistics, or *out = null when the
// accesses touch too many regions (the sparse path then handles the trace).
static int region_compact(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, uint64_t n, cudaStream_t s,
                          const uint64_t** out, unsigned long long* stats) {
  *out = nullptr;
  CK(grow(ctx->reg_keys, REG_SLOTS * 8));
  CK(grow(ctx->reg_vals, REG_SLOTS * 4));
  CK(grow(ctx->reg_misc, 64));
  unsigned long long* keys = P<unsigned long long>(ctx->reg_keys);
  uint32_t* misc = P<uint32_t>(ctx->reg_misc);
  CK(cudaMemsetAsync(keys, 0xFF, REG_SLOTS * 8, s));
  CK(cudaMemsetAsync(misc, 0, 64, s));
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->n_sms * 8);
  region_mark_kernel<<<grid, 256, 0, s>>>(kind, payload, n, keys, misc);
  uint32_t hm[2];
  CK(cudaMemcpyAsync(hm, misc, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  ctx->kernels += 1;
  if (hm[1] || hm[0] == 0 || hm[0] > REG_MAX) return AIWC_OK;
  std::vector<unsigned long long> hk(REG_SLOTS);
  CK(cudaMemcpyAsync(hk.data(), keys, REG_SLOTS * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<unsigned long long> regs;
  for (unsigned long long k : hk)
    if (k != REG_EMPTY) regs.push_back(k);
  std::sort(regs.begin(), regs.end());  // slots in address order
  std::vector<uint32_t> hv(REG_SLOTS, 0);
  for (uint32_t i = 0; i < REG_SLOTS; ++i)
    if (hk[i] != REG_EMPTY) hv[i] = (uint32_t)(std::lower_bound(regs.begin(), regs.end(), hk[i]) - regs.begin());
  CK(cudaMemcpyAsync(ctx->reg_vals.p, hv.data(), REG_SLOTS * 4, cudaMemcpyHostToDevice, s));
  // the remapped span (regions squeezed together) must then fit the dense rule, or
  // the remap would be wasted: decide from the region count before writing anything
  // (the remap keeps the low REG_SHIFT bits: min(k, REG_SHIFT) of them stay constant)
  const uint64_t span_keys = ((uint64_t)regs.size() << REG_SHIFT) >> std::min<uint32_t>(ctx->am.k, REG_SHIFT);
  const uint64_t M = ctx->n_rd + ctx->n_wr;
  if (span_keys > 4 * M + (1ull << 20) || span_keys * 4 > ctx->opts.dense_budget_bytes) return AIWC_OK;
  if (grow(ctx->remap_pay, (n + 1) * 8) != cudaSuccess) {  // no room for the remapped column: sparse path
    cudaGetLastError();
    return AIWC_OK;
  }
  unsigned long long* st = reinterpret_cast<unsigned long long*>(misc + 4);
  const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  CK(cudaMemcpyAsync(st, init, 32, cudaMemcpyHostToDevice, s));
  region_remap_kernel<<<grid, 256, 0, s>>>(kind, payload, n, keys, P<uint32_t>(ctx->reg_vals),
                                           P<uint64_t>(ctx->remap_pay), st);
  CK(cudaMemcpyAsync(stats, st, 32, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  ctx->kernels += 1;
  *out = P<uint64_t>(ctx->remap_pay);
  return AIWC_OK;
}

// First half of an ingest: argument checks, tensor maps, the dense-table pre-clear
// (declared statistics), pass 1 and the class totals (a device->host round trip
// unless the producer declared them).
static int ingest_begin(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, const aiwc_trace_info* info,
                        void* stream) {
  if (!ctx || !info) return AIWC_ERR_ARGUMENT;
  if (ctx->state != 0) return fail(ctx, AIWC_ERR_ARGUMENT, "ctx already holds a trace: call aiwc_reset first");
  const uint64_t n = info->n_events;
  if (n && (!kind || !payload)) return fail(ctx, AIWC_ERR_ARGUMENT, "null column pointer");
  if ((reinterpret_cast<uintptr_t>(kind) & 15) || (reinterpret_cast<uintptr_t>(payload) & 15))
    return fail(ctx, AIWC_ERR_ARGUMENT, "columns must be 16-byte aligned");
  if (n >= (1ull << 32)) return fail(ctx, AIWC_ERR_UNSUPPORTED, "more than 2^32-1 events in one ingest");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  ctx->info = *info;
  ctx->stream_checked = false;
  ctx->state_ok = false;
  ctx->state_n_runs = 0;
  ctx->kernels = 0;
  ctx->d2h = 0;
  ctx->marked = 0;
  ctx->mark(AIWC_PH_INGEST_TOTAL, 0, s);
  DevState* st = P<DevState>(ctx->dev_state);
  const uint64_t n_tiles = (n + TILE - 1) / TILE;
  const bool with_stats = !info->has_addr_stats;
  // Declared class totals (and address statistics, or no memory events) fix every
  // host decision up front: pass 1 and the ingest are queued back to back with
  // no device->host round trip in between; pass 1's totals are checked against
  // the declaration at finalize.
  const bool declared = n && info->has_counts && (!with_stats || info->n_reads + info->n_writes == 0);
  ctx->one_pass = declared;
  uint32_t G = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(n_tiles, 1), (uint64_t)ctx->n_sms * CTAS_PER_SM);
  uint32_t tpc = (uint32_t)((std::max<uint64_t>(n_tiles, 1) + G - 1) / G);
  G = (uint32_t)((std::max<uint64_t>(n_tiles, 1) + tpc - 1) / tpc);
  init_trace_kernel<<<64, 256, 0, s>>>(st, P<unsigned long long>(ctx->wcount), P<unsigned long long>(ctx->wfirst),
                                       nullptr, 0);
  ctx->kernels += 1;
  // opcode counters live in DevState (part of finalize's one read) unless the dictionary is large
  const bool opc_big = info->n_opcodes > (uint32_t)MAX_SMALL_LIST;
  if (opc_big) {
    CK(grow(ctx->opc, (size_t)info->n_opcodes * 8));
    CK(cudaMemsetAsync(ctx->opc.p, 0, (size_t)info->n_opcodes * 8, s));
  }
  // tensor maps depend only on the columns: encode them before any round trip
  CUtensorMap km, pm;
  const uint64_t rows = n / 16;
  if (n) {
    const int rc = encode_maps(ctx, kind, payload, rows, &km, &pm);
    if (rc) return rc;
  }

  // Declared address statistics fix the key map up front: clear a u32 table of
  // that size on the side stream (unless the previous finalize left it clean).
  // Bounded waste when the trace later takes another path: <= 4 keys / event + 2^20.
  ctx->pre_zeroed = 0;
  const bool shard = ctx->opts.flags & AIWC_OPT_SHARD;
  bool light = false;
  if (n && !with_stats && info->addr_min <= info->addr_max && !shard) {
    const uint64_t b0 = info->addr_min & ~1023ull, vary = info->addr_and ^ info->addr_or;
    const uint32_t k0 = vary ? std::min<uint32_t>((uint32_t)__builtin_ctzll(vary), 32u) : 0u;
    const uint64_t sk = (info->addr_max - b0) >> k0;
    if (sk + 1 < DENSE_MAX_KEYS && dense_alloc_keys(sk + 1) * 4 <= ctx->opts.dense_budget_bytes &&
        sk + 1 <= 4 * n + (1ull << 20)) {
      const size_t tb = (size_t)dense_alloc_keys(sk + 1) * 4;  // + the sentinel slot of invalid addresses
      // a dense table and no branches: nothing is staged, so pass 1 need not count
      // instructions or branches (finalize checks the declared instruction total against
      // the opcode counts; a wrong prediction re-runs the full pass 1 in ingest_finish)
      light = declared && info->n_branches == 0 && ctx->bins_off && info->n_reads + info->n_writes > 0 &&
              info->n_opcodes <= (uint32_t)MAX_SMALL_LIST;  // (instructions: checked from the opcode counts)
      if (ctx->dtab_clean >= tb && ctx->dtab.cap >= tb) {
        ctx->pre_zeroed = ctx->dtab_clean;  // cleared after the previous trace (join_ev)
      } else {
        if (ctx->dtab.cap < tb) {
          CK(cudaStreamSynchronize(ctx->aux));
          CK(grow(ctx->dtab, tb));
        }
        CK(cudaEventRecord(ctx->fork_ev, s));
        CK(cudaStreamWaitEvent(ctx->aux, ctx->fork_ev, 0));
        CK(cudaMemsetAsync(ctx->dtab.p, 0, tb, ctx->aux));
        CK(cudaEventRecord(ctx->join_ev, ctx->aux));
        ctx->pre_zeroed = tb;
      }
    }
  }
  const size_t clean_prev = ctx->dtab_clean;  // undeclared traces: the previous finalize's clear may suffice
  ctx->dtab_clean = 0;

  // ---- pass 1: range summaries ----
  const uint32_t n_sub = G * P1_SUB;
  CK(grow(ctx->ranges, (size_t)n_sub * sizeof(RangeSum)));
  if (n) {
    CK(cudaEventRecord(ctx->p1_ev, s));  // the columns (and DevState init) are ready here
    ctx->mark(AIWC_PH_PASS1, 0, s);
    launch_pass1(kind, payload, n, G, tpc, with_stats, P<RangeSum>(ctx->ranges), st, s, light);
    ctx->mark(AIWC_PH_PASS1, 1, s);
    ctx->kernels += 1;
    CK(cudaGetLastError());
  } else {
    CK(cudaMemsetAsync(ctx->ranges.p, 0, (size_t)n_sub * sizeof(RangeSum), s));
  }
  if (declared) {
    ctx->n_instr = info->n_instr; ctx->n_rd = info->n_reads; ctx->n_wr = info->n_writes;
    ctx->n_br = info->n_branches; ctx->n_wgb = info->n_groups; ctx->n_bres = info->any_barrier_or_resume;
  } else {
    // addr_min .. addr_or and the pass-1 totals are contiguous: one 80-byte read
    CK(cudaMemcpyAsync(&ctx->h_state->addr_min, &st->addr_min, 10 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    ctx->d2h += 10 * sizeof(unsigned long long);
    CK(cudaStreamSynchronize(s));
    const unsigned long long* tt = ctx->h_state->p1_tot;
    ctx->n_instr = tt[0]; ctx->n_rd = tt[1]; ctx->n_wr = tt[2]; ctx->n_br = tt[3]; ctx->n_wgb = tt[4];
    ctx->n_bres = tt[5];
  }
  ctx->n_events_seen = n;
  ctx->pend.kind = kind; ctx->pend.payload = payload; ctx->pend.rows = rows;
  ctx->pend.km = km; ctx->pend.pm = pm;
  ctx->pend.opc_big = opc_big; ctx->pend.with_stats = with_stats; ctx->pend.clean_prev = clean_prev;
  ctx->pend.G = G; ctx->pend.tpc = tpc; ctx->pend.light = light;
  return AIWC_OK;
}

// Second half: the memory path from address statistics (the trace's own, or in
// the shard path the whole job's), buffers, the ingest kernel.
static int ingest_finish(aiwc_ctx* ctx, uint64_t amin, uint64_t amax, uint64_t aand, uint64_t aor, uint64_t M,
                         bool want_dense, void* stream) {
  const aiwc_trace_info* info = &ctx->info;
  const uint64_t n = info->n_events;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint8_t* kind = ctx->pend.kind;
  const uint64_t* payload = ctx->pend.payload;
  const uint64_t rows = ctx->pend.rows;
  CUtensorMap km = ctx->pend.km, pm = ctx->pend.pm;
  const bool opc_big = ctx->pend.opc_big;
  const size_t clean_prev = ctx->pend.clean_prev;
  const uint32_t G = ctx->pend.G, tpc = ctx->pend.tpc;
  const bool shard = ctx->opts.flags & AIWC_OPT_SHARD;
  DevState* st = P<DevState>(ctx->dev_state);
  const uint64_t M_local = ctx->n_rd + ctx->n_wr;
  // ---- memory path decision ----
  auto decide_memory = [&](uint64_t amin, uint64_t amax, uint64_t aand, uint64_t aor) {
    ctx->dense = false;
    ctx->dense32 = M < E32_MAX_ACCESSES;
    ctx->am = AddrMap{};
    if (M) {
      AddrMap& am = ctx->am;
      am.base = amin & ~1023ull;
      am.hi = amax;
      const uint64_t vary = aand ^ aor;
      // constant low bits dropped from keys; capped at 32 so the per-event check of
      // the dropped bits is one 32-bit compare in the ingest kernel
      am.k = vary ? std::min<uint32_t>((uint32_t)__builtin_ctzll(vary), 32u) : 0u;
      am.low_mask = am.k >= 64 ? ~0ull : ((1ull << am.k) - 1);
      am.low_const = (amin - am.base) & am.low_mask;
      const uint64_t span_keys = (amax - am.base) >> am.k;
      am.n_keys = span_keys + 1;
      am.off_max = (span_keys << am.k) | am.low_mask;
      // u32 entries cost a second (flag) RED per access but halve the table:
      // worth it when the table traffic dominates (few accesses per key)
      // With the hot-key window (keys of one contended 1024-key block counted in shared
      // memory) the flag RED of the u32 form stays cheap up to a few accesses per key.
      const bool hot_window = am.n_keys > SMEM_TABLE_KEYS && M >= HOT_MIN_ACCESSES && !ctx->hot_off;
      ctx->dense32 = M < E32_MAX_ACCESSES && (M <= am.n_keys || (hot_window && M <= 4 * am.n_keys));
      if (ctx->dense_entry == 32) ctx->dense32 = M < E32_MAX_ACCESSES && am.n_keys > SMEM_TABLE_KEYS;
      if (ctx->dense_entry == 64) ctx->dense32 = false;
      const bool fits = span_keys < DENSE_MAX_KEYS - 1 &&
                        dense_alloc_keys(am.n_keys) * (ctx->dense32 ? 4 : 8) <= ctx->opts.dense_budget_bytes &&
                        am.n_keys <= 4 * M + (1ull << 20);
      // a shard either fills a dense table over the whole job's key map (the dense
      // exchange) or keeps its addresses compacted for the owner exchange
      ctx->dense = fits && (!shard || want_dense);
    }
  };
  if (M_local && amin > amax) return fail(ctx, AIWC_ERR_ARGUMENT, "address statistics are empty but the trace has memory events");
  decide_memory(amin, amax, aand, aor);
  ctx->stats4[0] = amin; ctx->stats4[1] = amax; ctx->stats4[2] = aand; ctx->stats4[3] = aor;
  ctx->shard_dense = shard && ctx->dense;
  // a span too wide for the table: if the accesses sit in few 1 MB regions, squeeze
  // the regions together (exact for every memory statistic) and keep the dense path
  if (M && n && !ctx->dense && !shard && !ctx->region_off) {
    const uint64_t* np = nullptr;
    unsigned long long rs[4];
    const int rc = region_compact(ctx, kind, payload, n, s, &np, rs);
    if (rc) return rc;
    if (np) {
      payload = np;
      const int rc2 = encode_maps(ctx, kind, payload, rows, &km, &pm);
      if (rc2) return rc2;
      decide_memory(rs[0], rs[1], rs[2], rs[3]);
      ctx->stats4[0] = rs[0]; ctx->stats4[1] = rs[1]; ctx->stats4[2] = rs[2]; ctx->stats4[3] = rs[3];
    }
  }
  const bool stage = !ctx->dense || ctx->n_br > 0;
  if (ctx->pend.light && (stage || shard)) {  // the light pass 1 was mispredicted: the staging needs its counts
    CK(cudaMemsetAsync(st->p1_tot, 0, sizeof(st->p1_tot), s));
    launch_pass1(kind, payload, n, G, tpc, ctx->pend.with_stats, P<RangeSum>(ctx->ranges), st, s, false);
    ctx->kernels += 1;
    ctx->pend.light = false;
  }

  // ---- buffers ----
  // an ITB / IPT sample >= HBINS spans >= HBINS distinct instructions: that bounds both overflow lists
  CK(grow(ctx->itb_ovf, (ctx->n_instr / HBINS + 2) * 4));
  CK(grow(ctx->ipt_ovf, (ctx->n_instr / HBINS + 2) * 4));
  ctx->ipt_tab_len = 0;
  if (ctx->n_bres) {
    ctx->ipt_tab_len = ctx->n_wgb * (uint64_t)std::max<uint32_t>(info->local_volume, 1);
    CK(grow(ctx->ipt_tab, ctx->ipt_tab_len * 8));
    CK(cudaMemsetAsync(ctx->ipt_tab.p, 0, ctx->ipt_tab_len * 8, s));
  }
  CK(grow(ctx->br, std::max<uint64_t>(ctx->n_br, 1) * 8));
  if (M) {
    if (ctx->dense) {
      const size_t tb = dense_alloc_keys(ctx->am.n_keys) * (ctx->dense32 ? 4 : 8);  // + the sentinel slot
      if (ctx->shard_dense) {  // bitmap of the 1024-key chunks this rank touches (the sentinel's included)
        ctx->n_chunk_words = ((ctx->am.n_keys + 1 + 1023) / 1024 + 31) / 32;
        CK(grow(ctx->chunk_bits, ctx->n_chunk_words * 4));
        CK(cudaMemsetAsync(ctx->chunk_bits.p, 0, ctx->n_chunk_words * 4, s));
      }
      size_t zeroed = ctx->pre_zeroed;
      if (!zeroed && clean_prev >= tb && ctx->dtab.cap >= tb) zeroed = clean_prev;  // cleared on aux (join_ev)
      if (zeroed) CK(cudaStreamWaitEvent(s, ctx->join_ev, 0));
      if (zeroed < tb) {
        CK(grow(ctx->dtab, tb));
        CK(cudaMemsetAsync(ctx->dtab.p, 0, tb, s));
      }
      ctx->dtab_used = tb;
    } else {
      CK(grow(ctx->rd, std::max<uint64_t>(ctx->n_rd, 1) * 8));
      CK(grow(ctx->wr, std::max<uint64_t>(ctx->n_wr, 1) * 8));
    }
    CK(grow(ctx->lvl0_ovf, (M / CBINS + 2) * 8));
  }
  if (ctx->pre_zeroed && !ctx->dense) CK(cudaStreamWaitEvent(s, ctx->join_ev, 0));

  ctx->n_ranges = G;
  ctx->tiles_per_cta = tpc;
  const uint32_t pres_blocks = (tpc + PRES_TILES - 1) / PRES_TILES;
  CK(grow(ctx->wpres, (size_t)G * P1_SUB * pres_blocks * 4));
  CK(cudaMemsetAsync(ctx->wpres.p, 0, (size_t)G * P1_SUB * pres_blocks * 4, s));

  // ---- main ingest pass ----
  if (n) {
    IngestArgs a{};
    a.kind = kind; a.payload = payload; a.n = n; a.tma_rows = rows;
    a.tiles_per_cta = tpc; a.n_opcodes = info->n_opcodes; a.local_volume = std::max<uint32_t>(info->local_volume, 1);
    a.ranges = P<RangeSum>(ctx->ranges); a.st = st;
    a.opc_counts = opc_big ? P<unsigned long long>(ctx->opc) : st->opc_small;
    a.width_count = P<unsigned long long>(ctx->wcount); a.width_first = P<unsigned long long>(ctx->wfirst);
    a.width_presence = P<uint32_t>(ctx->wpres);
    a.pres_blocks = pres_blocks;
    a.itb_ovf = P<uint32_t>(ctx->itb_ovf); a.ipt_ovf = P<uint32_t>(ctx->ipt_ovf);
    a.ipt_tab = ctx->ipt_tab_len ? P<unsigned long long>(ctx->ipt_tab) : nullptr; a.ipt_tab_len = ctx->ipt_tab_len;
    a.am = ctx->am;
    a.dense = ctx->dense ? ctx->dtab.p : nullptr;
    a.dense32 = ctx->dense32;
    a.smem_keys = 0; a.hot_lo = 0; a.hot_dev = nullptr;
    if (ctx->dense && !ctx->dense32 && ctx->am.n_keys <= SMEM_TABLE_KEYS) {
      a.smem_keys = SMEM_TABLE_KEYS;  // the whole (small) table per CTA: a full window (the bank swizzle
                                      // permutes inside 1024 keys; keys >= n_keys are never flushed)
    } else if (ctx->dense && ctx->am.n_keys > SMEM_TABLE_KEYS && M >= HOT_MIN_ACCESSES && !ctx->hot_off) {
      // a 1024-key window holding many accesses (shared scratch, lookup tables) is
      // counted per CTA in shared memory: its keys would otherwise serialise in L2
      a.smem_keys = SMEM_TABLE_KEYS;
      a.hot_dev = &st->hot_key;
      CK(cudaStreamWaitEvent(ctx->aux2, ctx->p1_ev, 0));
      launch_hot_sample(kind, payload, n, ctx->am, &st->hot_key, ctx->aux2);
      CK(cudaEventRecord(ctx->hot_ev, ctx->aux2));
      CK(cudaStreamWaitEvent(s, ctx->hot_ev, 0));
      ctx->kernels += 1;
    }
    a.rd_out = P<uint64_t>(ctx->rd); a.wr_out = P<uint64_t>(ctx->wr); a.br_out = P<uint64_t>(ctx->br);
    a.chunk_bits = ctx->shard_dense ? P<uint32_t>(ctx->chunk_bits) : nullptr;
    // in-pass StreamChecker for untrusted columns; with barriers / resumes the
    // per-work-item order rules take three words per (group, lid) slot
    ctx->stream_checked = info->check_stream;
    a.check = ctx->stream_checked;
    ctx->wi_rules_on = false;
    if (a.check) {
      a.dup_len = std::max<uint64_t>(ctx->n_wgb, 1) * a.local_volume;
      ctx->dup_len = a.dup_len;
      CK(grow(ctx->dup_bits, (a.dup_len + 31) / 32 * 4));
      CK(cudaMemsetAsync(ctx->dup_bits.p, 0, (a.dup_len + 31) / 32 * 4, s));
      a.dup_bits = P<uint32_t>(ctx->dup_bits);
      if (ctx->n_bres) {
        CK(grow(ctx->wi_rules, a.dup_len * 24));
        CK(cudaMemsetAsync(ctx->wi_rules.p, 0, a.dup_len * 24, s));
        a.wi_rules = P<unsigned long long>(ctx->wi_rules);
        ctx->wi_rules_on = true;
      }
    }
    // key-block bins: a dense table well beyond L2 with many accesses -- the zone
    // sampler (beside pass 1, on the device) decides whether any key zone is random
    const size_t tab_bytes = dense_alloc_keys(ctx->am.n_keys) * (ctx->dense32 ? 4 : 8);
    ctx->bins = ctx->dense && !ctx->shard_dense && !ctx->bins_off && M < (1ull << 32) &&
                ((tab_bytes > (256ull << 20) && M >= (1ull << 22)) || ctx->bins_force);
    a.bin_zones = nullptr;
    if (ctx->bins) {
      const uint32_t nw = G * P1_SUB;
      CK(grow(ctx->bin_seg, M * 4));
      CK(grow(ctx->bin_base, (size_t)nw * 8));
      CK(grow(ctx->bin_fill, (size_t)nw * 4));
      CK(cudaMemsetAsync(ctx->bin_fill.p, 0, (size_t)nw * 4, s));
      const uint32_t keybits = 64 - __builtin_clzll(std::max<uint64_t>(ctx->am.n_keys - 1, 1));
      a.zone_shift = (uint32_t)std::max<int>(15, (int)keybits - 6);
      CK(cudaStreamWaitEvent(ctx->aux2, ctx->p1_ev, 0));
      launch_zone_sample(kind, payload, n, ctx->am, a.zone_shift, st->zone_counts, &st->bin_zones, ctx->aux2);
      CK(cudaEventRecord(ctx->hot_ev, ctx->aux2));
      CK(cudaStreamWaitEvent(s, ctx->hot_ev, 0));
      ctx->kernels += 2;
      a.bin_seg = P<uint32_t>(ctx->bin_seg);
      a.bin_base = P<unsigned long long>(ctx->bin_base);
      a.bin_fill = P<uint32_t>(ctx->bin_fill);
      a.bin_zones = &st->bin_zones;
    }
    ctx->mark(AIWC_PH_INGEST, 0, s);
    CK(launch_ingest(a, km, pm, G, ctx->dense, stage, s));
    ctx->mark(AIWC_PH_INGEST, 1, s);
    ctx->kernels += 1;
    if (ctx->n_instr) {  // first index of each width 1..16 (the columns are only ours until here)
      launch_width_first(kind, payload, n, P<uint32_t>(ctx->wpres), G * P1_SUB, pres_blocks, tpc, WARP_TILE,
                         P<unsigned long long>(ctx->wfirst), st, s);
      ctx->kernels += 2;
    }
  }
  ctx->mark(AIWC_PH_INGEST_TOTAL, 1, s);
  ctx->state = 1;
  return AIWC_OK;
}

static int job_ingest(aiwc_ctx* ctx, void* stream);

extern "C" int aiwc_ingest(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, const aiwc_trace_info* info,
                           void* stream) {
  int rc = ingest_begin(ctx, kind, payload, info, stream);
  if (rc) return rc;
  if (ctx->comm) return job_ingest(ctx, stream);
  const bool own = ctx->pend.with_stats;  // pass 1 measured the statistics, else they were declared
  const DevState& h = *ctx->h_state;
  return ingest_finish(ctx, own ? h.addr_min : info->addr_min, own ? h.addr_max : info->addr_max,
                       own ? h.addr_and : info->addr_and, own ? h.addr_or : info->addr_or, ctx->n_rd + ctx->n_wr,
                       false, stream);
}

extern "C" int aiwc_ingest_host(aiwc_ctx* ctx, const uint8_t* kind_host, const uint64_t* payload_host,
                                const aiwc_trace_info* info, void* stream) {
  if (!ctx || !info) return AIWC_ERR_ARGUMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t n = info->n_events;
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->kind_stage, (n + 16) * 1));
  CK(grow(ctx->pay_stage, (n + 16) * 8));
  if (n) {
    CK(cudaMemcpyAsync(ctx->kind_stage.p, kind_host, n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->pay_stage.p, payload_host, n * 8, cudaMemcpyHostToDevice, s));
  }
  return aiwc_ingest(ctx, P<uint8_t>(ctx->kind_stage), P<uint64_t>(ctx->pay_stage), info, stream);
}

// smallest k with the top-k counts covering >= 9/10 of the total (entropy.py:49-66),
// counts given as a descending list of big values followed by a histogram of small ones
static uint64_t coverage_from(const std::vector<uint64_t>& big_desc, const unsigned long long* small_hist,
                              uint32_t n_small_bins, unsigned __int128 total) {
  if (total == 0) return 0;
  unsigned __int128 cum = 0;
  uint64_t k = 0;
  for (uint64_t c : big_desc) {
    cum += c; ++k;
    if (cum * 10 >= total * 9) return k;
  }
  for (int64_t c = (int64_t)n_small_bins - 1; c >= 1; --c) {
    const uint64_t h = small_hist ? small_hist[c] : 0;
    if (!h) continue;
    const unsigned __int128 need = total * 9 - cum * 10;  // > 0 here
    const unsigned __int128 per = (unsigned __int128)c * 10;
    const unsigned __int128 take = (need + per - 1) / per;
    if (take <= h) return k + (uint64_t)take;
    cum += (unsigned __int128)h * c;
    k += h;
  }
  return k;
}

static void order_stats(const unsigned long long* hist, const std::vector<uint64_t>& ovf_sorted, aiwc_dist* d) {
  uint64_t small = 0;
  for (int i = 0; i < HBINS; ++i) small += hist[i];
  d->n = small + ovf_sorted.size();
  if (!d->n) return;
  auto at = [&](uint64_t rank) -> uint64_t {
    if (rank >= small) return ovf_sorted[rank - small];
    uint64_t c = 0;
    for (int i = 0; i < HBINS; ++i) {
      c += hist[i];
      if (rank < c) return (uint64_t)i;
    }
    return 0;
  };
  d->min = at(0);
  d->max = at(d->n - 1);
  d->mid_lo = at((d->n - 1) / 2);
  d->mid_hi = at(d->n / 2);
}

static int fetch_sorted_u32(aiwc_ctx* ctx, Buf& src, uint64_t n, std::vector<uint64_t>& out, cudaStream_t s) {
  out.clear();
  if (!n) return AIWC_OK;
  CK(grow(ctx->sort_a, n * 8));
  CK(grow(ctx->sort_b, n * 8));
  CK(grow(ctx->sort_h, radix_hist_bytes(n)));
  widen_u32_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1024), 256, 0, s>>>(P<uint32_t>(src), n,
                                                                                      P<uint64_t>(ctx->sort_a));
  int k = 1;
  radix_sort_u64(P<uint64_t>(ctx->sort_a), P<uint64_t>(ctx->sort_b), n, 0, 32, P<uint32_t>(ctx->sort_h), s, &k);
  ctx->kernels += k;
  out.resize(n);
  CK(cudaMemcpyAsync(out.data(), ctx->sort_a.p, n * 8, cudaMemcpyDeviceToHost, s));
  ctx->d2h += n * 8;
  return AIWC_OK;
}

static int finalize_local(aiwc_ctx* ctx, aiwc_result* out, void* stream) {
  if (!ctx || !out) return AIWC_ERR_ARGUMENT;
  if (ctx->state != 1) return fail(ctx, AIWC_ERR_ARGUMENT, "finalize needs exactly one ingest since reset");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  DevState* st = P<DevState>(ctx->dev_state);
  const bool shard = ctx->opts.flags & AIWC_OPT_SHARD;
  const uint64_t M = shard ? 0 : ctx->n_rd + ctx->n_wr;  // a shard's memory is finished by the key owners
  ctx->mark(AIWC_PH_FINALIZE_TOTAL, 0, s);
  if (ctx->stream_checked && ctx->info.n_events) {  // set bits of the duplicate-begin map -> DevState
    const uint64_t words = (ctx->dup_len + 31) / 32;
    popcount_kernel<<<(unsigned)std::min<uint64_t>((words + 255) / 256, (uint64_t)ctx->n_sms * 4), 256, 0, s>>>(
        P<uint32_t>(ctx->dup_bits), words, &st->dup_set);
    ctx->kernels += 1;
    if (ctx->wi_rules_on) {
      const uint32_t lv = std::max<uint32_t>(ctx->info.local_volume, 1);
      const uint64_t groups = ctx->dup_len / lv;
      wi_rules_kernel<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 7) / 8, (uint64_t)ctx->n_sms * 8)),
                        256, 0, s>>>(P<unsigned long long>(ctx->wi_rules), groups, lv, st);
      ctx->kernels += 1;
    }
  }

  // ---- device finishing: IPT slots, widths, memory ----
  if (ctx->ipt_tab_len) {
    launch_ipt_table(P<unsigned long long>(ctx->ipt_tab), ctx->ipt_tab_len, st, P<uint32_t>(ctx->ipt_ovf), s);
    ctx->kernels += 1;
  }
  launch_width_list(P<unsigned long long>(ctx->wcount), P<unsigned long long>(ctx->wfirst), st, s);
  ctx->kernels += 1;
  ctx->mark(AIWC_PH_MEMORY, 0, s);
  ctx->binned = 0;
  if (M && ctx->dense && ctx->bins) {  // the binned accesses into the table first
    unsigned long long nb = 0;
    CK(cudaMemcpyAsync(&nb, &st->bin_total, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->d2h += 8;
    ctx->binned = nb;
    if (nb) {
      const uint32_t nw = ctx->n_ranges * P1_SUB;
      CK(grow(ctx->bin_scr, bin_scratch_bytes(nb, nw, (ctx->am.n_keys >> 14) + 2)));
      ctx->kernels += bin_finish(P<uint32_t>(ctx->bin_seg), P<unsigned long long>(ctx->bin_base),
                                 P<uint32_t>(ctx->bin_fill), nw, nb, ctx->dtab.p, ctx->dense32, ctx->am.n_keys,
                                 ctx->bin_scr.p, s);
    }
  }
  if (M) {
    if (ctx->dense) {
      const uint64_t chunks = (ctx->am.n_keys + 1023) / 1024;
      const uint32_t nct = (uint32_t)std::min<uint64_t>(chunks, ctx->n_parts);
      // the per-key state as runs for a later state merge -- tables up to 512 MB (a sweep of a
      // larger table would cost a sizeable part of its ingest; such merges re-ingest)
      const bool export_runs = ctx->info.export_state && !ctx->remap_pay.p &&
                               dense_alloc_keys(ctx->am.n_keys) * (ctx->dense32 ? 4 : 8) <= (512ull << 20);
      // Without a later reader, tables of >= 1 GiB are zeroed by the statistics pass as it
      // reads them (C3: step 12.04 -> 11.64 ms): a separate clear of that size competes
      // with the next trace's memory-bound ingest.  Smaller tables keep the side-stream
      // clear, which hides behind compute-bound passes (C2: fused 0.988 vs 0.969 ms).
      const size_t tab_bytes = (size_t)ctx->am.n_keys * (ctx->dense32 ? 4 : 8);
      const bool clear_in_stats = !export_runs && tab_bytes >= (1ull << 30);
      launch_dense_stats(ctx->dtab.p, ctx->dense32, ctx->am.n_keys, ctx->am.k, M, st,
                         P<double>(ctx->partials), nct, P<uint64_t>(ctx->lvl0_ovf), s, nullptr, 0, 0, 1,
                         clear_in_stats);
      if (export_runs) {
        // one pass, no round trip: runs are claimed chunk by chunk into a buffer of a
        // quarter run per key (runs that do not compress the table that much -- random
        // accesses -- overflow it and the state is dropped: such merges re-ingest)
        const uint64_t cap = std::max<uint64_t>(1ull << 16, ctx->am.n_keys / 4);
        CK(grow(ctx->state_runs, cap * 16));
        launch_pack_all(ctx->dtab.p, ctx->dense32, ctx->am.n_keys, &st->state_runs_n, P<uint64_t>(ctx->state_runs), 1,
                        (uint32_t)ctx->n_sms, s, cap);
        ctx->state_cap = cap;
        ctx->state_ok = true;  // confirmed against the claimed count after the state read below
        ctx->kernels += 1;
      }
      // the table is clean again for the next trace: zeroed by the statistics pass up to
      // n_keys (the words after it -- the sentinel slot, allocation padding -- here), or
      // cleared on the side stream now
      if (clear_in_stats) {
        if (ctx->dtab_used > tab_bytes)
          CK(cudaMemsetAsync(reinterpret_cast<uint8_t*>(ctx->dtab.p) + tab_bytes, 0, ctx->dtab_used - tab_bytes, s));
        CK(cudaEventRecord(ctx->join_ev, s));
      } else {
        CK(cudaEventRecord(ctx->fork_ev, s));
        CK(cudaStreamWaitEvent(ctx->aux, ctx->fork_ev, 0));
        CK(cudaMemsetAsync(ctx->dtab.p, 0, ctx->dtab_used, ctx->aux));
        CK(cudaEventRecord(ctx->join_ev, ctx->aux));
      }
      ctx->dtab_clean = ctx->dtab_used;
      launch_entropy_finish(st, P<double>(ctx->partials), nct, M, ctx->am.k, s);
      ctx->kernels += 2;
    } else {
      CK(grow(ctx->sparse_scr, sparse_scratch_bytes(M)));
      const int raw = bitwidth64((ctx->am.hi - ctx->am.base) >> ctx->am.k) > 63;
      const uint32_t parts = std::min<uint32_t>(ctx->n_parts, 256);
      ctx->kernels += sparse_memory_stats(P<uint64_t>(ctx->rd), ctx->n_rd, P<uint64_t>(ctx->wr), ctx->n_wr, ctx->am, M,
                                          st, P<double>(ctx->partials), parts, P<uint64_t>(ctx->lvl0_ovf),
                                          ctx->sparse_scr.p, ctx->sparse_scr.cap, s);
      launch_entropy_finish(st, P<double>(ctx->partials), parts, M, raw ? 64u : ctx->am.k, s);
      ctx->kernels += 1;
    }
  }
  ctx->mark(AIWC_PH_MEMORY, 1, s);
  // branch walk phase 1 before the read-back: its site-table overflow flag comes back with it
  if (ctx->n_br) {
    CK(grow(ctx->branch_scr, branch_scratch_bytes(ctx->n_br)));
    ctx->mark(AIWC_PH_BRANCH, 0, s);
    ctx->kernels += branch_walk_prepare(P<uint64_t>(ctx->br), ctx->n_br, ctx->opts.history_len, st,
                                        ctx->branch_scr.p, s);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ctx->h_state, st, offsetof(DevState, host_end), cudaMemcpyDeviceToHost, s));
  ctx->d2h += offsetof(DevState, host_end);
  CK(cudaStreamSynchronize(s));

  // ---- branches ----
  if (ctx->n_br) {
    const uint32_t site_bits = (uint32_t)bitwidth64(ctx->h_state->max_site);
    ctx->kernels += branch_stats(P<uint64_t>(ctx->br), ctx->n_br, site_bits, ctx->opts.history_len,
                                 ctx->h_state->bw_overflow == 0, st,
                                 P<unsigned long long>(ctx->branch_tab), ctx->branch_scr.p, ctx->branch_scr.cap, s);
    ctx->mark(AIWC_PH_BRANCH, 1, s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_state, st, offsetof(DevState, host_end), cudaMemcpyDeviceToHost, s));
    ctx->d2h += offsetof(DevState, host_end);
    CK(cudaStreamSynchronize(s));
  }
  DevState& h = *ctx->h_state;
  if (ctx->one_pass) {  // the declared class totals against what the pass counted
    const aiwc_trace_info& in = ctx->info;
    unsigned long long n_in = h.p1_tot[0];
    if (ctx->pend.light) {  // light pass 1: every instruction event landed in an opcode counter
      n_in = 0;
      for (uint32_t i = 0; i < in.n_opcodes; ++i) n_in += h.opc_small[i];
    }
    const bool same = n_in == in.n_instr && h.p1_tot[1] == in.n_reads && h.p1_tot[2] == in.n_writes &&
                      h.p1_tot[3] == in.n_branches && h.p1_tot[4] == in.n_groups &&
                      (h.p1_tot[5] != 0) == (in.any_barrier_or_resume != 0);
    if (!same) return fail(ctx, AIWC_ERR_ARGUMENT, "declared class counts differ from the trace");
  }
  // compacted (sort-path) addresses: the ingest measured their statistics; a declared
  // hint the keys were built from must cover them (the dense path checks per access)
  if (!ctx->dense && ctx->info.has_addr_stats && ctx->n_rd + ctx->n_wr && h.addr_min <= h.addr_max) {
    const AddrMap& am = ctx->am;
    const bool ok = h.addr_min >= am.base && h.addr_max <= am.hi && ((h.addr_and ^ h.addr_or) & am.low_mask) == 0 &&
                    ((h.addr_min - am.base) & am.low_mask) == am.low_const;
    if (!ok) h.flags |= F_ADDR_HINT;
  }
  if (ctx->state_ok) {  // the exported runs fit their buffer?
    ctx->state_n_runs = h.state_runs_n;
    ctx->state_ok = h.state_runs_n <= ctx->state_cap;
  }
  // every wi_begin set its own (group, lid) bit: fewer set bits than begins = a duplicate
#if !defined(AIWC_ABL) || !(AIWC_ABL & 128)  // (measurement builds without the duplicate-begin REDs)
  if (ctx->stream_checked && ctx->info.n_events && h.dup_set != h.n_wib) h.flags |= F_STREAM;
#endif
  if (h.flags & F_STREAM) {
    fail(ctx, AIWC_ERR_INVALID_STREAM, "stream invariant violated (aiwc_validate locates the first violation)");
    return AIWC_ERR_INVALID_STREAM;
  }
  if (h.flags) {
    char m[160];
    const char* what = (h.flags & F_ADDR_HINT) ? "memory address outside the declared address statistics"
                       : (h.flags & F_BAD_OPCODE) ? "opcode id outside the opcode dictionary"
                       : (h.flags & F_BAD_WIDTH)  ? "instruction width >= 65536 is not supported"
                       : (h.flags & F_BAD_SITE)   ? "branch site >= 2^32 is not supported"
                       : (h.flags & F_BAD_GROUP)  ? "group key >= 2^31 is not supported"
                       : (h.flags & F_SLOT_RANGE) ? "work-item slot outside the group table (invalid stream)"
                                                  : "unknown kind byte in the trace";
    snprintf(m, sizeof m, "%s (flags=0x%llx)", what, (unsigned long long)h.flags);
    const int code = (h.flags & (F_ADDR_HINT)) ? AIWC_ERR_ARGUMENT
                     : (h.flags & (F_SLOT_RANGE | F_BAD_KIND)) ? AIWC_ERR_INCONSISTENT : AIWC_ERR_UNSUPPORTED;
    return fail(ctx, code, m);
  }

  // ---- second-round small reads ----
  int rc;
  if ((rc = fetch_sorted_u32(ctx, ctx->itb_ovf, h.itb_ovf_n, ctx->itb_ovf_sorted, s))) return rc;
  if ((rc = fetch_sorted_u32(ctx, ctx->ipt_ovf, h.ipt_ovf_n, ctx->ipt_ovf_sorted, s))) return rc;
  ctx->lvl0_sorted.clear();
  if (h.lvl0_ovf_n) {
    const uint64_t L = h.lvl0_ovf_n;
    CK(grow(ctx->sort_b, L * 8));
    CK(grow(ctx->sort_h, radix_hist_bytes(L)));
    int k = 0;
    radix_sort_u64(P<uint64_t>(ctx->lvl0_ovf), P<uint64_t>(ctx->sort_b), L, 0, bitwidth64(M), P<uint32_t>(ctx->sort_h),
                   s, &k);
    ctx->kernels += k;
    ctx->lvl0_sorted.resize(L);
    CK(cudaMemcpyAsync(ctx->lvl0_sorted.data(), ctx->lvl0_ovf.p, L * 8, cudaMemcpyDeviceToHost, s));
    ctx->d2h += L * 8;
  }
  const uint32_t n_opc = ctx->info.n_opcodes;
  if (n_opc > (uint32_t)MAX_SMALL_LIST) {
    ctx->opc_counts.assign(n_opc, 0);
    CK(cudaMemcpyAsync(ctx->opc_counts.data(), ctx->opc.p, (size_t)n_opc * 8, cudaMemcpyDeviceToHost, s));
    ctx->d2h += (size_t)n_opc * 8;
  } else {
    ctx->opc_counts.assign(h.opc_small, h.opc_small + n_opc);
  }
  std::vector<unsigned long long> big_sites;
  if (h.n_sites > (unsigned long long)MAX_SMALL_LIST) {
    big_sites.resize(2 * h.n_sites);
    // big list lives after the sort scratch inside branch_scr (see branch_stats)
    const size_t off = branch_site_list_offset(ctx->n_br);
    CK(cudaMemcpyAsync(big_sites.data(), reinterpret_cast<uint8_t*>(ctx->branch_scr.p) + off, 2 * h.n_sites * 8,
                       cudaMemcpyDeviceToHost, s));
  }
  std::vector<unsigned long long> wc_full, wf_full;
  if (h.n_widths_listed > (unsigned long long)MAX_SMALL_LIST) {
    wc_full.resize(WIDTH_TABLE); wf_full.resize(WIDTH_TABLE);
    CK(cudaMemcpyAsync(wc_full.data(), ctx->wcount.p, WIDTH_TABLE * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(wf_full.data(), ctx->wfirst.p, WIDTH_TABLE * 8, cudaMemcpyDeviceToHost, s));
  }
  ctx->mark(AIWC_PH_FINALIZE_TOTAL, 1, s);
  // a second round trip only when the second round queued work (overflow lists,
  // big dictionaries) or the phase events must be read
  const bool second_round = h.itb_ovf_n || h.ipt_ovf_n || h.lvl0_ovf_n || n_opc > (uint32_t)MAX_SMALL_LIST ||
                            h.n_sites > (unsigned long long)MAX_SMALL_LIST ||
                            h.n_widths_listed > (unsigned long long)MAX_SMALL_LIST;
  if (second_round || ctx->timing) CK(cudaStreamSynchronize(s));
  std::reverse(ctx->lvl0_sorted.begin(), ctx->lvl0_sorted.end());

  // ---- assemble ----
  aiwc_result r{};
  r.n_events = ctx->n_events_seen;
  r.total_instructions = ctx->n_instr;
  r.work_items = h.n_wib;
  r.barriers_hit = h.n_bar;
  {
    std::vector<uint64_t> oc;
    for (uint64_t c : ctx->opc_counts) if (c) oc.push_back(c);
    std::sort(oc.begin(), oc.end(), std::greater<uint64_t>());
    unsigned __int128 tot = 0;
    for (uint64_t c : oc) tot += c;
    r.opcode_coverage = coverage_from(oc, nullptr, 0, tot);
  }
  order_stats(h.itb_hist, ctx->itb_ovf_sorted, &r.itb);
  r.itb.sum = h.itb_sum;
  order_stats(h.ipt_hist, ctx->ipt_ovf_sorted, &r.ipt);
  r.ipt.sum = h.ipt_sum;
  r.total_reads = ctx->n_rd;
  r.total_writes = ctx->n_wr;
  r.unique_reads = h.unique_r;
  r.unique_writes = h.unique_w;
  r.footprint = h.footprint;
  r.footprint_90 = M ? coverage_from(ctx->lvl0_sorted, h.cnt_hist0, CBINS, M) : 0;
  for (int i = 0; i < NLEVELS; ++i) {
    const double v = M ? h.entropy[i] : 0.0;
    if (i == 0) r.gmae = v; else r.lmae[i - 1] = v;
  }
  r.branch_executions = ctx->n_br;
  r.branch_observations = ctx->n_br ? h.n_obs : 0;
  r.branch_excluded = ctx->n_br - r.branch_observations;
  r.yokota = ctx->n_br ? h.yokota : 0.0;
  r.linear = ctx->n_br ? h.linear : 0.0;
  // sites: (site, first position) pairs -> counts
  ctx->site_ids.clear(); ctx->site_counts.clear();
  if (ctx->n_br) {
    std::vector<std::pair<uint64_t, uint64_t>> heads;  // (position, site)
    const uint64_t ns = h.n_sites;
    for (uint64_t i = 0; i < ns; ++i) {
      if (ns <= (uint64_t)MAX_SMALL_LIST) heads.emplace_back(h.site_list[2 * i + 1], h.site_list[2 * i]);
      else heads.emplace_back(big_sites[2 * i + 1], big_sites[2 * i]);
    }
    std::sort(heads.begin(), heads.end());
    for (size_t i = 0; i < heads.size(); ++i) {
      const uint64_t end = i + 1 < heads.size() ? heads[i + 1].first : ctx->n_br;
      ctx->site_ids.push_back(heads[i].second);
      ctx->site_counts.push_back(end - heads[i].first);
    }
    std::vector<uint64_t> sc(ctx->site_counts);
    std::sort(sc.begin(), sc.end(), std::greater<uint64_t>());
    r.branch_90 = coverage_from(sc, nullptr, 0, ctx->n_br);
  }
  r.n_sites = ctx->site_ids.size();
  // widths in first-appearance order
  ctx->width_vals.clear(); ctx->width_counts.clear(); ctx->width_firsts.clear();
  if (h.n_widths_listed <= (unsigned long long)MAX_SMALL_LIST) {
    for (uint64_t i = 0; i < h.n_widths_listed; ++i) {
      ctx->width_vals.push_back(h.width_list[3 * i]);
      ctx->width_counts.push_back(h.width_list[3 * i + 1]);
      ctx->width_firsts.push_back(h.width_list[3 * i + 2]);
    }
  } else {
    std::vector<std::pair<uint64_t, uint32_t>> order;
    for (uint32_t w = 0; w < WIDTH_TABLE; ++w) if (wc_full[w]) order.emplace_back(wf_full[w], w);
    std::sort(order.begin(), order.end());
    for (auto& o : order) {
      ctx->width_vals.push_back(o.second); ctx->width_counts.push_back(wc_full[o.second]);
      ctx->width_firsts.push_back(o.first);
    }
  }
  if (shard || ctx->info.export_state) {  // the pooled pattern table (summed across ranks / merged parts)
    const size_t tb = (size_t(1) << ctx->opts.history_len);
    ctx->branch_tab_host.assign(tb, 0);
    if (ctx->n_br) {
      CK(cudaMemcpyAsync(ctx->branch_tab_host.data(), ctx->branch_tab.p, tb * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      ctx->d2h += tb * 8;
    }
  }
  r.entries = r.unique_reads + r.unique_writes + r.branch_executions;
  r.n_opcodes = n_opc;
  r.opcode_counts = ctx->opc_counts.data();
  r.n_widths = (uint32_t)ctx->width_vals.size();
  r.width_values = ctx->width_vals.data();
  r.width_counts = ctx->width_counts.data();
  r.n_site_list = (uint32_t)ctx->site_ids.size();
  r.site_ids = ctx->site_ids.data();
  r.site_counts = ctx->site_counts.data();
  r.used_dense_table = ctx->dense;
  r.binned_accesses = ctx->binned;
  r.stream_checked = ctx->stream_checked;
  r.kernels_launched = ctx->kernels;
  r.d2h_bytes = ctx->d2h;
  if (ctx->timing) {
    for (int ph = 0; ph < AIWC_N_PHASES; ++ph) {
      float ms = 0.f;
      if (!(ctx->marked >> ph & 1u)) continue;
      if (cudaEventElapsedTime(&ms, ctx->ev[2 * ph], ctx->ev[2 * ph + 1]) == cudaSuccess) r.phase_ms[ph] = ms;
      else cudaGetLastError();
    }
  }
  *out = r;
  ctx->state = 2;

  // conservation (metrics.py:276-285)
  uint64_t opc_total = 0, w_total = 0;
  for (uint64_t c : ctx->opc_counts) opc_total += c;
  for (uint64_t c : ctx->width_counts) w_total += c;
  const char* bad = nullptr;
  if (opc_total != r.total_instructions) bad = "accumulator inconsistent: opcode counts != total instructions";
  else if (w_total != r.total_instructions) bad = "accumulator inconsistent: width samples != total instructions";
  else if (r.itb.sum != r.total_instructions) bad = "accumulator inconsistent: ITB samples do not cover all instructions";
  else if (r.ipt.sum != r.total_instructions) bad = "accumulator inconsistent: IPT samples do not cover all instructions";
  else if (r.ipt.n != r.work_items) bad = "accumulator inconsistent: one IPT sample per work-item expected";
  if (bad && !(ctx->opts.flags & AIWC_OPT_NO_CONSERVATION)) return fail(ctx, AIWC_ERR_INCONSISTENT, bad);
  if (ctx->opts.entry_cap && r.entries > ctx->opts.entry_cap && !ctx->comm) {
    fail(ctx, AIWC_ERR_TOO_LARGE, "trace state exceeds the in-memory cap");
    ctx->err.entries = ctx->opts.entry_cap + 1;
    ctx->err.cap = ctx->opts.entry_cap;
    return AIWC_ERR_TOO_LARGE;
  }
  return AIWC_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU: shard tables, owner partition, owned-key memory partials
// ---------------------------------------------------------------------------
namespace {

constexpr int PA_T = 256, PA_MAXR = 64, PA_ITEMS = 8;

__device__ __forceinline__ uint32_t owner_of(uint64_t addr, uint64_t base, uint32_t k, uint64_t kpr, uint32_t nranks) {
  const uint64_t o = ((addr - base) >> k) / kpr;
  return o < nranks ? (uint32_t)o : nranks - 1;
}

// per-owner totals of one address array
__global__ void partition_count_kernel(const uint64_t* __restrict__ a, uint64_t n, uint64_t base, uint32_t k,
                                       uint64_t kpr, uint32_t nranks, unsigned long long* counts) {
  __shared__ unsigned int h[PA_MAXR];
  for (int i = threadIdx.x; i < PA_MAXR; i += PA_T) h[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * PA_T + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PA_T)
    atomicAdd(&h[owner_of(a[i], base, k, kpr, nranks)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < (int)nranks; i += PA_T)
    if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

// owner-grouped copy: block-level reservation on per-owner cursors (order inside
// an owner's run is irrelevant -- the owner only counts addresses)
__global__ void partition_scatter_kernel(const uint64_t* __restrict__ a, uint64_t n, uint64_t base, uint32_t k,
                                         uint64_t kpr, uint32_t nranks, unsigned long long* cursor,
                                         uint64_t* __restrict__ out) {
  __shared__ unsigned int h[PA_MAXR];
  __shared__ unsigned long long b[PA_MAXR];
  for (uint64_t c0 = (uint64_t)blockIdx.x * PA_T * PA_ITEMS; c0 < n; c0 += (uint64_t)gridDim.x * PA_T * PA_ITEMS) {
    for (int i = threadIdx.x; i < PA_MAXR; i += PA_T) h[i] = 0;
    __syncthreads();
    uint32_t own[PA_ITEMS], slot[PA_ITEMS];
    uint64_t v[PA_ITEMS];
#pragma unroll
    for (int j = 0; j < PA_ITEMS; ++j) {
      const uint64_t i = c0 + (uint64_t)j * PA_T + threadIdx.x;
      own[j] = PA_MAXR;
      if (i < n) {
        v[j] = a[i];
        own[j] = owner_of(v[j], base, k, kpr, nranks);
        slot[j] = atomicAdd(&h[own[j]], 1u);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (int)nranks; i += PA_T)
      b[i] = h[i] ? atomicAdd(&cursor[i], (unsigned long long)h[i]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PA_ITEMS; ++j)
      if (own[j] < PA_MAXR) out[b[own[j]] + slot[j]] = v[j];
    __syncthreads();
  }
}

// owned-range hot window: the most frequent 1024-key block among 4096 sampled
// received addresses (>= 1/64 of them), else ~0 -- a block many ranks' accesses
// hit (shared scratch) would otherwise serialise as same-address REDs in L2
__global__ void __launch_bounds__(1024) owned_hot_sample_kernel(const uint64_t* __restrict__ a, uint64_t n,
                                                                uint64_t base, uint32_t k, uint64_t key_lo,
                                                                uint64_t n_keys, unsigned long long* hot_out,
                                                                uint32_t stride = 1, bool keys = false) {
  constexpr int SLOTS = 4096, PER = 4;
  __shared__ uint32_t hk[SLOTS], hc[SLOTS];
  __shared__ unsigned long long red[32];
  const int t = threadIdx.x;
  for (int i = t; i < SLOTS; i += 1024) { hk[i] = ~0u; hc[i] = 0; }
  __syncthreads();
  uint64_t v[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    uint64_t x = (uint64_t)(t * PER + j) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    x = (x ^ (x >> 31)) * 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    v[j] = n ? a[(x % n) * stride] : 0ull;
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const uint64_t key = (keys ? v[j] : (v[j] - base) >> k) - key_lo;
    if (!n || key >= n_keys) continue;
    const uint32_t blk = (uint32_t)(key >> 10);
    uint32_t h = (blk * 2654435761u) >> 20;
    for (int probe = 0; probe < 64; ++probe, h = (h + 1) & (SLOTS - 1)) {
      const uint32_t old = atomicCAS(&hk[h], ~0u, blk);
      if (old == ~0u || old == blk) { atomicAdd(&hc[h], 1u); break; }
    }
  }
  __syncthreads();
  unsigned long long best = 0;
  for (int i = t; i < SLOTS; i += 1024)
    if (hc[i]) best = max(best, ((unsigned long long)hc[i] << 32) | hk[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((t & 31) == 0) red[t >> 5] = best;
  __syncthreads();
  if (t == 0) {
    unsigned long long b = 0;
    for (int w = 0; w < 32; ++w) b = max(b, red[w]);
    const uint32_t cnt = (uint32_t)(b >> 32);
    *hot_out = (n >= (1u << 20) && cnt >= 64) ? (unsigned long long)(uint32_t)b << 10 : ~0ull;
  }
}

// owned-range dense table from received addresses (keys of the hot window are
// counted per CTA in shared memory and added once)
__global__ void fill_owned_kernel(const uint64_t* __restrict__ a, uint64_t n, unsigned long long inc, uint64_t base,
                                  uint32_t k, uint64_t key_lo, uint64_t n_keys, unsigned long long* __restrict__ tab,
                                  DevState* st, const unsigned long long* hot) {
  __shared__ uint32_t win[1024];
  const uint64_t hot_lo = *hot;
  const uint32_t hn = hot_lo == ~0ull ? 0u : 1024u;
  for (uint32_t i = threadIdx.x; i < hn; i += blockDim.x) win[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ((a[i] - base) >> k) - key_lo;
    if (key < n_keys) {
      const uint64_t rel = key - hot_lo;
      if (rel < hn) atomicAdd(&win[rel], 1u);
      else atomicAdd(&tab[key], inc);
    } else {
      atomicOr(&st->flags, (unsigned long long)F_SLOT_RANGE);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hn; i += blockDim.x)
    if (win[i]) atomicAdd(&tab[hot_lo + i], (unsigned long long)win[i] * inc);
}

// ---- run-length exchange (pre-aggregation on the sending rank) ----
// A run is a maximal stretch of one compacted address array whose keys go up by
// one with a single owner (streaming traces: a whole shard is a few runs),
// capped at RUN_MAX keys.  It travels as two words: global key, length | write << 63.
constexpr int RN_T = 256, RN_I = 8, RN_TILE = RN_T * RN_I;
constexpr uint64_t RUN_MAX = 1ull << 16;

// run heads of one tile, warp-contiguous (element warp_base + 32 j + lane, all loads
// coalesced; the predecessor comes from the neighbouring lane): bit j of the
// returned ballot word hm[j] marks lane `lane`'s element j as a head
__device__ __forceinline__ void tile_heads(const uint64_t* __restrict__ a, uint64_t n, uint64_t base, uint32_t k,
                                           uint64_t kpr, uint32_t nranks, uint32_t (&hm)[RN_I]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wb = (uint64_t)blockIdx.x * RN_TILE + (uint64_t)warp * 32 * RN_I;
  uint64_t v[RN_I];
#pragma unroll
  for (int j = 0; j < RN_I; ++j) {
    const uint64_t i = wb + 32 * j + lane;
    v[j] = i < n ? __ldcs(a + i) : 0ull;
  }
  uint64_t prev_last = (wb && wb - 1 < n) ? a[wb - 1] : 0ull;  // element before the warp's first
#pragma unroll
  for (int j = 0; j < RN_I; ++j) {
    const uint64_t i = wb + 32 * j + lane;
    uint64_t p = __shfl_up_sync(0xffffffffu, v[j], 1);
    const uint64_t last_prev_row = __shfl_sync(0xffffffffu, j ? v[j - 1] : prev_last, 31);
    if (lane == 0) p = last_prev_row;
    bool h = false;
    if (i < n) {
      if (i == 0 || (i & (RUN_MAX - 1)) == 0) {
        h = true;
      } else {
        const uint64_t k1 = (v[j] - base) >> k, k0 = (p - base) >> k;
        h = k1 != k0 + 1;
        for (uint32_t o = 1; o < nranks && !h; ++o) h = k1 == (uint64_t)o * kpr;
      }
    }
    hm[j] = __ballot_sync(0xffffffffu, h);
  }
}

// heads per tile
__global__ void __launch_bounds__(RN_T) run_count_kernel(const uint64_t* __restrict__ a, uint64_t n, uint64_t base,
                                                          uint32_t k, uint64_t kpr, uint32_t nranks,
                                                          uint32_t* __restrict__ blk) {
  __shared__ uint32_t ws[RN_T / 32];
  uint32_t hm[RN_I];
  tile_heads(a, n, base, k, kpr, nranks, hm);
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < RN_I; ++j) c += __popc(hm[j]);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < RN_T / 32; ++w) t += ws[w];
    blk[blockIdx.x] = t;
  }
}

// head indices in stream order (blk holds the exclusive scan of the tile counts)
__global__ void __launch_bounds__(RN_T) run_pos_kernel(const uint64_t* __restrict__ a, uint64_t n, uint64_t base,
                                                        uint32_t k, uint64_t kpr, uint32_t nranks,
                                                        const uint32_t* __restrict__ blk, uint64_t* __restrict__ pos) {
  __shared__ uint32_t ws[RN_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t hm[RN_I];
  tile_heads(a, n, base, k, kpr, nranks, hm);
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < RN_I; ++j) c += __popc(hm[j]);
  if (lane == 0) ws[warp] = c;
  __syncthreads();
  uint32_t o = blk[blockIdx.x];
  for (int w = 0; w < warp; ++w) o += ws[w];
  const uint64_t wb = (uint64_t)blockIdx.x * RN_TILE + (uint64_t)warp * 32 * RN_I;
#pragma unroll
  for (int j = 0; j < RN_I; ++j) {
    if ((hm[j] >> lane) & 1u) pos[o + __popc(hm[j] & ((1u << lane) - 1u))] = wb + 32 * j + lane;
    o += __popc(hm[j]);
  }
}

// runs per owner (pass 0) / owner-grouped runs (pass 1, cursors hold the offsets)
__global__ void run_emit_kernel(const uint64_t* __restrict__ a, uint64_t n, const uint64_t* __restrict__ pos,
                                uint64_t n_runs, uint64_t base, uint32_t k, uint64_t kpr, uint32_t nranks,
                                unsigned long long wflag, int pass, unsigned long long* cursor,
                                uint64_t* __restrict__ out) {
  // whole warps iterate together; a warp whose runs share one owner (the common
  // case) reserves its slots with a single atomic
  const int lane = threadIdx.x & 31;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n_pad = (n_runs + 31) & ~31ull;
  for (uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; h < n_pad; h += T) {
    const bool valid = h < n_runs;
    uint64_t st = 0, en = 0;
    uint32_t o = PA_MAXR;
    if (valid) {
      st = pos[h];
      en = h + 1 < n_runs ? pos[h + 1] : n;
      o = owner_of(a[st], base, k, kpr, nranks);
    }
    const uint32_t o0 = __shfl_sync(0xffffffffu, o, 0);
    const uint32_t vm = __ballot_sync(0xffffffffu, valid);
    unsigned long long slot = 0;
    if (__all_sync(0xffffffffu, !valid || o == o0)) {
      unsigned long long b = 0;
      if (lane == 0 && vm) b = atomicAdd(&cursor[o0], (unsigned long long)__popc(vm));
      slot = __shfl_sync(0xffffffffu, b, 0) + __popc(vm & ((1u << lane) - 1u));
    } else if (valid) {
      slot = atomicAdd(&cursor[o], 1ull);
    }
    if (pass == 1 && valid) {
      out[2 * slot] = (a[st] - base) >> k;
      out[2 * slot + 1] = (en - st) | wflag;
    }
  }
}

// owned-range dense table from runs: one warp per run; keys of the hot window
// are counted per CTA in shared memory
__global__ void apply_runs_kernel(const uint64_t* __restrict__ runs, uint64_t n_runs, uint64_t key_lo,
                                  uint64_t n_keys, unsigned long long* __restrict__ tab, DevState* st,
                                  const unsigned long long* hot) {
  __shared__ uint32_t win[2][1024];
  const uint64_t hot_lo = *hot;
  const uint32_t hn = hot_lo == ~0ull ? 0u : 1024u;
  for (uint32_t i = threadIdx.x; i < 2 * hn; i += blockDim.x) (&win[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_runs; r += nw) {
    const uint64_t key = runs[2 * r] - key_lo, lw = runs[2 * r + 1];
    const uint64_t len = lw & 0xFFFFFFFFull;
    const uint32_t w = (uint32_t)(lw >> 63);
    if (key >= n_keys || len > n_keys - key) {
      if (lane == 0) atomicOr(&st->flags, (unsigned long long)F_SLOT_RANGE);
      continue;
    }
    for (uint64_t i = lane; i < len; i += 32) {
      const uint64_t rel = key + i - hot_lo;
      if (rel < hn) atomicAdd(&win[w][rel], 1u);
      else atomicAdd(&tab[key + i], w ? (1ull << 32) : 1ull);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hn; i += blockDim.x)
    if (win[0][i] | win[1][i])
      atomicAdd(&tab[hot_lo + i], (unsigned long long)win[0][i] | ((unsigned long long)win[1][i] << 32));
}

}  // namespace

extern "C" int aiwc_shard_tables_get(aiwc_ctx* ctx, aiwc_shard_tables* out) {
  if (!ctx || !out) return AIWC_ERR_ARGUMENT;
  if (!(ctx->opts.flags & AIWC_OPT_SHARD) || ctx->state != 2)
    return fail(ctx, AIWC_ERR_ARGUMENT, "shard tables need a shard ctx after aiwc_finalize");
  aiwc_shard_tables t{};
  t.itb_hist = reinterpret_cast<const uint64_t*>(ctx->h_state->itb_hist);
  t.ipt_hist = reinterpret_cast<const uint64_t*>(ctx->h_state->ipt_hist);
  t.n_itb_ovf = ctx->itb_ovf_sorted.size(); t.itb_ovf = ctx->itb_ovf_sorted.data();
  t.n_ipt_ovf = ctx->ipt_ovf_sorted.size(); t.ipt_ovf = ctx->ipt_ovf_sorted.data();
  t.branch_table_size = (uint32_t)ctx->branch_tab_host.size();
  t.branch_table = ctx->branch_tab_host.data();
  t.width_first = ctx->width_firsts.data();
  const DevState& h = *ctx->h_state;
  t.addr_stats[0] = h.addr_min; t.addr_stats[1] = h.addr_max; t.addr_stats[2] = h.addr_and; t.addr_stats[3] = h.addr_or;
  t.rd_dev = P<uint64_t>(ctx->rd); t.wr_dev = P<uint64_t>(ctx->wr);
  *out = t;
  return AIWC_OK;
}

extern "C" int aiwc_partition_addresses(aiwc_ctx* ctx, uint64_t base, uint32_t k, uint64_t keys_per_rank,
                                        uint32_t nranks, uint64_t** reads_dev, uint64_t** writes_dev,
                                        uint64_t* counts, void* stream) {
  if (!ctx || !reads_dev || !writes_dev || !counts || nranks == 0 || nranks > (uint32_t)PA_MAXR || keys_per_rank == 0)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad partition arguments");
  if (!(ctx->opts.flags & AIWC_OPT_SHARD) || ctx->state != 2)
    return fail(ctx, AIWC_ERR_ARGUMENT, "partition needs a shard ctx after aiwc_finalize");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->part_entries, std::max<uint64_t>(ctx->n_rd + ctx->n_wr, 1) * 8));
  CK(grow(ctx->part_cursor, 2 * PA_MAXR * 8));
  unsigned long long* cur = P<unsigned long long>(ctx->part_cursor);
  CK(cudaMemsetAsync(cur, 0, 2 * PA_MAXR * 8, s));
  const uint64_t* src[2] = {P<uint64_t>(ctx->rd), P<uint64_t>(ctx->wr)};
  const uint64_t len[2] = {ctx->n_rd, ctx->n_wr};
  auto blocks = [&](uint64_t n) {
    return (uint32_t)std::min<uint64_t>(std::max<uint64_t>((n + PA_T * PA_ITEMS - 1) / (PA_T * PA_ITEMS), 1),
                                        (uint64_t)ctx->n_sms * 8);
  };
  for (int q = 0; q < 2; ++q)
    if (len[q]) partition_count_kernel<<<blocks(len[q]), PA_T, 0, s>>>(src[q], len[q], base, k, keys_per_rank, nranks,
                                                                       cur + q * PA_MAXR);
  std::vector<unsigned long long> c(2 * PA_MAXR, 0);
  CK(cudaMemcpyAsync(c.data(), cur, 2 * PA_MAXR * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<unsigned long long> off(2 * PA_MAXR, 0);
  for (int q = 0; q < 2; ++q) {
    unsigned long long run = q ? ctx->n_rd : 0;  // reads first, then writes
    for (uint32_t i = 0; i < nranks; ++i) {
      off[q * PA_MAXR + i] = run;
      run += c[q * PA_MAXR + i];
      counts[q * nranks + i] = c[q * PA_MAXR + i];
    }
  }
  CK(cudaMemcpyAsync(cur, off.data(), 2 * PA_MAXR * 8, cudaMemcpyHostToDevice, s));
  for (int q = 0; q < 2; ++q)
    if (len[q]) partition_scatter_kernel<<<blocks(len[q]), PA_T, 0, s>>>(src[q], len[q], base, k, keys_per_rank,
                                                                         nranks, cur + q * PA_MAXR,
                                                                         P<uint64_t>(ctx->part_entries));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  *reads_dev = P<uint64_t>(ctx->part_entries);
  *writes_dev = P<uint64_t>(ctx->part_entries) + ctx->n_rd;
  return AIWC_OK;
}

// the owner's statistics back to the host (both owner entry points)
static int owned_result(aiwc_ctx* ctx, DevState* st, uint64_t m, uint32_t launched, aiwc_memory_part* out,
                        cudaStream_t s) {
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ctx->h_state, st, offsetof(DevState, host_end), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const DevState& h = *ctx->h_state;
  if (h.flags & F_SLOT_RANGE) return fail(ctx, AIWC_ERR_ARGUMENT, "received address outside the owned key range");
  ctx->mp_hist0.assign(h.cnt_hist0, h.cnt_hist0 + CBINS);
  ctx->mp_big.resize(h.lvl0_ovf_n);
  if (h.lvl0_ovf_n) {
    CK(cudaMemcpyAsync(ctx->mp_big.data(), ctx->mp_ovf.p, h.lvl0_ovf_n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  aiwc_memory_part r{};
  r.unique_reads = h.unique_r; r.unique_writes = h.unique_w; r.footprint = h.footprint;
  for (int i = 0; i < NLEVELS; ++i) r.level_sum[i] = m ? -h.entropy[i] : 0.0;
  r.cnt_hist0 = ctx->mp_hist0.data();
  r.n_big = ctx->mp_big.size();
  r.big = ctx->mp_big.data();
  r.kernels_launched = launched;
  *out = r;
  return AIWC_OK;
}

extern "C" int aiwc_partition_runs(aiwc_ctx* ctx, uint64_t base, uint32_t k, uint64_t keys_per_rank,
                                   uint32_t nranks, uint64_t** runs_dev, uint64_t* counts, void* stream) {
  if (!ctx || !runs_dev || !counts || nranks == 0 || nranks > (uint32_t)PA_MAXR || keys_per_rank == 0)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad partition arguments");
  if (!(ctx->opts.flags & AIWC_OPT_SHARD) || ctx->state != 2)
    return fail(ctx, AIWC_ERR_ARGUMENT, "partition needs a shard ctx after aiwc_finalize");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  const uint64_t* src[2] = {P<uint64_t>(ctx->rd), P<uint64_t>(ctx->wr)};
  const uint64_t len[2] = {ctx->n_rd, ctx->n_wr};
  CK(grow(ctx->run_pos, std::max<uint64_t>(ctx->n_rd + ctx->n_wr, 1) * 8));
  CK(grow(ctx->part_cursor, 2 * PA_MAXR * 8));
  uint64_t* pos = P<uint64_t>(ctx->run_pos);
  uint64_t nrun[2] = {0, 0};
  for (int q = 0; q < 2; ++q) {
    if (!len[q]) continue;
    const uint64_t nb = (len[q] + RN_TILE - 1) / RN_TILE;
    CK(grow(ctx->run_blk, (nb + 1) * 4));
    CK(grow(ctx->run_scan, (scan_scratch_elems(nb) + 16) * 4));
    uint32_t* blk = P<uint32_t>(ctx->run_blk);
    run_count_kernel<<<(unsigned)nb, RN_T, 0, s>>>(src[q], len[q], base, k, keys_per_rank, nranks, blk);
    scan_exclusive_u32(blk, nb, P<uint32_t>(ctx->run_scan), blk + nb, s, nullptr);
    uint32_t tot = 0;
    CK(cudaMemcpyAsync(&tot, blk + nb, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    nrun[q] = tot;
    run_pos_kernel<<<(unsigned)nb, RN_T, 0, s>>>(src[q], len[q], base, k, keys_per_rank, nranks, blk,
                                                pos + (q ? nrun[0] : 0));
  }
  const uint64_t R = nrun[0] + nrun[1];
  CK(grow(ctx->part_entries, std::max<uint64_t>(R, 1) * 16));
  unsigned long long* cur = P<unsigned long long>(ctx->part_cursor);
  CK(cudaMemsetAsync(cur, 0, PA_MAXR * 8, s));
  auto grid = [&](uint64_t n) { return (unsigned)std::min<uint64_t>(std::max<uint64_t>((n + 255) / 256, 1), 148 * 16); };
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      std::vector<unsigned long long> c(PA_MAXR, 0), off(PA_MAXR, 0);
      CK(cudaMemcpyAsync(c.data(), cur, PA_MAXR * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      unsigned long long run = 0;
      for (uint32_t o = 0; o < nranks; ++o) { off[o] = run; run += c[o]; counts[o] = c[o]; }
      CK(cudaMemcpyAsync(cur, off.data(), PA_MAXR * 8, cudaMemcpyHostToDevice, s));
    }
    for (int q = 0; q < 2; ++q)
      if (nrun[q])
        run_emit_kernel<<<grid(nrun[q]), 256, 0, s>>>(src[q], len[q], pos + (q ? nrun[0] : 0), nrun[q], base, k,
                                                     keys_per_rank, nranks, q ? (1ull << 63) : 0ull, pass, cur,
                                                     P<uint64_t>(ctx->part_entries));
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  *runs_dev = P<uint64_t>(ctx->part_entries);
  return AIWC_OK;
}

extern "C" int aiwc_memory_partial_runs(aiwc_ctx* ctx, const uint64_t* runs, uint64_t n_runs, uint32_t k,
                                        uint64_t key_lo, uint64_t n_keys, uint64_t total_m, aiwc_memory_part* out,
                                        void* stream) {
  if (!ctx || !out || (n_runs && !runs) || (key_lo & 1023) || k > 32)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad memory partial");
  if (n_keys * 8 > ctx->opts.dense_budget_bytes)
    return fail(ctx, AIWC_ERR_UNSUPPORTED, "owned key range exceeds the dense-table budget");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->mp_state, sizeof(DevState)));
  DevState* st = P<DevState>(ctx->mp_state);
  init_state_kernel<<<64, 256, 0, s>>>(st);
  uint32_t launched = 1;
  const uint64_t tm = std::max<uint64_t>(total_m, 1);
  CK(grow(ctx->mp_ovf, (tm / CBINS + 2) * 8));
  if (n_runs) {
    CK(grow(ctx->mp_tab, std::max<uint64_t>(n_keys, 1) * 8));
    CK(cudaMemsetAsync(ctx->mp_tab.p, 0, std::max<uint64_t>(n_keys, 1) * 8, s));
    owned_hot_sample_kernel<<<1, 1024, 0, s>>>(runs, n_runs, 0, 0, key_lo, n_keys, &st->hot_key, 2, true);
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((n_runs + 7) / 8, (uint64_t)ctx->n_sms * 8);
    apply_runs_kernel<<<blocks, 256, 0, s>>>(runs, n_runs, key_lo, n_keys, P<unsigned long long>(ctx->mp_tab), st,
                                             &st->hot_key);
    const uint32_t nct = (uint32_t)std::min<uint64_t>((n_keys + 1023) / 1024, ctx->n_parts);
    launch_dense_stats(ctx->mp_tab.p, false, n_keys, k, tm, st, P<double>(ctx->partials), nct,
                       P<uint64_t>(ctx->mp_ovf), s);
    launch_entropy_finish(st, P<double>(ctx->partials), nct, tm, k, s);
    launched += 4;
  }
  return owned_result(ctx, st, n_runs, launched, out, s);
}

extern "C" int aiwc_memory_partial(aiwc_ctx* ctx, const uint64_t* rd, uint64_t n_rd, const uint64_t* wr, uint64_t n_wr,
                                   uint64_t base, uint32_t k, uint64_t key_lo, uint64_t n_keys, uint64_t total_m,
                                   aiwc_memory_part* out, void* stream) {
  if (!ctx || !out || (n_rd && !rd) || (n_wr && !wr) || (key_lo & 1023) || k > 32)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad memory partial");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->mp_state, sizeof(DevState)));
  DevState* st = P<DevState>(ctx->mp_state);
  init_state_kernel<<<64, 256, 0, s>>>(st);
  uint32_t launched = 1;
  const uint64_t m = n_rd + n_wr, tm = std::max<uint64_t>(total_m, 1);
  CK(grow(ctx->mp_ovf, (tm / CBINS + 2) * 8));
  const bool dense = n_keys * 8 <= ctx->opts.dense_budget_bytes && n_keys <= 4 * m + (1ull << 20);
  if (m && dense) {
    CK(grow(ctx->mp_tab, std::max<uint64_t>(n_keys, 1) * 8));
    CK(cudaMemsetAsync(ctx->mp_tab.p, 0, std::max<uint64_t>(n_keys, 1) * 8, s));
    const uint64_t* src[2] = {rd, wr};
    const uint64_t len[2] = {n_rd, n_wr};
    for (int q = 0; q < 2; ++q)
      if (len[q]) {
        const uint32_t blocks = (uint32_t)std::min<uint64_t>((len[q] + 255) / 256, (uint64_t)ctx->n_sms * 8);
        owned_hot_sample_kernel<<<1, 1024, 0, s>>>(src[q], len[q], base, k, key_lo, n_keys, &st->hot_key);
        fill_owned_kernel<<<blocks, 256, 0, s>>>(src[q], len[q], q ? (1ull << 32) : 1ull, base, k, key_lo, n_keys,
                                                 P<unsigned long long>(ctx->mp_tab), st, &st->hot_key);
        launched += 2;
      }
    const uint32_t nct = (uint32_t)std::min<uint64_t>((n_keys + 1023) / 1024, ctx->n_parts);
    launch_dense_stats(ctx->mp_tab.p, false, n_keys, k, tm, st, P<double>(ctx->partials), nct,
                       P<uint64_t>(ctx->mp_ovf), s);
    launch_entropy_finish(st, P<double>(ctx->partials), nct, tm, k, s);
    launched += 2;
  } else if (m) {
    // sort path over the received addresses with the global base / k
    AddrMap am{};
    am.base = base; am.k = k;
    const uint64_t hi_key = key_lo + (n_keys ? n_keys - 1 : 0);
    am.hi = base + (hi_key << k);
    const bool raw = bitwidth64(hi_key) > 63;
    CK(grow(ctx->sparse_scr, sparse_scratch_bytes(m)));
    const uint32_t parts = std::min<uint32_t>(ctx->n_parts, 256);
    launched += sparse_memory_stats(rd, n_rd, wr, n_wr, am, tm, st, P<double>(ctx->partials), parts,
                                    P<uint64_t>(ctx->mp_ovf), ctx->sparse_scr.p, ctx->sparse_scr.cap, s);
    launch_entropy_finish(st, P<double>(ctx->partials), parts, tm, raw ? 64u : k, s);
    launched += 1;
  }
  return owned_result(ctx, st, m, launched, out, s);
}


// ---------------------------------------------------------------------------
// multi-GPU dense exchange (aiwc_exchange.cu)
// ---------------------------------------------------------------------------
extern "C" int aiwc_shard_prepare(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload,
                                  const aiwc_trace_info* info, aiwc_shard_stats* local, void* stream) {
  if (!ctx || !info || !local) return AIWC_ERR_ARGUMENT;
  if (!(ctx->opts.flags & AIWC_OPT_SHARD)) return fail(ctx, AIWC_ERR_ARGUMENT, "aiwc_shard_prepare needs a shard ctx");
  const int rc = ingest_begin(ctx, kind, payload, info, stream);
  if (rc) return rc;
  const bool own = ctx->pend.with_stats;
  const DevState& h = *ctx->h_state;
  aiwc_shard_stats l{};
  l.n_accesses = ctx->n_rd + ctx->n_wr;
  if (l.n_accesses) {
    l.addr_min = own ? h.addr_min : info->addr_min; l.addr_max = own ? h.addr_max : info->addr_max;
    l.addr_and = own ? h.addr_and : info->addr_and; l.addr_or = own ? h.addr_or : info->addr_or;
  } else {
    l.addr_min = ~0ull; l.addr_max = 0; l.addr_and = ~0ull; l.addr_or = 0;
  }
  l.dense_budget_bytes = ctx->opts.dense_budget_bytes;
  l.n_branches = ctx->n_br;
  *local = l;
  ctx->state = 3;
  return AIWC_OK;
}

extern "C" int aiwc_shard_ingest(aiwc_ctx* ctx, const aiwc_shard_stats* job, uint32_t* dense, void* stream) {
  if (!ctx || !job || !dense) return AIWC_ERR_ARGUMENT;
  if (ctx->state != 3) return fail(ctx, AIWC_ERR_ARGUMENT, "aiwc_shard_ingest needs aiwc_shard_prepare first");
  if (job->n_accesses < ctx->n_rd + ctx->n_wr || (job->n_accesses && job->addr_min > job->addr_max))
    return fail(ctx, AIWC_ERR_ARGUMENT, "job statistics do not cover this shard");
  const uint64_t budget = ctx->opts.dense_budget_bytes;
  ctx->opts.dense_budget_bytes = std::min<uint64_t>(budget, job->dense_budget_bytes);  // every rank decides alike
  const int rc = ingest_finish(ctx, job->addr_min, job->addr_max, job->addr_and, job->addr_or, job->n_accesses, true,
                               stream);
  ctx->opts.dense_budget_bytes = budget;
  if (rc) return rc;
  *dense = ctx->shard_dense ? 1u : 0u;
  return AIWC_OK;
}

extern "C" int aiwc_shard_chunks(aiwc_ctx* ctx, uint32_t** bits, uint64_t* n_words) {
  if (!ctx || !bits || !n_words) return AIWC_ERR_ARGUMENT;
  if (!ctx->shard_dense || ctx->state != 2)
    return fail(ctx, AIWC_ERR_ARGUMENT, "chunk bitmap needs a dense shard ingest and aiwc_finalize");
  *bits = P<uint32_t>(ctx->chunk_bits);
  *n_words = ctx->n_chunk_words;
  return AIWC_OK;
}

extern "C" int aiwc_shard_pack(aiwc_ctx* ctx, const uint32_t* all_bits, uint32_t rank, uint32_t nranks,
                               uint64_t** runs_dev, uint64_t* counts, void* stream) {
  if (!ctx || !all_bits || !runs_dev || !counts || nranks == 0 || rank >= nranks || nranks > (uint32_t)PA_MAXR)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad pack arguments");
  if (!ctx->shard_dense || ctx->state != 2) return fail(ctx, AIWC_ERR_ARGUMENT, "pack needs a dense shard ingest");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->part_cursor, PA_MAXR * 8));
  unsigned long long* cur = P<unsigned long long>(ctx->part_cursor);
  CK(cudaMemsetAsync(cur, 0, PA_MAXR * 8, s));
  const uint64_t words = ctx->n_chunk_words;
  ctx->kernels += launch_pack(ctx->dtab.p, ctx->dense32, all_bits, words, rank, nranks, 0, cur, nullptr,
                              (uint32_t)ctx->n_sms, s);
  std::vector<unsigned long long> c(PA_MAXR, 0), off(PA_MAXR, 0);
  CK(cudaMemcpyAsync(c.data(), cur, PA_MAXR * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  unsigned long long tot = 0;
  for (uint32_t o = 0; o < nranks; ++o) { off[o] = tot; tot += c[o]; counts[o] = c[o]; }
  CK(grow(ctx->part_entries, std::max<uint64_t>(tot, 1) * 16));
  if (tot) {
    CK(cudaMemcpyAsync(cur, off.data(), PA_MAXR * 8, cudaMemcpyHostToDevice, s));
    ctx->kernels += launch_pack(ctx->dtab.p, ctx->dense32, all_bits, words, rank, nranks, 1, cur,
                                P<uint64_t>(ctx->part_entries), (uint32_t)ctx->n_sms, s);
  }
  CK(cudaGetLastError());
  *runs_dev = P<uint64_t>(ctx->part_entries);
  return AIWC_OK;
}

extern "C" int aiwc_shard_owned(aiwc_ctx* ctx, const uint64_t* runs, uint64_t n_runs, const uint32_t* all_bits,
                                uint32_t rank, uint32_t nranks, uint64_t total_m, aiwc_memory_part* out, void* stream) {
  if (!ctx || !out || !all_bits || (n_runs && !runs) || nranks == 0 || rank >= nranks)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad owned-statistics arguments");
  if (!ctx->shard_dense || ctx->state != 2) return fail(ctx, AIWC_ERR_ARGUMENT, "owned statistics need a dense shard");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->mp_state, sizeof(DevState)));
  DevState* st = P<DevState>(ctx->mp_state);
  init_state_kernel<<<64, 256, 0, s>>>(st);
  uint32_t launched = 1;
  const uint64_t tm = std::max<uint64_t>(total_m, 1);
  CK(grow(ctx->mp_ovf, (tm / CBINS + 2) * 8));
  const uint64_t words = ctx->n_chunk_words;
  const uint64_t n_keys = ctx->am.n_keys;
  launched += launch_apply_runs(ctx->dtab.p, ctx->dense32, runs, n_runs, n_keys, all_bits, words, rank, nranks,
                                &st->flags, (uint32_t)ctx->n_sms, s);
  const uint32_t nct = (uint32_t)std::min<uint64_t>((n_keys + 1023) / 1024, ctx->n_parts);
  launch_dense_stats(ctx->dtab.p, ctx->dense32, n_keys, ctx->am.k, tm, st, P<double>(ctx->partials), nct,
                     P<uint64_t>(ctx->mp_ovf), s, all_bits, words, rank, nranks);
  launch_entropy_finish(st, P<double>(ctx->partials), nct, tm, ctx->am.k, s);
  // the table is clean again: zero what this rank wrote, reset its bitmap
  launched += 2 + launch_clear_chunks(ctx->dtab.p, ctx->dense32, dense_alloc_keys(n_keys), all_bits, words, rank,
                                      nranks, P<uint32_t>(ctx->chunk_bits), (uint32_t)ctx->n_sms, s);
  ctx->dtab_clean = ctx->dtab.cap;
  return owned_result(ctx, st, total_m, launched, out, s);
}

// ---------------------------------------------------------------------------
// accumulator state export and state merges (merge_accumulators, metrics.py:235-270)
// ---------------------------------------------------------------------------
extern "C" int aiwc_state_export(aiwc_ctx* ctx, aiwc_state* out) {
  if (!ctx || !out) return AIWC_ERR_ARGUMENT;
  if (ctx->state != 2 || !ctx->info.export_state)
    return fail(ctx, AIWC_ERR_ARGUMENT, "state export needs info.export_state and aiwc_finalize");
  aiwc_state o{};
  o.exported = ctx->state_ok || !(ctx->n_rd + ctx->n_wr);
  o.n_runs = ctx->state_ok ? ctx->state_n_runs : 0;
  o.runs_dev = P<uint64_t>(ctx->state_runs);
  o.base = ctx->am.base; o.low_const = ctx->am.low_const; o.k = ctx->am.k;
  for (int i = 0; i < 4; ++i) o.addr_stats[i] = ctx->stats4[i];
  o.itb_hist = reinterpret_cast<const uint64_t*>(ctx->h_state->itb_hist);
  o.ipt_hist = reinterpret_cast<const uint64_t*>(ctx->h_state->ipt_hist);
  o.n_itb_ovf = ctx->itb_ovf_sorted.size(); o.itb_ovf = ctx->itb_ovf_sorted.data();
  o.n_ipt_ovf = ctx->ipt_ovf_sorted.size(); o.ipt_ovf = ctx->ipt_ovf_sorted.data();
  o.branch_table_size = (uint32_t)ctx->branch_tab_host.size();
  o.branch_table = ctx->branch_tab_host.data();
  o.width_first = ctx->width_firsts.data();
  *out = o;
  return AIWC_OK;
}

extern "C" int aiwc_memory_merge(aiwc_ctx* ctx, const aiwc_runs_part* parts, uint32_t n_parts, const uint64_t* stats,
                                 uint64_t total_m, aiwc_memory_part* out, void* stream) {
  if (!ctx || !out || !stats || (n_parts && !parts)) return AIWC_ERR_ARGUMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  CK(grow(ctx->mp_state, sizeof(DevState)));
  DevState* st = P<DevState>(ctx->mp_state);
  init_state_kernel<<<64, 256, 0, s>>>(st);
  uint32_t launched = 1;
  if (!total_m) return owned_result(ctx, st, 0, launched, out, s);
  // the merged key map by the engine's rule (aiwc_ingest's decide_memory)
  const uint64_t base = stats[0] & ~1023ull, vary = stats[2] ^ stats[3];
  const uint32_t k = vary ? std::min<uint32_t>((uint32_t)__builtin_ctzll(vary), 32u) : 0u;
  const uint64_t span = (stats[1] - base) >> k, n_keys = span + 1;
  if (span >= DENSE_MAX_KEYS - 1 || n_keys * 8 > ctx->opts.dense_budget_bytes || n_keys > 4 * total_m + (1ull << 20))
    return fail(ctx, AIWC_ERR_UNSUPPORTED, "merged address span does not fit a dense table");
  const uint64_t tm = total_m;
  CK(grow(ctx->mp_ovf, (tm / CBINS + 2) * 8));
  CK(grow(ctx->mp_tab, n_keys * 8));
  CK(cudaMemsetAsync(ctx->mp_tab.p, 0, n_keys * 8, s));
  for (uint32_t i = 0; i < n_parts; ++i) {
    launch_merge_apply(parts[i].runs_dev, parts[i].n_runs, parts[i].base, parts[i].low_const, parts[i].k, base, k, n_keys,
                       P<unsigned long long>(ctx->mp_tab), &st->flags, (uint32_t)ctx->n_sms, s);
    launched += parts[i].n_runs ? 1 : 0;
  }
  const uint32_t nct = (uint32_t)std::min<uint64_t>((n_keys + 1023) / 1024, ctx->n_parts);
  launch_dense_stats(ctx->mp_tab.p, false, n_keys, k, tm, st, P<double>(ctx->partials), nct, P<uint64_t>(ctx->mp_ovf), s);
  launch_entropy_finish(st, P<double>(ctx->partials), nct, tm, k, s);
  launched += 2;
  return owned_result(ctx, st, tm, launched, out, s);
}

// ---------------------------------------------------------------------------
// job mode: NCCL in the engine (aiwc_ctx_set_comm).  aiwc_ingest takes this
// rank's work-group shard, aiwc_finalize returns the whole job's result on every
// rank; every collective is an NCCL call on the caller's stream, with no Python
// between them (SURVEY.md §8b aiwc_ctx_set_comm, §8e).
// ---------------------------------------------------------------------------
#define NC(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      char m_[200];                                                                     \
      snprintf(m_, sizeof m_, "%s: %s", #call, ncclGetErrorString(r_));                 \
      return fail(ctx, AIWC_ERR_NCCL, m_);                                              \
    }                                                                                   \
  } while (0)

extern "C" int aiwc_nccl_unique_id(void* id_out) {
  if (!id_out) return AIWC_ERR_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AIWC_ERR_NCCL;
  memcpy(id_out, &id, sizeof id);
  return AIWC_OK;
}

extern "C" int aiwc_ctx_set_comm(aiwc_ctx* ctx, const void* id, int rank, int nranks) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks || nranks > PA_MAXR)
    return fail(ctx, AIWC_ERR_ARGUMENT, "bad communicator arguments");
  if (ctx->comm) return fail(ctx, AIWC_ERR_ARGUMENT, "ctx already has a communicator");
  CK(cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  NC(ncclCommInitRank(&ctx->comm, nranks, uid, rank));
  ctx->rank = (uint32_t)rank;
  ctx->nranks = (uint32_t)nranks;
  ctx->opts.flags |= AIWC_OPT_SHARD;  // memory statistics come from the job's exchange
  return AIWC_OK;
}

// all-gather of n u64 per rank through device memory: out = [nranks][n] on the host
static int job_allgather_u64(aiwc_ctx* ctx, const uint64_t* mine, size_t n, std::vector<uint64_t>& out,
                             cudaStream_t s) {
  const size_t R = ctx->nranks;
  CK(grow(ctx->nc_small, (R + 1) * n * 8));
  uint64_t* d = P<uint64_t>(ctx->nc_small);
  CK(cudaMemcpyAsync(d + R * n, mine, n * 8, cudaMemcpyHostToDevice, s));
  NC(ncclAllGather(d + R * n, d, n, ncclUint64, ctx->comm, s));
  out.resize(R * n);
  CK(cudaMemcpyAsync(out.data(), d, R * n * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AIWC_OK;
}

// second half of a job-mode ingest: the job's statistics from every rank's, then
// the ingest with the job's key map (a dense table when it fits on every rank)
static int job_ingest(aiwc_ctx* ctx, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const aiwc_trace_info* info = &ctx->info;
  const bool own = ctx->pend.with_stats;
  const DevState& h = *ctx->h_state;
  uint64_t l[7];
  l[4] = ctx->n_rd + ctx->n_wr;
  if (l[4]) {
    l[0] = own ? h.addr_min : info->addr_min; l[1] = own ? h.addr_max : info->addr_max;
    l[2] = own ? h.addr_and : info->addr_and; l[3] = own ? h.addr_or : info->addr_or;
  } else {
    l[0] = ~0ull; l[1] = 0; l[2] = ~0ull; l[3] = 0;
  }
  l[5] = ctx->opts.dense_budget_bytes;
  l[6] = ctx->n_br;
  std::vector<uint64_t> all;
  int rc = job_allgather_u64(ctx, l, 7, all, s);
  if (rc) return rc;
  uint64_t* j = ctx->job;
  j[0] = ~0ull; j[1] = 0; j[2] = ~0ull; j[3] = 0; j[4] = 0; j[5] = ~0ull; j[6] = 0;
  for (uint32_t r = 0; r < ctx->nranks; ++r) {
    const uint64_t* x = &all[7 * r];
    if (x[4]) { j[0] = std::min(j[0], x[0]); j[1] = std::max(j[1], x[1]); j[2] &= x[2]; j[3] |= x[3]; }
    j[4] += x[4]; j[5] = std::min(j[5], x[5]); j[6] += x[6];
  }
  const uint64_t budget = ctx->opts.dense_budget_bytes;
  ctx->opts.dense_budget_bytes = j[5];  // every rank decides alike
  rc = ingest_finish(ctx, j[0], j[1], j[2], j[3], j[4], true, stream);
  ctx->opts.dense_budget_bytes = budget;
  return rc;
}

// runs / addresses to their owners: send counts[o] u64 words to rank o, receive
// into ctx->nc_recv; *n_recv = words received (the counts matrix is all-gathered first)
static int job_exchange(aiwc_ctx* ctx, const uint64_t* send, const uint64_t* counts, uint64_t* n_recv,
                        cudaStream_t s) {
  const uint32_t R = ctx->nranks, me = ctx->rank;
  std::vector<uint64_t> m;
  int rc = job_allgather_u64(ctx, counts, R, m, s);
  if (rc) return rc;
  uint64_t tot = 0;
  for (uint32_t p = 0; p < R; ++p) tot += m[(size_t)p * R + me];
  CK(grow(ctx->nc_recv, std::max<uint64_t>(tot, 1) * 8));
  uint64_t* recv = P<uint64_t>(ctx->nc_recv);
  NC(ncclGroupStart());
  uint64_t so = 0, ro = 0;
  for (uint32_t p = 0; p < R; ++p) {
    const uint64_t sc = counts[p], rcnt = m[(size_t)p * R + me];
    if (sc) NC(ncclSend(send + so, sc, ncclUint64, (int)p, ctx->comm, s));
    if (rcnt) NC(ncclRecv(recv + ro, rcnt, ncclUint64, (int)p, ctx->comm, s));
    so += sc; ro += rcnt;
  }
  NC(ncclGroupEnd());
  *n_recv = tot;
  return AIWC_OK;
}

static void merge_sorted(std::vector<uint64_t>& acc, const uint64_t* v, size_t n) {
  const size_t a = acc.size();
  acc.insert(acc.end(), v, v + n);
  std::inplace_merge(acc.begin(), acc.begin() + (ptrdiff_t)a, acc.end());
}

static int finalize_job(aiwc_ctx* ctx, aiwc_result* out, void* stream) {
  aiwc_result loc{};
  int rc = finalize_local(ctx, &loc, stream);
  if (rc) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t R = ctx->nranks, me = ctx->rank;
  const uint64_t M = ctx->job[4];
  const bool has_br = ctx->job[6] > 0;
  // the shard's histograms (the owner statistics below reuse the host state block)
  std::vector<uint64_t> itb_h(ctx->h_state->itb_hist, ctx->h_state->itb_hist + HBINS);
  std::vector<uint64_t> ipt_h(ctx->h_state->ipt_hist, ctx->h_state->ipt_hist + HBINS);
  const uint64_t itb_sum = loc.itb.sum, ipt_sum = loc.ipt.sum;

  // ---- memory: the owners' statistics ----
  aiwc_memory_part mp{};
  std::vector<uint64_t> hist0(CBINS, 0), big;
  if (M) {
    if (ctx->shard_dense) {
      const uint64_t words = ctx->n_chunk_words;
      CK(grow(ctx->nc_bits, (size_t)R * words * 4));
      NC(ncclAllGather(ctx->chunk_bits.p, ctx->nc_bits.p, words, ncclUint32, ctx->comm, s));
      uint64_t* runs = nullptr;
      std::vector<uint64_t> cnt(R);
      if ((rc = aiwc_shard_pack(ctx, P<uint32_t>(ctx->nc_bits), me, R, &runs, cnt.data(), stream))) return rc;
      for (auto& c : cnt) c *= 2;  // two words per run
      uint64_t n_words = 0;
      if ((rc = job_exchange(ctx, runs, cnt.data(), &n_words, s))) return rc;
      if ((rc = aiwc_shard_owned(ctx, P<uint64_t>(ctx->nc_recv), n_words / 2, P<uint32_t>(ctx->nc_bits), me, R, M,
                                 &mp, stream))) return rc;
    } else {
      // compacted addresses to key-range owners (ranges aligned to 1024 keys)
      const uint64_t base = ctx->job[0] & ~1023ull, vary = ctx->job[2] ^ ctx->job[3];
      const uint32_t k = vary ? std::min<uint32_t>((uint32_t)__builtin_ctzll(vary), 32u) : 0u;
      const uint64_t n_keys = ((ctx->job[1] - base) >> k) + 1;
      uint64_t kpr = (n_keys + R - 1) / R;
      kpr = (kpr + 1023) / 1024 * 1024;
      uint64_t *rd = nullptr, *wr = nullptr;
      std::vector<uint64_t> c2(2 * R);
      if ((rc = aiwc_partition_addresses(ctx, base, k, kpr, R, &rd, &wr, c2.data(), stream))) return rc;
      // reads and writes travel in one exchange: [reads for o | writes for o] per owner
      const uint64_t nr = ctx->n_rd, nw = ctx->n_wr;
      CK(grow(ctx->nc_send, std::max<uint64_t>(nr + nw, 1) * 8));
      std::vector<uint64_t> cnt(R);
      uint64_t so = 0, ro = 0, wo = 0;
      for (uint32_t o = 0; o < R; ++o) {
        CK(cudaMemcpyAsync(P<uint64_t>(ctx->nc_send) + so, rd + ro, c2[o] * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(P<uint64_t>(ctx->nc_send) + so + c2[o], wr + wo, c2[R + o] * 8, cudaMemcpyDeviceToDevice, s));
        cnt[o] = c2[o] + c2[R + o];
        so += cnt[o]; ro += c2[o]; wo += c2[R + o];
      }
      // per-owner read counts travel too, so the owner can split what it receives
      std::vector<uint64_t> rc_all;
      if ((rc = job_allgather_u64(ctx, c2.data(), 2 * R, rc_all, s))) return rc;
      uint64_t n_words = 0;
      if ((rc = job_exchange(ctx, P<uint64_t>(ctx->nc_send), cnt.data(), &n_words, s))) return rc;
      // regroup: reads of every sender first, then writes
      const uint64_t* recv = P<uint64_t>(ctx->nc_recv);
      uint64_t tr = 0, tw = 0;
      for (uint32_t p = 0; p < R; ++p) { tr += rc_all[(size_t)p * 2 * R + me]; tw += rc_all[(size_t)p * 2 * R + R + me]; }
      CK(grow(ctx->nc_pack, std::max<uint64_t>(tr + tw, 1) * 8));
      uint64_t* rw = P<uint64_t>(ctx->nc_pack);
      uint64_t off = 0, orr = 0, ow = tr;
      for (uint32_t p = 0; p < R; ++p) {
        const uint64_t a = rc_all[(size_t)p * 2 * R + me], b = rc_all[(size_t)p * 2 * R + R + me];
        CK(cudaMemcpyAsync(rw + orr, recv + off, a * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(rw + ow, recv + off + a, b * 8, cudaMemcpyDeviceToDevice, s));
        off += a + b; orr += a; ow += b;
      }
      const uint64_t lo = (uint64_t)me * kpr, n_owned = lo < n_keys ? std::min(kpr, n_keys - lo) : 0;
      if ((rc = aiwc_memory_partial(ctx, rw, tr, rw + tr, tw, base, k, lo, n_owned, M, &mp, stream))) return rc;
    }
    hist0.assign(mp.cnt_hist0, mp.cnt_hist0 + CBINS);
    big.assign(mp.big, mp.big + mp.n_big);
  }

  // ---- one packed all-reduce: every summable integer, plus each rank's list lengths
  // in its own row of an [R][5] block (the sum hands every rank all lengths) ----
  const uint32_t n_opc = loc.n_opcodes, tb = (uint32_t)ctx->branch_tab_host.size();
  std::vector<uint64_t> pk;
  pk.reserve(12 + n_opc + 3 * 1024 + 5 * R + (has_br ? tb : 0));
  const uint64_t sc[12] = {loc.n_events, loc.total_instructions, loc.work_items, loc.barriers_hit, loc.total_reads,
                           loc.total_writes, itb_sum, ipt_sum, loc.branch_executions, mp.unique_reads,
                           mp.unique_writes, mp.footprint};
  pk.insert(pk.end(), sc, sc + 12);
  pk.insert(pk.end(), loc.opcode_counts, loc.opcode_counts + n_opc);
  pk.insert(pk.end(), itb_h.begin(), itb_h.end());
  pk.insert(pk.end(), ipt_h.begin(), ipt_h.end());
  pk.insert(pk.end(), hist0.begin(), hist0.end());
  const size_t lens_at = pk.size();
  pk.resize(pk.size() + 5 * R, 0);
  pk[lens_at + 5 * me + 0] = ctx->itb_ovf_sorted.size();
  pk[lens_at + 5 * me + 1] = ctx->ipt_ovf_sorted.size();
  pk[lens_at + 5 * me + 2] = big.size();
  pk[lens_at + 5 * me + 3] = loc.n_widths;
  pk[lens_at + 5 * me + 4] = loc.n_site_list;
  if (has_br) pk.insert(pk.end(), ctx->branch_tab_host.begin(), ctx->branch_tab_host.end());
  CK(grow(ctx->nc_pack, pk.size() * 8));
  CK(cudaMemcpyAsync(ctx->nc_pack.p, pk.data(), pk.size() * 8, cudaMemcpyHostToDevice, s));
  NC(ncclAllReduce(ctx->nc_pack.p, ctx->nc_pack.p, pk.size(), ncclUint64, ncclSum, ctx->comm, s));
  CK(cudaMemcpyAsync(pk.data(), ctx->nc_pack.p, pk.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));

  // ---- one all-gather of the variable parts, padded to the longest ----
  std::vector<uint64_t> blob;
  double ls[NLEVELS];
  for (int i = 0; i < NLEVELS; ++i) ls[i] = mp.level_sum[i];
  blob.insert(blob.end(), reinterpret_cast<uint64_t*>(ls), reinterpret_cast<uint64_t*>(ls) + NLEVELS);
  blob.insert(blob.end(), ctx->itb_ovf_sorted.begin(), ctx->itb_ovf_sorted.end());
  blob.insert(blob.end(), ctx->ipt_ovf_sorted.begin(), ctx->ipt_ovf_sorted.end());
  blob.insert(blob.end(), big.begin(), big.end());
  for (uint32_t i = 0; i < loc.n_widths; ++i) {
    blob.push_back(loc.width_values[i]); blob.push_back(loc.width_counts[i]);
    blob.push_back(ctx->width_firsts[i] + ctx->info.first_event);  // job-wide first appearance
  }
  for (uint32_t i = 0; i < loc.n_site_list; ++i) { blob.push_back(loc.site_ids[i]); blob.push_back(loc.site_counts[i]); }
  size_t width = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const uint64_t* L = &pk[lens_at + 5 * r];
    width = std::max<size_t>(width, NLEVELS + L[0] + L[1] + L[2] + 3 * L[3] + 2 * L[4]);
  }
  blob.resize(width, 0);
  CK(grow(ctx->nc_blob, (size_t)(R + 1) * width * 8));
  uint64_t* db = P<uint64_t>(ctx->nc_blob);
  CK(cudaMemcpyAsync(db + (size_t)R * width, blob.data(), width * 8, cudaMemcpyHostToDevice, s));
  NC(ncclAllGather(db + (size_t)R * width, db, width, ncclUint64, ctx->comm, s));
  std::vector<uint64_t> all((size_t)R * width);
  CK(cudaMemcpyAsync(all.data(), db, all.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));

  // ---- assemble the job's result (the rules of aiwc_finalize) ----
  size_t o = 0;
  auto take = [&](size_t n) { o += n; return &pk[o - n]; };
  const uint64_t* S = take(12);
  const uint64_t* opc = take(n_opc);
  const uint64_t* ih = take(HBINS);
  const uint64_t* ph = take(HBINS);
  const uint64_t* h0 = take(CBINS);
  take(5 * R);
  const uint64_t* btab = has_br ? take(tb) : nullptr;
  double lsum[NLEVELS] = {0};
  std::vector<uint64_t> itb_o, ipt_o, big_all;
  std::vector<std::pair<uint64_t, std::pair<uint64_t, uint64_t>>> wmap;  // width -> (count, first)
  std::vector<std::pair<uint64_t, uint64_t>> smap;                       // (site, count)
  for (uint32_t r = 0; r < R; ++r) {  // rank order: the fp64 level sums are deterministic
    const uint64_t* L = &pk[lens_at + 5 * r];
    const uint64_t* b = &all[(size_t)r * width];
    const double* d = reinterpret_cast<const double*>(b);
    for (int i = 0; i < NLEVELS; ++i) lsum[i] += d[i];
    size_t q = NLEVELS;
    merge_sorted(itb_o, b + q, L[0]); q += L[0];
    merge_sorted(ipt_o, b + q, L[1]); q += L[1];
    big_all.insert(big_all.end(), b + q, b + q + L[2]); q += L[2];
    for (uint64_t i = 0; i < L[3]; ++i, q += 3) wmap.push_back({b[q], {b[q + 1], b[q + 2]}});
    for (uint64_t i = 0; i < L[4]; ++i, q += 2) smap.push_back({b[q], b[q + 1]});
  }
  aiwc_result rj{};
  rj.n_events = S[0]; rj.total_instructions = S[1]; rj.work_items = S[2]; rj.barriers_hit = S[3];
  rj.total_reads = S[4]; rj.total_writes = S[5];
  rj.branch_executions = S[8];
  rj.unique_reads = S[9]; rj.unique_writes = S[10]; rj.footprint = S[11];
  ctx->opc_counts.assign(opc, opc + n_opc);
  {
    std::vector<uint64_t> oc;
    unsigned __int128 tot = 0;
    for (uint32_t i = 0; i < n_opc; ++i) if (opc[i]) { oc.push_back(opc[i]); tot += opc[i]; }
    std::sort(oc.begin(), oc.end(), std::greater<uint64_t>());
    rj.opcode_coverage = coverage_from(oc, nullptr, 0, tot);
  }
  ctx->job_itb_ovf = itb_o; ctx->job_ipt_ovf = ipt_o;
  std::vector<unsigned long long> ihv(ih, ih + HBINS), phv(ph, ph + HBINS), h0v(h0, h0 + CBINS);
  order_stats(ihv.data(), itb_o, &rj.itb); rj.itb.sum = S[6];
  order_stats(phv.data(), ipt_o, &rj.ipt); rj.ipt.sum = S[7];
  std::sort(big_all.begin(), big_all.end(), std::greater<uint64_t>());
  rj.footprint_90 = M ? coverage_from(big_all, h0v.data(), CBINS, M) : 0;
  for (int i = 0; i < NLEVELS; ++i) {
    const double v = M ? -lsum[i] : 0.0;
    if (i == 0) rj.gmae = v; else rj.lmae[i - 1] = v;
  }
  // branch entropies from the job's pooled pattern table (entropy.py:123-132)
  if (btab && rj.branch_executions) {
    unsigned long long obs = 0;
    double y = 0.0, l = 0.0;
    for (uint32_t i = 0; i < tb; ++i) {
      const uint64_t tot = btab[i] >> 32;
      if (!tot) continue;
      obs += tot;
      const double dt = (double)tot, p = (double)(btab[i] & 0xFFFFFFFFull) / dt, q = 1.0 - p;
      const double hh = -((p > 0 ? p * log2(p) : 0.0) + (q > 0 ? q * log2(q) : 0.0));
      y += dt * hh;
      l += dt * (p < q ? p : q);
    }
    rj.branch_observations = obs;
    rj.yokota = obs ? y / (double)obs : 0.0;
    rj.linear = obs ? l / (double)obs : 0.0;
  }
  rj.branch_excluded = rj.branch_executions - rj.branch_observations;
  // sites ascending with summed executions; widths in first-appearance order
  std::sort(smap.begin(), smap.end());
  ctx->site_ids.clear(); ctx->site_counts.clear();
  for (auto& sc2 : smap) {
    if (!ctx->site_ids.empty() && ctx->site_ids.back() == sc2.first) ctx->site_counts.back() += sc2.second;
    else { ctx->site_ids.push_back(sc2.first); ctx->site_counts.push_back(sc2.second); }
  }
  {
    std::vector<uint64_t> scs(ctx->site_counts);
    std::sort(scs.begin(), scs.end(), std::greater<uint64_t>());
    rj.branch_90 = rj.branch_executions ? coverage_from(scs, nullptr, 0, rj.branch_executions) : 0;
  }
  rj.n_sites = ctx->site_ids.size();
  std::sort(wmap.begin(), wmap.end());
  std::vector<std::pair<uint64_t, std::pair<uint64_t, uint64_t>>> wm;  // (first, (width, count))
  for (size_t i = 0; i < wmap.size();) {
    uint64_t c = 0, f = ~0ull;
    size_t e = i;
    for (; e < wmap.size() && wmap[e].first == wmap[i].first; ++e) { c += wmap[e].second.first; f = std::min(f, wmap[e].second.second); }
    wm.push_back({f, {wmap[i].first, c}});
    i = e;
  }
  std::sort(wm.begin(), wm.end());
  ctx->width_vals.clear(); ctx->width_counts.clear(); ctx->width_firsts.clear();
  for (auto& w : wm) {
    ctx->width_vals.push_back(w.second.first); ctx->width_counts.push_back(w.second.second);
    ctx->width_firsts.push_back(w.first);
  }
  rj.entries = rj.unique_reads + rj.unique_writes + rj.branch_executions;
  rj.n_opcodes = n_opc;
  rj.opcode_counts = ctx->opc_counts.data();
  rj.n_widths = (uint32_t)ctx->width_vals.size();
  rj.width_values = ctx->width_vals.data();
  rj.width_counts = ctx->width_counts.data();
  rj.n_site_list = (uint32_t)ctx->site_ids.size();
  rj.site_ids = ctx->site_ids.data();
  rj.site_counts = ctx->site_counts.data();
  rj.used_dense_table = ctx->shard_dense;
  rj.kernels_launched = ctx->kernels;
  rj.d2h_bytes = ctx->d2h;
  for (int i = 0; i < AIWC_N_PHASES; ++i) rj.phase_ms[i] = loc.phase_ms[i];
  *out = rj;
  if (ctx->opts.entry_cap && rj.entries > ctx->opts.entry_cap) {
    fail(ctx, AIWC_ERR_TOO_LARGE, "trace state exceeds the in-memory cap");
    ctx->err.entries = ctx->opts.entry_cap + 1;
    ctx->err.cap = ctx->opts.entry_cap;
    return AIWC_ERR_TOO_LARGE;
  }
  return AIWC_OK;
}

extern "C" int aiwc_finalize(aiwc_ctx* ctx, aiwc_result* out, void* stream) {
  if (ctx && ctx->comm) return finalize_job(ctx, out, stream);
  return finalize_local(ctx, out, stream);
}


// ---------------------------------------------------------------------------
// stream validation (aiwc_validate.cu)
// ---------------------------------------------------------------------------
namespace {

__global__ void v_init_kernel(ValidateState* vs) {
  vs->first_ke = ~0ull; vs->winner = ~0ull;
  vs->n_struct = 0; vs->n_groups = 0; vs->bad_kind = 0; vs->counts_used = 0; vs->kb0 = 0; vs->dp = 0;
}

std::string tup(const int64_t v[3]) {
  return "(" + std::to_string(v[0]) + ", " + std::to_string(v[1]) + ", " + std::to_string(v[2]) + ")";
}

// group tuple of a key: linear index in the launch grid, else a dictionary key
bool group_of(uint64_t key, const int64_t grid[3], int64_t out[3]) {
  const uint64_t vol = (uint64_t)(grid[0] * grid[1] * grid[2]);
  if (key >= vol) return false;
  out[0] = (int64_t)(key % (uint64_t)grid[0]);
  out[1] = (int64_t)((key / (uint64_t)grid[0]) % (uint64_t)grid[1]);
  out[2] = (int64_t)(key / (uint64_t)(grid[0] * grid[1]));
  return true;
}

}  // namespace

extern "C" int aiwc_validate(aiwc_ctx* ctx, const uint8_t* kind, const uint64_t* payload, const aiwc_trace_info* info,
                             const int64_t global_size[3], const int64_t local_size[3], aiwc_violation* out,
                             void* stream) {
  if (!ctx || !info || !out || !global_size || !local_size) return AIWC_ERR_ARGUMENT;
  const uint64_t n = info->n_events;
  if (n && (!kind || !payload)) return fail(ctx, AIWC_ERR_ARGUMENT, "null column pointer");
  if (n >= (1ull << 32)) return fail(ctx, AIWC_ERR_UNSUPPORTED, "more than 2^32-1 events in one trace");
  int64_t grid[3];
  uint64_t lv = 1;
  for (int d = 0; d < 3; ++d) {
    if (global_size[d] < 1 || local_size[d] < 1) return fail(ctx, AIWC_ERR_ARGUMENT, "launch sizes must be positive");
    grid[d] = (global_size[d] + local_size[d] - 1) / local_size[d];
    lv *= (uint64_t)local_size[d];
  }
  if (lv > VALIDATE_LV_MAX)
    return fail(ctx, AIWC_ERR_UNSUPPORTED, "device validation holds work-groups of at most 1024 work-items");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  *out = aiwc_violation{};
  out->event_index = -1;
  const uint64_t tiles = (n + VALIDATE_TILE - 1) / VALIDATE_TILE;
  CK(grow(ctx->v_state, sizeof(ValidateState)));
  CK(grow(ctx->v_tiles, std::max<uint64_t>(tiles, 1) * 8));
  CK(grow(ctx->v_scan, (std::max<uint64_t>(tiles, 1) / 1024 + 2) * 4 * 4));
  ValidateState* vs = P<ValidateState>(ctx->v_state);
  ValidateBufs b{};
  b.tile_s = P<uint32_t>(ctx->v_tiles);
  b.tile_g = b.tile_s + std::max<uint64_t>(tiles, 1);
  b.scan_scratch = P<uint32_t>(ctx->v_scan);
  int kernels = 0;
  v_init_kernel<<<1, 1, 0, s>>>(vs);
  validate_phase1(kind, n, vs, b, s, &kernels);
  ValidateState hv{};
  CK(cudaMemcpyAsync(&hv, vs, sizeof hv, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hv.bad_kind) return fail(ctx, AIWC_ERR_UNSUPPORTED, "kind byte outside the columnar alphabet");
  const uint64_t S = hv.n_struct, NG = hv.n_groups;
  CK(grow(ctx->v_spos, std::max<uint64_t>(S, 1) * 8));
  CK(grow(ctx->v_spay, std::max<uint64_t>(S, 1) * 8));
  CK(grow(ctx->v_sgap, std::max<uint64_t>(S, 1) * 8));
  CK(grow(ctx->v_gstart, std::max<uint64_t>(NG, 1) * 4));
  CK(grow(ctx->v_recs, (NG + 3) * sizeof(ValidateRecord)));
  CK(grow(ctx->v_srange, std::max<uint64_t>(S, 1) * 4));
  CK(grow(ctx->v_fwge, (NG + 1) * 4));
  CK(grow(ctx->v_keys, std::max<uint64_t>(S, 1) * 8));
  CK(grow(ctx->v_keys_tmp, std::max<uint64_t>(S, 1) * 8));
  CK(grow(ctx->v_hist, radix_hist_bytes(std::max<uint64_t>(S, 1))));
  CK(grow(ctx->v_prevk, std::max<uint64_t>(S, 1)));
  CK(grow(ctx->v_unf, (NG + 1) * 8));
  CK(grow(ctx->v_bmm, (NG + 1) * 8));
  const uint32_t counts_cap = 1u << 20;
  CK(grow(ctx->v_counts, counts_cap * 4));
  b.spos = P<uint64_t>(ctx->v_spos); b.spay = P<uint64_t>(ctx->v_spay); b.sgap = P<uint64_t>(ctx->v_sgap);
  b.gstart = P<uint32_t>(ctx->v_gstart); b.recs = P<ValidateRecord>(ctx->v_recs);
  b.counts = P<uint32_t>(ctx->v_counts); b.counts_cap = counts_cap;
  b.srange = P<uint32_t>(ctx->v_srange); b.first_wge = P<uint32_t>(ctx->v_fwge);
  b.keys = P<uint64_t>(ctx->v_keys); b.keys_tmp = P<uint64_t>(ctx->v_keys_tmp); b.sort_hist = P<uint32_t>(ctx->v_hist);
  b.prevk = P<uint8_t>(ctx->v_prevk); b.unf = P<unsigned long long>(ctx->v_unf);
  b.bmin = P<uint32_t>(ctx->v_bmm); b.bmax = b.bmin + (NG + 1);
  const uint32_t n_ctas = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((NG + 1 + 3) / 4, (uint64_t)ctx->n_sms * 8));
  validate_phase2(kind, payload, n, (uint32_t)lv, vs, b, S, NG, n_ctas, (ctx->opts.flags & AIWC_OPT_VALIDATE_REPLAY) != 0,
                  s, &kernels);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&hv, vs, sizeof hv, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // ---- the first violation, or the end-of-stream rules (finish(), trace.py:420-424) ----
  uint32_t code = AIWC_V_NONE;
  ValidateRecord rec{};
  std::vector<uint32_t> counts;
  if (hv.winner != ~0ull) {
    const uint64_t low = hv.winner & 0xFFFFFFFFull;
    const uint64_t slot = low == 0xFFFFFFFFull ? NG + 2 : hv.dp ? NG + 1 : low;
    CK(cudaMemcpy(&rec, P<ValidateRecord>(ctx->v_recs) + slot, sizeof rec, cudaMemcpyDeviceToHost));
    code = rec.code;
    if (rec.n_counts) {
      counts.resize(rec.n_counts);
      CK(cudaMemcpy(counts.data(), P<uint32_t>(ctx->v_counts) + rec.counts_off, rec.n_counts * 4,
                    cudaMemcpyDeviceToHost));
    }
  } else if (n == 0) {
    code = AIWC_V_EMPTY; rec.index = 0;
  } else if (hv.first_ke == ~0ull) {
    code = AIWC_V_NO_KE; rec.index = n - 1;
  }
  if (code == AIWC_V_NONE) return AIWC_OK;
  out->event_index = (int64_t)rec.index;
  out->detail_code = code;
  out->metric_kind = rec.cls;
  out->group_key = rec.group_key;
  out->local_id = rec.local_id;
  std::sort(counts.begin(), counts.end());
  counts.erase(std::unique(counts.begin(), counts.end()), counts.end());
  out->n_counts = (uint32_t)std::min<size_t>(counts.size(), 64);
  for (uint32_t i = 0; i < out->n_counts; ++i) out->counts[i] = counts[i];
  // the reference's rule ids and detail text (trace.py:278-424)
  std::string rule, detail;
  int64_t g[3];
  const bool in_grid = group_of(rec.group_key, grid, g);
  switch (code) {
    case AIWC_V_KB_NOT_FIRST: rule = "kernel_begin.first"; detail = "first event must be kernel_begin"; break;
    case AIWC_V_KB_DUP: rule = "kernel_begin.first"; detail = "duplicate kernel_begin"; break;
    case AIWC_V_EMPTY: rule = "kernel_begin.first"; detail = "empty stream"; break;
    case AIWC_V_AFTER_KE: rule = "kernel_end.last"; detail = "event after kernel_end"; break;
    case AIWC_V_NO_KE: rule = "kernel_end.last"; detail = "stream has no kernel_end"; break;
    case AIWC_V_KE_OPEN_GROUP: rule = "wg.nesting"; detail = "kernel_end with open work-group"; break;
    case AIWC_V_OUTSIDE_SEG:
      rule = "event.outside_segment";
      detail = std::string(rec.cls == AIWC_K_INSTR ? "Instruction" : rec.cls == AIWC_K_BRANCH ? "Branch" : "Memory") +
               " outside a work-item segment";
      break;
    case AIWC_V_BAR_OUTSIDE: rule = "event.outside_segment"; detail = "Barrier outside a work-item segment"; break;
    case AIWC_V_WGB_OPEN: rule = "wg.nesting"; detail = "wg_begin while another group is open"; break;
    case AIWC_V_WGE_MISMATCH: rule = "wg.nesting"; detail = "wg_end does not match open group"; break;
    case AIWC_V_WGE_OPEN_SEG: rule = "wi.nesting"; detail = "wg_end with open work-item segment"; break;
    case AIWC_V_UNFINISHED: {
      rule = "wi.unfinished";
      if (in_grid) {
        const int64_t l[3] = {(int64_t)(rec.local_id % (uint64_t)local_size[0]),
                              (int64_t)((rec.local_id / (uint64_t)local_size[0]) % (uint64_t)local_size[1]),
                              (int64_t)(rec.local_id / (uint64_t)(local_size[0] * local_size[1]))};
        const int64_t gid[3] = {g[0] * local_size[0] + l[0], g[1] * local_size[1] + l[1], g[2] * local_size[2] + l[2]};
        detail = "work-item " + tup(gid) + " never ended";
      } else {
        detail = "work-item (local " + std::to_string(rec.local_id) + " of group key " + std::to_string(rec.group_key) +
                 ") never ended";
      }
      break;
    }
    case AIWC_V_DIVERGENCE: {
      rule = "barrier.divergence";
      std::string lst = "[";
      for (size_t i = 0; i < counts.size(); ++i) lst += (i ? ", " : "") + std::to_string(counts[i]);
      lst += "]";
      detail = "work-items of group " + (in_grid ? tup(g) : "key " + std::to_string(rec.group_key)) +
               " hit differing barrier counts " + lst;
      break;
    }
    case AIWC_V_WI_OUTSIDE_GROUP: rule = "wi.nesting"; detail = "work-item event outside a work-group"; break;
    case AIWC_V_WI_ID: rule = "wi.id_arithmetic"; detail = "local_id[2] >= local_size[2]"; break;
    case AIWC_V_OPEN_WHILE_OPEN: rule = "wi.nesting"; detail = "segment opened while another is open"; break;
    case AIWC_V_WIB_STARTED: rule = "wi.nesting"; detail = "wi_begin for an already-started work-item"; break;
    case AIWC_V_WIR_NOT_BARRIER: rule = "wi.resume_without_barrier"; detail = "resume of a work-item not waiting at a barrier"; break;
    case AIWC_V_WIE_NO_SEG: rule = "wi.nesting"; detail = "wi_end without matching open segment"; break;
    default: rule = "unknown"; break;
  }
  snprintf(out->rule, sizeof out->rule, "%s", rule.c_str());
  snprintf(out->detail, sizeof out->detail, "%s", detail.c_str());
  ctx->err = aiwc_error{};
  ctx->err.code = AIWC_ERR_INVALID_STREAM;
  ctx->err.event_index = out->event_index;
  snprintf(ctx->err.rule, sizeof ctx->err.rule, "%s", rule.c_str());
  snprintf(ctx->err.message, sizeof ctx->err.message, "%s", detail.c_str());
  return AIWC_ERR_INVALID_STREAM;
}
