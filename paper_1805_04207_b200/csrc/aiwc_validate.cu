// aiwc_validate.cu -- first stream violation of a columnar trace, on the device.
//
// The reference validates every stream inside consume() with StreamChecker
// (pkg/src/aiwc/trace.py:289-424; metrics.py:126-129,181-184) and raises
// InvalidStream(event_index, rule, detail) at the first violation.  A
// columnar trace decodes to events as ColumnarTrace.iter_events does (group
// from the last wg_begin, work-item ids from the local linear id), so the
// same rules apply to it.  Three steps:
//
//  K1  compaction of the structural events (everything except instructions,
//      memory accesses and branches: kernel / group / work-item boundaries and
//      barriers) with, for each, the first metric event of the gap after it;
//      work-group begins are listed separately.  Two passes (counts, writes)
//      around a device scan.
//  K2  one warp per work-group range (a wg_begin up to the next one; range 0
//      is the prefix before the first) replays the checker over the range's
//      structural events with per-local-id status / barrier-count tables in
//      shared memory, checking every gap against the open segment.  Each
//      range assumes a valid prefix (no group or segment open, header seen,
//      ended iff a kernel_end precedes it), which holds for the range holding
//      the true first violation -- so the minimum over ranges is exact.
//  K3  the host reads the winning range's record and formats the message.
#include "aiwc_internal.cuh"
#include "aiwc_util.cuh"

namespace aiwc {

namespace {

constexpr int VT = 256;       // K1 threads
constexpr int VEPT = 16;      // events per thread
constexpr int VTILE = VT * VEPT;
static_assert(VTILE == VALIDATE_TILE, "tile size shared with the host");
constexpr int K2_WARPS = 4;   // ranges per K2 CTA
constexpr uint32_t LV_MAX = VALIDATE_LV_MAX;

__device__ __forceinline__ bool structural(uint32_t k) { return (k & 0x0Fu) == 0u && k != 0u; }
__device__ __forceinline__ bool metric(uint32_t k) {
  return k == AIWC_K_INSTR || k == AIWC_K_LOAD || k == AIWC_K_ATOMIC_LOAD || k == AIWC_K_STORE ||
         k == AIWC_K_ATOMIC_STORE || k == AIWC_K_BRANCH;
}
__device__ __forceinline__ bool known(uint32_t k) {
  return metric(k) || k == AIWC_K_WI_END || k == AIWC_K_BARRIER || k == AIWC_K_WI_BEGIN || k == AIWC_K_WI_RESUME ||
         k == AIWC_K_WG_BEGIN || k == AIWC_K_WG_END || k == AIWC_K_KERNEL_BEGIN || k == AIWC_K_KERNEL_END;
}

__device__ __forceinline__ uint8_t kind_at(const uint8_t* kind, uint64_t i, uint64_t n) { return i < n ? kind[i] : 0; }

// the 16 kind bytes of one thread (columns are 16-byte aligned): one 16-byte load
__device__ __forceinline__ void load_kinds(const uint8_t* kind, uint64_t e0, uint64_t n, uint8_t (&ks)[VEPT]) {
  if (e0 + VEPT <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(kind + e0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < VEPT; ++j) ks[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
  } else {
#pragma unroll
    for (int j = 0; j < VEPT; ++j) ks[j] = kind_at(kind, e0 + j, n);
  }
}

// per kind byte: known (bit 0) | structural (bit 8) | wg_begin (bit 16) | kernel_end (bit 24);
// a 1 KB shared table turns the per-byte class tests into one load and one add
__device__ __forceinline__ uint32_t kind_flags(uint32_t k) {
  return (known(k) ? 1u : 0u) | (structural(k) ? 1u << 8 : 0u) | (k == AIWC_K_WG_BEGIN ? 1u << 16 : 0u) |
         (k == AIWC_K_KERNEL_END ? 1u << 24 : 0u);
}
__device__ __forceinline__ void fill_flags(uint32_t* tbl) {
  for (uint32_t k = threadIdx.x; k < 256; k += blockDim.x) tbl[k] = kind_flags(k);
  __syncthreads();
}

// K1a: per-tile counts of structural events and of work-group begins
__global__ void __launch_bounds__(VT) v_count_kernel(const uint8_t* __restrict__ kind, uint64_t n,
                                                     uint32_t* __restrict__ s_cnt, uint32_t* __restrict__ g_cnt,
                                                     ValidateState* vs) {
  __shared__ uint32_t red[2][VT / 32];
  const uint64_t tile = blockIdx.x;
  const uint64_t e0 = tile * VTILE + (uint64_t)threadIdx.x * VEPT;
  __shared__ uint32_t tbl[256];
  fill_flags(tbl);
  unsigned long long first_ke = ~0ull;
  uint8_t ks[VEPT];
  load_kinds(kind, e0, n, ks);
  const uint32_t valid = e0 >= n ? 0u : (uint32_t)min((uint64_t)VEPT, n - e0);
  uint32_t acc = 0;  // four 8-bit sums of the flags (<= 16 each)
#pragma unroll
  for (int j = 0; j < VEPT; ++j)
    if ((uint32_t)j < valid) acc += tbl[ks[j]];
  if (acc >> 24) {  // a kernel_end among my events (rare): its first index
    for (uint32_t j = 0; j < valid; ++j)
      if (ks[j] == AIWC_K_KERNEL_END) { first_ke = e0 + j; break; }
  }
  const bool bad = (acc & 0xFFu) != valid;
  uint32_t sc = (acc >> 8) & 0xFFu, gc = (acc >> 16) & 0xFFu;
  if (first_ke != ~0ull) atomicMin(&vs->first_ke, first_ke);
  if (tile == 0 && threadIdx.x == 0) vs->kb0 = n && kind[0] == AIWC_K_KERNEL_BEGIN;
  if (bad) atomicOr(&vs->bad_kind, 1u);
  sc = warp_sum(sc); gc = warp_sum(gc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = sc; red[1][warp] = gc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0, b = 0;
    for (int w = 0; w < VT / 32; ++w) { a += red[0][w]; b += red[1][w]; }
    s_cnt[tile] = a; g_cnt[tile] = b;
  }
}

// K1b: write the structural entries (position | kind << 32), their payloads,
// the gap after each (first metric index << 8 | its kind, or ~0) and the
// compact indices of the work-group begins
__global__ void __launch_bounds__(VT) v_write_kernel(const uint8_t* __restrict__ kind, const uint64_t* __restrict__ payload,
                                                     uint64_t n, const uint32_t* __restrict__ s_off,
                                                     const uint32_t* __restrict__ g_off, uint64_t* __restrict__ spos,
                                                     uint64_t* __restrict__ spay, uint64_t* __restrict__ sgap,
                                                     uint32_t* __restrict__ gstart, uint32_t* __restrict__ srange,
                                                     uint32_t* __restrict__ first_wge) {
  __shared__ uint32_t wsum[2][VT / 32];
  const uint64_t tile = blockIdx.x;
  const uint64_t e0 = tile * VTILE + (uint64_t)threadIdx.x * VEPT;
  uint32_t smask = 0, gmask = 0;
  uint8_t ks[VEPT];
  load_kinds(kind, e0, n, ks);
#pragma unroll
  for (int j = 0; j < VEPT; ++j) {
    if (structural(ks[j])) smask |= 1u << j;
    if (ks[j] == AIWC_K_WG_BEGIN) gmask |= 1u << j;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t sc = __popc(smask), gc = __popc(gmask);
  uint32_t si = sc, gi = gc;  // inclusive warp scans
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, si, o), b = __shfl_up_sync(0xffffffffu, gi, o);
    if (lane >= o) { si += a; gi += b; }
  }
  if (lane == 31) { wsum[0][warp] = si; wsum[1][warp] = gi; }
  __syncthreads();
  uint32_t sb = s_off[tile], gb = g_off[tile];
  for (int w = 0; w < warp; ++w) { sb += wsum[0][w]; gb += wsum[1][w]; }
  uint32_t s = sb + si - sc, g = gb + gi - gc;
  for (int j = 0; j < VEPT; ++j) {
    if (!((smask >> j) & 1u)) continue;
    const uint64_t e = e0 + j;
    spos[s] = e | ((uint64_t)ks[j] << 32);
    spay[s] = payload[e];
    const uint32_t nk = j + 1 < VEPT ? ks[j + 1] : kind_at(kind, e + 1, n);
    sgap[s] = metric(nk) ? (((e + 1) << 8) | nk) : ~0ull;
    if (ks[j] == AIWC_K_WG_BEGIN) gstart[g++] = s;
    srange[s] = g;  // range = work-group begins at or before this entry
    if (ks[j] == AIWC_K_WG_END) atomicMin(&first_wge[g], s);
    ++s;
  }
}

// K2 violation codes (host formats the reference's detail text)
enum : uint32_t {
  V_NONE = 0, V_KB_NOT_FIRST, V_KB_DUP, V_AFTER_KE, V_KE_OPEN_GROUP, V_OUTSIDE_SEG, V_BAR_OUTSIDE, V_WGB_OPEN,
  V_WGE_MISMATCH, V_WGE_OPEN_SEG, V_UNFINISHED, V_DIVERGENCE, V_WI_OUTSIDE_GROUP, V_WI_ID, V_OPEN_WHILE_OPEN,
  V_WIB_STARTED, V_WIR_NOT_BARRIER, V_WIE_NO_SEG
};

enum : uint8_t { S_ABSENT = 0, S_OPEN = 1, S_AT_BARRIER = 2, S_DONE = 3 };

struct WarpTables {
  uint8_t status[LV_MAX];
  uint32_t bcount[LV_MAX];
  uint32_t order[LV_MAX];  // insertion rank in the status dict (for "never ended")
};

__global__ void __launch_bounds__(K2_WARPS * 32) v_check_kernel(const uint64_t* __restrict__ spos,
                                                                const uint64_t* __restrict__ spay,
                                                                const uint64_t* __restrict__ sgap, uint64_t S,
                                                                const uint32_t* __restrict__ gstart, uint64_t NG,
                                                                uint32_t lv, ValidateState* vs, ValidateRecord* recs,
                                                                uint32_t* counts_buf, uint32_t counts_cap) {
  __shared__ WarpTables T[K2_WARPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  WarpTables& tb = T[wib];
  const unsigned long long first_ke = vs->first_ke;
  for (uint64_t r = (uint64_t)blockIdx.x * K2_WARPS + wib; r <= NG; r += (uint64_t)gridDim.x * K2_WARPS) {
    const uint64_t lo = r == 0 ? 0 : gstart[r - 1];
    const uint64_t hi = r < NG ? gstart[r] : S;
    // state at the range start under a valid prefix
    bool header = r != 0 && vs->kb0, ended = false, gopen = false, sopen = false;
    uint64_t gkey = 0;
    uint32_t slid = 0, n_ins = 0;
    if (r != 0) ended = first_ke < (spos[lo] & 0xFFFFFFFFull);
    uint32_t code = V_NONE, cls = 0;
    uint64_t at = 0, aux_g = 0, aux_l = 0;
    auto clear = [&]() {
      for (uint32_t i = lane; i < lv; i += 32) { tb.status[i] = S_ABSENT; tb.bcount[i] = 0; }
      n_ins = 0;
      __syncwarp();
    };
    clear();
    // 32 entries per coalesced warp load, broadcast one by one with shuffles
    uint64_t c_pos = 0, c_pay = 0, c_gap = ~0ull;
    for (uint64_t s = lo; s < hi && code == V_NONE; ++s) {
      const uint32_t jj = (uint32_t)((s - lo) & 31u);
      if (jj == 0) {
        const uint64_t q = s + lane;
        c_pos = q < hi ? spos[q] : 0ull;
        c_pay = q < hi ? spay[q] : 0ull;
        c_gap = q < hi ? sgap[q] : ~0ull;
      }
      const uint64_t pk = __shfl_sync(0xffffffffu, c_pos, jj);
      const uint64_t pos = pk & 0xFFFFFFFFull;
      const uint32_t k = (uint32_t)(pk >> 32);
      const uint64_t p = __shfl_sync(0xffffffffu, c_pay, jj);
      const uint64_t gp = __shfl_sync(0xffffffffu, c_gap, jj);
      // ---- the structural event (StreamChecker.feed order of checks) ----
      if (ended) { code = V_AFTER_KE; at = pos; break; }
      if (!header) {
        if (k == AIWC_K_KERNEL_BEGIN) { header = true; goto gap; }
        code = V_KB_NOT_FIRST; at = pos; break;
      }
      switch (k) {
        case AIWC_K_BARRIER:
          if (!sopen) { code = V_BAR_OUTSIDE; at = pos; break; }
          if (lane == 0) { tb.status[slid] = S_AT_BARRIER; tb.bcount[slid] += 1; }
          sopen = false;
          break;
        case AIWC_K_KERNEL_BEGIN: code = V_KB_DUP; at = pos; break;
        case AIWC_K_KERNEL_END:
          if (gopen) { code = V_KE_OPEN_GROUP; at = pos; break; }
          ended = true;
          break;
        case AIWC_K_WG_BEGIN:
          if (gopen) { code = V_WGB_OPEN; at = pos; break; }
          gopen = true; gkey = p;
          clear();
          break;
        case AIWC_K_WG_END: {
          if (!gopen || p != gkey) { code = V_WGE_MISMATCH; at = pos; break; }
          if (sopen) { code = V_WGE_OPEN_SEG; at = pos; break; }
          // first work-item (insertion order) not done
          uint32_t best = 0xFFFFFFFFu, best_lid = 0;
          for (uint32_t i = lane; i < lv; i += 32)
            if (tb.status[i] != S_ABSENT && tb.status[i] != S_DONE && tb.order[i] < best) { best = tb.order[i]; best_lid = i; }
          for (int o = 16; o > 0; o >>= 1) {
            const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o), ol = __shfl_xor_sync(0xffffffffu, best_lid, o);
            if (ob < best) { best = ob; best_lid = ol; }
          }
          if (best != 0xFFFFFFFFu) { code = V_UNFINISHED; at = pos; aux_g = gkey; aux_l = best_lid; break; }
          // barrier counts of every work-item seen (barrier_counts keys) must agree
          uint32_t lo_c = 0xFFFFFFFFu, hi_c = 0;
          for (uint32_t i = lane; i < lv; i += 32)
            if (tb.status[i] != S_ABSENT) { lo_c = min(lo_c, tb.bcount[i]); hi_c = max(hi_c, tb.bcount[i]); }
          for (int o = 16; o > 0; o >>= 1) {
            lo_c = min(lo_c, __shfl_xor_sync(0xffffffffu, lo_c, o));
            hi_c = max(hi_c, __shfl_xor_sync(0xffffffffu, hi_c, o));
          }
          if (lo_c != 0xFFFFFFFFu && lo_c != hi_c) { code = V_DIVERGENCE; at = pos; aux_g = gkey; break; }
          gopen = false;
          clear();
          break;
        }
        default: {  // work-item events
          const uint32_t lid = (uint32_t)min(p, (uint64_t)0xFFFFFFFFull);
          if (!gopen) { code = V_WI_OUTSIDE_GROUP; at = pos; break; }
          if (p >= lv) { code = V_WI_ID; at = pos; break; }
          if (k == AIWC_K_WI_BEGIN) {
            if (sopen) { code = V_OPEN_WHILE_OPEN; at = pos; break; }
            if (tb.status[lid] != S_ABSENT) { code = V_WIB_STARTED; at = pos; break; }
            if (lane == 0) { tb.status[lid] = S_OPEN; tb.order[lid] = n_ins; }
            ++n_ins;
            sopen = true; slid = lid;
          } else if (k == AIWC_K_WI_RESUME) {
            if (sopen) { code = V_OPEN_WHILE_OPEN; at = pos; break; }
            if (tb.status[lid] != S_AT_BARRIER) { code = V_WIR_NOT_BARRIER; at = pos; break; }
            if (lane == 0) tb.status[lid] = S_OPEN;
            sopen = true; slid = lid;
          } else {
            if (!sopen || slid != lid) { code = V_WIE_NO_SEG; at = pos; break; }
            sopen = false;
            if (lane == 0) tb.status[lid] = S_DONE;
          }
          break;
        }
      }
      if (code != V_NONE) break;
    gap:
      __syncwarp();
      {  // the first metric event between this structural event and the next
        if (gp != ~0ull) {
          if (ended) { code = V_AFTER_KE; at = gp >> 8; }
          else if (!sopen) { code = V_OUTSIDE_SEG; at = gp >> 8; cls = (uint32_t)(gp & 0xFF); }
        }
      }
    }
    // the next range's wg_begin meets a group this range left open
    if (code == V_NONE && gopen && r < NG) { code = V_WGB_OPEN; at = spos[hi] & 0xFFFFFFFFull; }
    if (code != V_NONE && lane == 0) {
      ValidateRecord& rec = recs[r];
      rec.index = at; rec.code = code; rec.cls = cls; rec.group_key = aux_g; rec.local_id = aux_l;
      rec.n_counts = 0; rec.counts_off = 0;
      if (code == V_DIVERGENCE) {  // the distinct counts, for the message (rare)
        uint32_t m = 0;
        const uint32_t off = atomicAdd(&vs->counts_used, lv);
        if (off + lv <= counts_cap) {
          for (uint32_t i = 0; i < lv; ++i)
            if (tb.status[i] != S_ABSENT) counts_buf[off + m++] = tb.bcount[i];
          rec.n_counts = m; rec.counts_off = off;
        }
      }
      atomicMin(&vs->winner, ((unsigned long long)at << 32) | (unsigned long long)min(r, (uint64_t)0xFFFFFFFFull));
    }
    __syncwarp();
  }
}

// ---- data-parallel checker ----------------------------------------------------------
// Every rule but the per-work-item status ones needs only the previous
// structural entry (segments alternate open/close in a valid prefix) and the
// range's first wg_end; the status rules need the previous entry of the same
// work-item, which a stable sort by (range, local id) provides.  Each entry
// yields its first failing check in StreamChecker order (event, then the gap
// after it); the minimum index over entries is the first violation.
constexpr uint8_t PK_NONE = 0xFF;
constexpr uint64_t PREFIX_MARK = 0xFFFFFFFFull;  // winner low bits of the index-0 metric-event record

struct DPView {
  const uint64_t *spos, *spay, *sgap;
  const uint32_t *srange, *gstart, *first_wge;
  const uint8_t* prevk;                // kind of the previous entry of the same (range, local id)
  const unsigned long long* unf;       // per range: min(first entry << 10 | local id) of unfinished work-items
  const uint32_t *bmin, *bmax;         // per range: min / max barrier count over work-items
  uint64_t S, NG;
  uint32_t lv, kb0;
  unsigned long long first_ke;
};

__device__ __forceinline__ bool is_open(uint32_t k) { return k == AIWC_K_WI_BEGIN || k == AIWC_K_WI_RESUME; }

// first failing check of entry s (0 = none); *at = event index, aux fields for the message
__device__ uint32_t check_entry(const DPView& v, uint64_t s, uint64_t* at, uint32_t* cls, uint64_t* aux_g,
                                uint64_t* aux_l) {
  const uint64_t pk = v.spos[s];
  const uint64_t pos = pk & 0xFFFFFFFFull;
  const uint32_t k = (uint32_t)(pk >> 32);
  const uint64_t p = v.spay[s];
  const uint32_t r = v.srange[s];
  *at = pos; *cls = 0;
  // state just before this event, under a valid prefix
  const bool ended = v.first_ke < pos;
  const bool header = pos != 0 && v.kb0;
  bool gopen = false;
  uint64_t gkey = 0;
  if (r != 0) {
    const uint64_t wgb = v.gstart[r - 1];
    gkey = v.spay[wgb];
    if (s == wgb) gopen = r >= 2 && v.first_wge[r - 1] == 0xFFFFFFFFu;  // the previous group never ended
    else gopen = s <= v.first_wge[r];
  }
  const bool prev_same = s > 0 && v.srange[s - 1] == r && s != (r ? (uint64_t)v.gstart[r - 1] : ~0ull);
  const uint32_t pk1 = prev_same ? (uint32_t)(v.spos[s - 1] >> 32) : 0u;
  const bool sopen = prev_same && is_open(pk1) && gopen;
  if (ended) return V_AFTER_KE;
  if (!header) {
    if (k != AIWC_K_KERNEL_BEGIN) return V_KB_NOT_FIRST;
  } else {
    switch (k) {
      case AIWC_K_BARRIER: if (!sopen) return V_BAR_OUTSIDE; break;
      case AIWC_K_KERNEL_BEGIN: return V_KB_DUP;
      case AIWC_K_KERNEL_END: if (gopen) return V_KE_OPEN_GROUP; break;
      case AIWC_K_WG_BEGIN: if (gopen) return V_WGB_OPEN; break;
      case AIWC_K_WG_END:
        if (!gopen || p != gkey) return V_WGE_MISMATCH;
        if (sopen) return V_WGE_OPEN_SEG;
        if (v.unf[r] != ~0ull) { *aux_g = gkey; *aux_l = v.unf[r] & 1023u; return V_UNFINISHED; }
        if (v.bmin[r] != 0xFFFFFFFFu && v.bmin[r] != v.bmax[r]) { *aux_g = gkey; return V_DIVERGENCE; }
        break;
      default:  // work-item events
        if (!gopen) return V_WI_OUTSIDE_GROUP;
        if (p >= v.lv) return V_WI_ID;
        if (k == AIWC_K_WI_BEGIN) {
          if (sopen) return V_OPEN_WHILE_OPEN;
          if (v.prevk[s] != PK_NONE) return V_WIB_STARTED;
        } else if (k == AIWC_K_WI_RESUME) {
          if (sopen) return V_OPEN_WHILE_OPEN;
          if (v.prevk[s] != AIWC_K_BARRIER) return V_WIR_NOT_BARRIER;
        } else {
          if (!sopen || v.spay[s - 1] != p) return V_WIE_NO_SEG;
        }
        break;
    }
  }
  // the first metric event of the gap after this one
  // (this event was valid: afterwards a segment is open iff it opened one)
  const uint64_t gp = v.sgap[s];
  if (gp != ~0ull) {
    *at = gp >> 8;
    if (v.first_ke <= pos) return V_AFTER_KE;
    if (!is_open(k)) { *cls = (uint32_t)(gp & 0xFF); return V_OUTSIDE_SEG; }
  }
  return V_NONE;
}

// sort keys: (range << lb | local id) << 32 | entry for work-item entries of a
// range up to its first wg_end (a barrier takes the local id of the segment it
// closes); everything else sorts last (~0)
__global__ void v_keys_kernel(const uint64_t* __restrict__ spos, const uint64_t* __restrict__ spay,
                              const uint32_t* __restrict__ srange, const uint32_t* __restrict__ gstart,
                              const uint32_t* __restrict__ first_wge, uint64_t S, uint32_t lv, int lb,
                              uint64_t* __restrict__ keys) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)(spos[s] >> 32), r = srange[s];
    uint64_t key = ~0ull;
    if (r != 0 && s < first_wge[r] && s != gstart[r - 1]) {
      uint64_t lid = ~0ull;
      if (k == AIWC_K_WI_BEGIN || k == AIWC_K_WI_RESUME || k == AIWC_K_WI_END) lid = spay[s];
      else if (k == AIWC_K_BARRIER && s > 0 && srange[s - 1] == r && is_open((uint32_t)(spos[s - 1] >> 32)))
        lid = spay[s - 1];
      if (lid < lv) key = ((((uint64_t)r << lb) | lid) << 32) | s;
    }
    keys[s] = key;
  }
}

// per sorted key: previous same-work-item kind; per work-item run (walked by its
// head): unfinished / barrier-count aggregates of its range
__global__ void v_runs_kernel(const uint64_t* __restrict__ keys, uint64_t S, const uint64_t* __restrict__ spos,
                              int lb, uint8_t* __restrict__ prevk, unsigned long long* unf, uint32_t* bmin,
                              uint32_t* bmax) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    if (key == ~0ull) continue;
    const uint64_t hi = key >> 32, s = key & 0xFFFFFFFFull;
    const bool head = i == 0 || (keys[i - 1] >> 32) != hi;
    prevk[s] = head ? PK_NONE : (uint8_t)(spos[keys[i - 1] & 0xFFFFFFFFull] >> 32);
    if (!head) continue;
    uint32_t nbar = 0, last = 0;
    for (uint64_t j = i; j < S && (keys[j] >> 32) == hi; ++j) {
      last = (uint32_t)(spos[keys[j] & 0xFFFFFFFFull] >> 32);
      nbar += last == AIWC_K_BARRIER;
    }
    const uint32_t r = (uint32_t)(hi >> lb);
    const uint64_t lid = hi & ((1ull << lb) - 1);
    if (last != AIWC_K_WI_END) atomicMin(&unf[r], (unsigned long long)((s << 10) | lid));
    atomicMin(&bmin[r], nbar);
    atomicMax(&bmax[r], nbar);
  }
}

__global__ void v_dp_check_kernel(DPView v, ValidateState* vs) {
  v.kb0 = vs->kb0;
  v.first_ke = vs->first_ke;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < v.S; s += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t at, ag = 0, al = 0;
    uint32_t cls;
    if (check_entry(v, s, &at, &cls, &ag, &al) != V_NONE) atomicMin(&vs->winner, (at << 32) | s);
  }
}

// the winner's record (and, for a barrier divergence, its range's counts)
__global__ void v_dp_record_kernel(DPView v, const uint64_t* __restrict__ keys, int lb, ValidateState* vs,
                                   ValidateRecord* rec, uint32_t* counts_buf, uint32_t counts_cap) {
  v.kb0 = vs->kb0;
  v.first_ke = vs->first_ke;
  const unsigned long long w = vs->winner;
  if (w == ~0ull || (w & 0xFFFFFFFFull) == PREFIX_MARK) return;
  const uint64_t s = w & 0xFFFFFFFFull;
  uint64_t at, ag = 0, al = 0;
  uint32_t cls;
  const uint32_t code = check_entry(v, s, &at, &cls, &ag, &al);
  rec->index = at; rec->code = code; rec->cls = cls; rec->group_key = ag; rec->local_id = al;
  rec->n_counts = 0; rec->counts_off = 0;
  if (code == V_DIVERGENCE) {
    const uint64_t r = v.srange[s];
    uint64_t a = 0, b = v.S;  // first key of range r
    while (a < b) {
      const uint64_t m = (a + b) / 2;
      if ((keys[m] >> 32) >> lb < r) a = m + 1; else b = m;
    }
    uint32_t m = 0, nbar = 0;
    for (uint64_t i = a; i < v.S && keys[i] != ~0ull && ((keys[i] >> 32) >> lb) == r && m < counts_cap; ++i) {
      nbar += (uint32_t)(v.spos[keys[i] & 0xFFFFFFFFull] >> 32) == AIWC_K_BARRIER;
      if (i + 1 == v.S || (keys[i + 1] >> 32) != (keys[i] >> 32)) { counts_buf[m++] = nbar; nbar = 0; }
    }
    rec->n_counts = m;
  }
}

__global__ void v_prefix_kernel(const uint8_t* kind, uint64_t n, ValidateState* vs, ValidateRecord* rec) {
  // a metric event at index 0 (no structural event before it): the header is missing
  if (n && metric(kind[0])) {
    rec->index = 0; rec->code = V_KB_NOT_FIRST; rec->cls = 0; rec->n_counts = 0;
    atomicMin(&vs->winner, PREFIX_MARK);
  }
}

}  // namespace

void validate_phase1(const uint8_t* kind, uint64_t n, ValidateState* vs, const ValidateBufs& b, cudaStream_t s,
                     int* kernels) {
  const uint64_t tiles = (n + VTILE - 1) / VTILE;
  if (!tiles) return;
  v_count_kernel<<<(unsigned)tiles, VT, 0, s>>>(kind, n, b.tile_s, b.tile_g, vs);
  ++*kernels;
  scan_exclusive_u32(b.tile_s, tiles, b.scan_scratch, &vs->n_struct, s, kernels);
  scan_exclusive_u32(b.tile_g, tiles, b.scan_scratch, &vs->n_groups, s, kernels);
}

static int bitwidth(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

namespace {
__global__ void vs_set_dp(ValidateState* vs) { vs->dp = 1; }
}  // namespace

void validate_phase2(const uint8_t* kind, const uint64_t* payload, uint64_t n, uint32_t lv, ValidateState* vs,
                     const ValidateBufs& b, uint64_t S, uint64_t NG, uint32_t n_ctas, bool force_replay,
                     cudaStream_t s, int* kernels) {
  const uint64_t tiles = (n + VTILE - 1) / VTILE;
  cudaMemsetAsync(b.first_wge, 0xFF, (NG + 1) * 4, s);
  if (tiles) {
    v_write_kernel<<<(unsigned)tiles, VT, 0, s>>>(kind, payload, n, b.tile_s, b.tile_g, b.spos, b.spay, b.sgap,
                                                  b.gstart, b.srange, b.first_wge);
    ++*kernels;
  }
  v_prefix_kernel<<<1, 1, 0, s>>>(kind, n, vs, b.recs + NG + 2);
  ++*kernels;
  const int lb = bitwidth(lv - 1), rb = bitwidth(NG + 1);
  if (rb + lb <= 32 && !force_replay) {  // data-parallel checker
    const unsigned grid = (unsigned)std::min<uint64_t>((S + 255) / 256 + 1, 148ull * 16);
    cudaMemsetAsync(b.prevk, 0xFF, std::max<uint64_t>(S, 1), s);
    cudaMemsetAsync(b.unf, 0xFF, (NG + 1) * 8, s);
    cudaMemsetAsync(b.bmin, 0xFF, (NG + 1) * 4, s);
    cudaMemsetAsync(b.bmax, 0, (NG + 1) * 4, s);
    v_keys_kernel<<<grid, 256, 0, s>>>(b.spos, b.spay, b.srange, b.gstart, b.first_wge, S, lv, lb, b.keys);
    radix_sort_u64(b.keys, b.keys_tmp, S, 32, 32 + rb + lb, b.sort_hist, s, kernels);
    v_runs_kernel<<<grid, 256, 0, s>>>(b.keys, S, b.spos, lb, b.prevk, b.unf, b.bmin, b.bmax);
    const DPView v{b.spos, b.spay, b.sgap, b.srange, b.gstart, b.first_wge, b.prevk, b.unf, b.bmin, b.bmax,
                   S, NG, lv, 0, 0};
    v_dp_check_kernel<<<grid, 256, 0, s>>>(v, vs);
    v_dp_record_kernel<<<1, 1, 0, s>>>(v, b.keys, lb, vs, b.recs + NG + 1, b.counts, b.counts_cap);
    *kernels += 4;
    vs_set_dp<<<1, 1, 0, s>>>(vs);
  } else {  // huge id spaces: replay each work-group range in one warp
    v_check_kernel<<<n_ctas, K2_WARPS * 32, 0, s>>>(b.spos, b.spay, b.sgap, S, b.gstart, NG, lv, vs, b.recs,
                                                    b.counts, b.counts_cap);
    ++*kernels;
  }
}

}  // namespace aiwc
