// aiwc_ingest.cu -- the streaming pass over the columnar trace.
//
// Replaces the per-event dispatch loop of the reference's consume()
// (pkg/src/aiwc/metrics.py:125-180).  Two launches:
//
//  pass1   P1_SUB CTAs per ingest range read ONLY the kind bytes (16 per
//          thread per load, nibble-packed SWAR popcounts) and write one
//          RangeSum per sub-range: per-class counts, the last work-item
//          boundary / work-group begin and the instructions after the last
//          boundary.  That is all the sequential state (open segment length,
//          open work-item, group) the next pass needs at its range start.
//  ingest  one persistent 256-thread CTA per range (two per SM).  Tiles of
//          4096 events arrive by TMA (kind rows + payload rows with 128 B
//          swizzle) through a 2-stage mbarrier ring; each thread owns 16
//          consecutive events.  An 8x8 bit-matrix transpose of the thread's
//          16 kind bytes gives one 16-bit mask per kind bit; a block scan of
//          the per-thread class counts gives every thread its exact carry-in
//          (segment length, work-item, group, output offsets).  Each event
//          class is then folded by its own converged set-bit loop:
//          instructions -> opcode / width bins counted from bit-planes (the
//          16 payloads' low bytes are packed and transposed like the kinds;
//          bin v's count is popc of its minterm, no per-event loop), memory ->
//          a per-warp list of event indices that the warp then folds into the
//          dense table with coalesced REDs (lane i takes the warp's i-th access,
//          so one RED instruction covers consecutive keys of streaming traces),
//          or ordered compaction; rare events in stream order -> segment
//          closes, branch records, group changes.  Segment closes are
//          histogrammed after the tile by all threads together.
#include <type_traits>

#include "aiwc_internal.cuh"

// AIWC_ABL: measurement-only ablation builds (tools/dbg/ablate.sh); 0 in the product
#ifndef AIWC_ABL
#define AIWC_ABL 0
#endif

namespace aiwc {

// ---------------------------------------------------------------------------
// pass 1
// ---------------------------------------------------------------------------
constexpr int P1_THREADS = 256;

__device__ __forceinline__ void load_kind16(const uint8_t* kind, uint64_t e0, uint64_t n, uint32_t w[4]) {
  if (e0 + 16 <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(kind + e0);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint64_t e = e0 + 4 * i + b;
        x |= (e < n ? (uint32_t)kind[e] : 0u) << (8 * b);
      }
      w[i] = x;
    }
  }
}

// Per-class counts of 16 kind bytes (w[i] = events 4i..4i+3).  Nibble packing:
// L0 / L1 hold bits 0..3 (instr, read, write, branch) of events 0..7 / 8..15,
// H0 / H1 bits 4..7 (boundary, open, group, variant): byte b of H0 has event b
// in its low nibble and event 4 + b in its high nibble (H1: 8 + b, 12 + b).
// Each class is one masked popcount per packed word; the boundary and
// work-group-begin positions stay in that nibble form (decoded once, at the end).
struct KindCounts {
  uint32_t instr = 0, rd = 0, wr = 0, br = 0, wgb = 0, bres = 0;
  // mb*: boundary bits (nibble bit 0), mw*: wg_begin bits (group bit without the variant bit)
  template <bool LIGHT>
  __device__ __forceinline__ void add(const uint32_t w[4], uint32_t& mb0, uint32_t& mb1, uint32_t& mw0,
                                      uint32_t& mw1, uint32_t& me0, uint32_t& me1) {
    const uint32_t L0 = (w[0] & 0x0F0F0F0Fu) | ((w[1] & 0x0F0F0F0Fu) << 4);
    const uint32_t L1 = (w[2] & 0x0F0F0F0Fu) | ((w[3] & 0x0F0F0F0Fu) << 4);
    const uint32_t H0 = ((w[0] >> 4) & 0x0F0F0F0Fu) | (w[1] & 0xF0F0F0F0u);
    const uint32_t H1 = ((w[2] >> 4) & 0x0F0F0F0Fu) | (w[3] & 0xF0F0F0F0u);
    rd += __popc(L0 & 0x22222222u) + __popc(L1 & 0x22222222u);
    wr += __popc(L0 & 0x44444444u) + __popc(L1 & 0x44444444u);
    if (!LIGHT) {  // (light: instructions are checked from the opcode counts, branches must be absent)
      instr += __popc(L0 & 0x11111111u) + __popc(L1 & 0x11111111u);
      br += __popc(L0 & 0x88888888u) + __popc(L1 & 0x88888888u);
    }
    mb0 = H0 & 0x11111111u;
    mb1 = H1 & 0x11111111u;
    mw0 = H0 & ~(H0 >> 1) & 0x44444444u;
    mw1 = H1 & ~(H1 >> 1) & 0x44444444u;
    me0 = H0 & (H0 >> 1) & 0x44444444u;  // wg_end: group bit with the variant bit
    me1 = H1 & (H1 >> 1) & 0x44444444u;
    wgb += __popc(mw0) + __popc(mw1);
    bres |= (H0 & (H0 >> 3)) | (H1 & (H1 >> 3));  // boundary with the variant bit: barrier / resume
  }
};

// last event index of a nibble-form mask pair of the chunk at e0 (-1 if none)
__device__ __forceinline__ long long last_nib_event(long long e0, uint32_t m0, uint32_t m1) {
  if (e0 < 0) return -1;
  if (m1 & 0xF0F0F0F0u) return e0 + 12 + ((31 - __clz(m1 & 0xF0F0F0F0u)) >> 3);
  if (m1 & 0x0F0F0F0Fu) return e0 + 8 + ((31 - __clz(m1 & 0x0F0F0F0Fu)) >> 3);
  if (m0 & 0xF0F0F0F0u) return e0 + 4 + ((31 - __clz(m0 & 0xF0F0F0F0u)) >> 3);
  if (m0 & 0x0F0F0F0Fu) return e0 + ((31 - __clz(m0 & 0x0F0F0F0Fu)) >> 3);
  return -1;
}

// LIGHT (declared totals, a dense table, no branches: nothing is staged): no
// instruction or branch counts -- finalize checks the declared instruction total
// against the opcode counts, and a branch makes the unstaged ingest fail
// (F_BAD_KIND); the carries use instr_after, which is the whole sub-range's
// instruction count when it holds no boundary.
template <bool LIGHT>
__global__ void __launch_bounds__(P1_THREADS) pass1_kernel(const uint8_t* __restrict__ kind,
                                                           const uint64_t* __restrict__ payload, uint64_t n,
                                                           uint32_t tiles_per_cta, bool with_stats,
                                                           RangeSum* __restrict__ out, DevState* st) {
  const uint64_t range_len = (uint64_t)tiles_per_cta * TILE;
  const uint64_t sub_len = range_len / P1_SUB;
  const uint32_t c = blockIdx.x / P1_SUB, sub = blockIdx.x % P1_SUB;
  const uint64_t rb = min(n, (uint64_t)c * range_len + sub * sub_len);
  const uint64_t re = min(n, rb + sub_len);
  const int t = threadIdx.x;
  KindCounts kc;
  long long lb_e0 = -1, lw_e0 = -1, le_e0 = -1;  // last chunk holding a boundary / wg_begin / wg_end, masks
  uint32_t lb_m0 = 0, lb_m1 = 0, lw_m0 = 0, lw_m1 = 0, le_m0 = 0, le_m1 = 0;
  unsigned long long amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  constexpr int U = 4;  // 16-byte loads in flight per thread
  for (uint64_t base = rb + 16ull * U * t; base < re; base += 16ull * U * P1_THREADS) {
    uint32_t w[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) load_kind16(kind, base + 16 * u, re, w[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t e0 = base + 16 * u;
      uint32_t mb0, mb1, mw0, mw1, me0, me1;
      kc.add<LIGHT>(w[u], mb0, mb1, mw0, mw1, me0, me1);
      if (mb0 | mb1) { lb_e0 = (long long)e0; lb_m0 = mb0; lb_m1 = mb1; }
      if (mw0 | mw1) { lw_e0 = (long long)e0; lw_m0 = mw0; lw_m1 = mw1; }
      if (me0 | me1) { le_e0 = (long long)e0; le_m0 = me0; le_m1 = me1; }
      if (with_stats) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t mm = w[u][i] & 0x06060606u;
          while (mm) {
            const int b = (__ffs(mm) - 1) >> 3;
            mm &= ~(0xFFu << (8 * b));
            const unsigned long long ad = payload[e0 + 4 * i + b];
            amin = min(amin, ad); amax = max(amax, ad); aand &= ad; aor |= ad;
          }
        }
      }
    }
  }
  long long last_bnd = last_nib_event(lb_e0, lb_m0, lb_m1), last_wgb = last_nib_event(lw_e0, lw_m0, lw_m1);
  long long last_wge = last_nib_event(le_e0, le_m0, le_m1);
  // block reduction
  constexpr int NW = P1_THREADS / 32;
  __shared__ uint32_t s_cnt[NW][6];
  __shared__ long long s_pos[NW][3];
  __shared__ unsigned long long s_addr[NW][4];
  __shared__ long long s_lb;
  uint32_t v[6] = {kc.instr, kc.rd, kc.wr, kc.br, kc.wgb, __reduce_or_sync(0xffffffffu, kc.bres & 0x11111111u) ? 1u : 0u};
  const int lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = warp_sum(v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    last_bnd = max(last_bnd, __shfl_xor_sync(0xffffffffu, last_bnd, o));
    last_wgb = max(last_wgb, __shfl_xor_sync(0xffffffffu, last_wgb, o));
    last_wge = max(last_wge, __shfl_xor_sync(0xffffffffu, last_wge, o));
    if (with_stats) {
      amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
      amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      aand &= __shfl_xor_sync(0xffffffffu, aand, o);
      aor |= __shfl_xor_sync(0xffffffffu, aor, o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) s_cnt[warp][i] = v[i];
    s_pos[warp][0] = last_bnd; s_pos[warp][1] = last_wgb; s_pos[warp][2] = last_wge;
    s_addr[warp][0] = amin; s_addr[warp][1] = amax; s_addr[warp][2] = aand; s_addr[warp][3] = aor;
  }
  __syncthreads();
  if (t == 0) {
    RangeSum r{};
    uint32_t tot[6] = {0};
    long long lb = -1, lw = -1, le = -1;
    unsigned long long mn = ~0ull, mx = 0, an = ~0ull, o = 0;
    for (int w = 0; w < NW; ++w) {
      for (int i = 0; i < 6; ++i) tot[i] += s_cnt[w][i];
      lb = max(lb, s_pos[w][0]); lw = max(lw, s_pos[w][1]); le = max(le, s_pos[w][2]);
      mn = min(mn, s_addr[w][0]); mx = max(mx, s_addr[w][1]); an &= s_addr[w][2]; o |= s_addr[w][3];
    }
    r.n_instr = tot[0]; r.n_rd = tot[1]; r.n_wr = tot[2]; r.n_br = tot[3];
    r.n_wgb = tot[4]; r.any_bres = tot[5] ? 1u : 0u;
    r.last_bnd = lb; r.last_wgb = lw; r.last_wge = le;
    out[blockIdx.x] = r;
    s_lb = lb;
    atomicAdd(&st->p1_tot[0], (unsigned long long)tot[0]);
    atomicAdd(&st->p1_tot[1], (unsigned long long)tot[1]);
    atomicAdd(&st->p1_tot[2], (unsigned long long)tot[2]);
    if (tot[3]) atomicAdd(&st->p1_tot[3], (unsigned long long)tot[3]);
    if (tot[4]) atomicAdd(&st->p1_tot[4], (unsigned long long)tot[4]);
    if (tot[5]) atomicAdd(&st->p1_tot[5], 1ull);
    if (with_stats && tot[1] + tot[2] > 0) {
      atomicMin(&st->addr_min, mn); atomicMax(&st->addr_max, mx);
      atomicAnd(&st->addr_and, an); atomicOr(&st->addr_or, o);
    }
  }
  __syncthreads();
  // instructions strictly after the sub-range's last boundary
  const long long lb = s_lb;
  uint32_t after = 0;
  const uint64_t start = lb < 0 ? rb : ((uint64_t)lb & ~15ull);
  for (uint64_t e0 = start + 16ull * t; e0 < re; e0 += 16ull * P1_THREADS) {
    uint32_t w[4];
    load_kind16(kind, e0, re, w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x = w[i] & 0x01010101u;
      const long long p0 = (long long)(e0 + 4 * i);
      if (p0 + 3 <= lb) x = 0;
      else if (p0 <= lb) x &= 0xFFFFFFFFu << (8 * (lb - p0 + 1));
      after += __popc(x);
    }
  }
  after = warp_sum(after);
  __shared__ uint32_t s_after[NW];
  if (lane == 0) s_after[warp] = after;
  __syncthreads();
  if (t == 0) {
    uint32_t a = 0;
    for (int w = 0; w < NW; ++w) a += s_after[w];
    out[blockIdx.x].instr_after = a;
  }
}

void launch_pass1(const uint8_t* kind, const uint64_t* payload, uint64_t n, uint32_t n_ranges, uint32_t tiles_per_cta,
                  bool with_stats, RangeSum* out, DevState* st, cudaStream_t s, bool light) {
  if (light)
    pass1_kernel<true><<<n_ranges * P1_SUB, P1_THREADS, 0, s>>>(kind, payload, n, tiles_per_cta, with_stats, out, st);
  else
    pass1_kernel<false><<<n_ranges * P1_SUB, P1_THREADS, 0, s>>>(kind, payload, n, tiles_per_cta, with_stats, out, st);
}

// ---------------------------------------------------------------------------
// main ingest pass
// ---------------------------------------------------------------------------
constexpr int NWARP = TPB / 32;
constexpr int WT = 32 * EPT;       // events per warp tile (one 16-event row per lane)
constexpr int WROWS = WT / 16;     // TMA box rows per warp tile
constexpr int WCL_CAP = 64;        // segment closes buffered per warp tile (overflow is processed inline)
constexpr uint32_t ACC_FLUSH_TILES = (65535 / EPT / PRES_TILES) * PRES_TILES;  // 16-bit fields take <= EPT per tile
static_assert(TILE == NWARP * WT && P1_SUB == NWARP && WT == WARP_TILE,
              "a CTA range is NWARP warp ranges (pass-1 sub-ranges) of the same tile count");

// TMA stages per warp (dynamic smem, 1024 B aligned for the 128 B swizzle):
// payload boxes [NWARP][STAGES][WT] u64, then kind boxes, then the mbarriers
struct StageSmem {
  uint64_t pay[NWARP][STAGES][WT];  // 16 B chunk c of box row r stored at chunk c ^ (r & 7)
  uint8_t kind[NWARP][STAGES][WT];
  uint64_t bar[NWARP][STAGES];
};

// CTA-private accumulators and per-warp scratch (static smem: direct addressing)
struct LocalSmem {
  uint16_t midx[NWARP][WT];       // per-warp memory-event list: tile position | write << 15
  uint32_t itb_h[HBINS];
  uint32_t ipt_h[HBINS];
  uint4 closes[NWARP][WCL_CAP];   // (segment length, local id, gseq | barrier << 31 | resumed << 30)
};

// 8x8 bit-matrix transpose: input byte i = event i (bit c = kind bit c);
// output byte c = kind bit c of events 0..7 (bit i = event i)
__device__ __forceinline__ uint64_t transpose8(uint64_t x) {
  uint64_t t;
  t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull; x ^= t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x ^= t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x ^= t ^ (t << 28);
  return x;
}

// Bit-planes 0..3 of the low nibbles of 16 bytes (b[q] = bytes of events
// 4q..4q+3).  Packing bytes q and q + 1 as nibbles puts event e + 4h, bit c
// at index [e1 e0 h c1 c0]; swapping index bits 4<->1 and 3<->0 (two delta
// swaps) gives index [c1 c0 h e1 e0] = byte c holds plane c of 8 events.
// Returns planes 0 | 1 << 16; planes 2 | 3 << 16 in p23.
__device__ __forceinline__ uint32_t nibble_planes(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3, uint32_t& p23) {
  uint32_t x = (b0 & 0x0F0F0F0Fu) | ((b1 & 0x0F0F0F0Fu) << 4);  // events 0..7
  uint32_t y = (b2 & 0x0F0F0F0Fu) | ((b3 & 0x0F0F0F0Fu) << 4);  // events 8..15
  uint32_t t;
  t = (x ^ (x >> 14)) & 0x0000CCCCu; x ^= t ^ (t << 14);
  t = (x ^ (x >> 7)) & 0x00AA00AAu; x ^= t ^ (t << 7);
  t = (y ^ (y >> 14)) & 0x0000CCCCu; y ^= t ^ (t << 14);
  t = (y ^ (y >> 7)) & 0x00AA00AAu; y ^= t ^ (t << 7);
  p23 = __byte_perm(x, y, 0x7362);
  return __byte_perm(x, y, 0x5140);
}

// bit 4 of each byte of x (events 4q..4q+3) as a 4-bit mask: the multiply moves
// bits 0, 8, 16, 24 to 21, 22, 23, 24 with no two partial products overlapping
__device__ __forceinline__ uint32_t bit4_nibble(uint32_t x) {
  return (((x >> 4) & 0x01010101u) * 0x00204081u >> 21) & 0xFu;
}

// Bin counts of 16 events from the 4 bit-planes of their values: bin v gets
// popc(minterm_v & fast), two bins per packed 32-bit counter (bin 2i low, 2i + 1
// high).  Planes 2 / 3 that no fast event of the warp sets are skipped
// (warp-uniform votes): traces with few opcode ids / narrow widths pay for 4 or 8
// minterms instead of 16.
__device__ __forceinline__ void bin_counts(uint32_t (&acc)[8], const uint32_t (&p)[4], uint32_t fast) {
  uint32_t q[4];
  q[0] = fast & ~p[0] & ~p[1]; q[1] = fast & p[0] & ~p[1]; q[2] = fast & ~p[0] & p[1]; q[3] = fast & p[0] & p[1];
  const bool hi3 = __any_sync(0xffffffffu, fast & p[3]);
  const bool hi2 = __any_sync(0xffffffffu, fast & p[2]);
  if (!hi3 && !hi2) {
    acc[0] += __popc(q[0]) + (__popc(q[1]) << 16);
    acc[1] += __popc(q[2]) + (__popc(q[3]) << 16);
  } else if (!hi3) {
    const uint32_t r[2] = {~p[2], p[2]};
#pragma unroll
    for (int v = 0; v < 8; v += 2)
      acc[v >> 1] += __popc(q[v & 3] & r[v >> 2]) + (__popc(q[(v + 1) & 3] & r[v >> 2]) << 16);
  } else {
    const uint32_t r[4] = {~p[2] & ~p[3], p[2] & ~p[3], ~p[2] & p[3], p[2] & p[3]};
#pragma unroll
    for (int v = 0; v < 16; v += 2)
      acc[v >> 1] += __popc(q[v & 3] & r[v >> 2]) + (__popc(q[(v + 1) & 3] & r[v >> 2]) << 16);
  }
}

// One segment close (metrics.py:156-174): ITB sample (barrier always, wi_end when
// non-empty); IPT either straight to the histogram (work-item never crossed a
// barrier) or accumulated in the work-item's lifetime slot.
__device__ __forceinline__ void do_close(LocalSmem& L, const IngestArgs& a, uint32_t seg, uint32_t lid, uint32_t gz,
                                         uint64_t pos, unsigned long long& itb_sum, unsigned long long& ipt_sum,
                                         unsigned long long& flags) {
  const bool bar = gz >> 31, byres = (gz >> 30) & 1u;
  const uint32_t gseq = gz & 0x3FFFFFFFu;
  if (a.dup_bits) {
    // in-pass check, per segment: the opener's local id inside the group, and for a
    // wi_begin-opened segment its (group, lid) bit (RED, no round trip); finalize
    // compares the set bits with the begins
    const uint64_t slot = (uint64_t)(gseq - 1) * a.local_volume + lid;
    if (lid >= a.local_volume || !gseq || slot >= a.dup_len) flags |= F_STREAM;
    else if (!byres && !(AIWC_ABL & 128)) atomicOr(&a.dup_bits[slot >> 5], 1u << (slot & 31));
  }
  if (a.wi_rules && !(AIWC_ABL & 256)) {  // per-work-item order (stream check of barrier / resume traces)
    const uint64_t slot = (uint64_t)(gseq - 1) * a.local_volume + lid;
    if (gseq == 0 || slot >= a.dup_len) {
      flags |= F_STREAM;
    } else {
      unsigned long long* const w = a.wi_rules + 3 * slot;
      atomicMax(w, ~((pos << 1) | (byres ? 1ull : 0ull)));     // the first segment: opened by wi_begin
      atomicMax(w + 1, ((pos + 1) << 1) | (bar ? 0ull : 1ull));  // the last: closed by wi_end
      atomicAdd(w + 2, bar ? 1ull : (1ull << 32));               // barriers | ends << 32
    }
  }
  if (bar || seg) {
    if (seg < (uint32_t)HBINS) atomicAdd(&L.itb_h[seg], 1u);
    else a.itb_ovf[atomicAdd(&a.st->itb_ovf_n, 1ull)] = seg;
    itb_sum += seg;
  }
  if (bar || byres) {
    const uint64_t slot = (uint64_t)(gseq - 1) * a.local_volume + lid;
    if (gseq == 0 || slot >= a.ipt_tab_len) flags |= F_SLOT_RANGE;
    else atomicAdd(&a.ipt_tab[slot], (unsigned long long)seg + (bar ? 0ull : IPT_END_FLAG));
  } else {
    if (seg < (uint32_t)HBINS) atomicAdd(&L.ipt_h[seg], 1u);
    else a.ipt_ovf[atomicAdd(&a.st->ipt_ovf_n, 1ull)] = seg;
    ipt_sum += seg;
  }
}

// add the per-thread packed bin counters (16-bit fields, bin 2i low / 2i + 1 high)
// to the global opcode / width counters; warp-converged.  Opcode bin v = opcode v,
// width bin v = width v + 1.
__device__ __forceinline__ void flush_counts(uint32_t (&oacc)[8], uint32_t (&wacc)[8], const IngestArgs& a, int lane,
                                             unsigned long long& flags) {
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    uint32_t co = (oacc[v >> 1] >> (16 * (v & 1))) & 0xFFFFu;
    uint32_t cw = (wacc[v >> 1] >> (16 * (v & 1))) & 0xFFFFu;
    co = warp_sum(co);
    cw = warp_sum(cw);
    if (lane == 0) {
      if (co) {
        atomicAdd(&a.opc_counts[v], (unsigned long long)co);
        if ((uint32_t)v >= a.n_opcodes) flags |= F_BAD_OPCODE;
      }
      if (cw) atomicAdd(&a.width_count[v + 1], (unsigned long long)cw);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) { oacc[i] = 0; wacc[i] = 0; }
}

// shared-memory slot of hot-window key `rel`: the low 5 bits XOR the next 5 (an
// involution inside every 1024 keys), so strided key patterns -- a scratch indexed
// by 4 * lid + i -- spread over all 32 banks instead of 8
__device__ __forceinline__ uint32_t hot_swz(uint32_t rel) { return rel ^ ((rel >> 5) & 31u); }

__device__ __forceinline__ uint64_t pay_at(const uint64_t* pay, uint32_t pos) {
  return pay[pos ^ (((pos >> 4) & 7u) << 1)];  // 128 B swizzle: chunk (j >> 1) ^ (row & 7)
}

// The ingest: every warp owns one contiguous warp range of the trace (pass 1's
// sub-range c * P1_SUB + warp) and walks it in 512-event warp tiles through its
// own 2-stage TMA ring -- no CTA barrier inside the loop.  Each lane holds one
// 16-event row of the tile; a warp scan of packed class counts gives every lane
// its exact carry-in; lane 31's end state is the next tile's carry-in.
// compiled-in features (a trace that needs none runs the plain variant)
enum : int { FEAT_CHECK = 1, FEAT_BINS = 2, FEAT_MARK = 4 };

template <bool DENSE, bool STAGE, int FEAT>
__global__ void __launch_bounds__(TPB, 2)
    ingest_kernel(const IngestArgs a, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap pmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ LocalSmem L;
  // 1024 B alignment for the swizzle; pointer arithmetic on the shared array
  // keeps the accesses in the shared window
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  StageSmem& S = *reinterpret_cast<StageSmem*>(smem_raw + pad);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // small dense tables: per-CTA read / write counters after the TMA stages
  uint32_t* const stab = reinterpret_cast<uint32_t*>(smem_raw + pad + sizeof(StageSmem));
  const uint64_t n = a.n;
  const uint64_t n_wtiles = (n + WT - 1) / WT;
  const uint32_t gw = blockIdx.x * NWARP + warp;  // == pass 1 sub-range index
  const uint64_t wt_begin = (uint64_t)gw * a.tiles_per_cta;
  const uint32_t my_tiles = wt_begin < n_wtiles ? (uint32_t)min((uint64_t)a.tiles_per_cta, n_wtiles - wt_begin) : 0u;
  DevState* st = a.st;
  uint64_t* const bars = S.bar[warp];

  // ---- prologue: smem init + this warp's TMA ring fill ----
  for (int i = t; i < HBINS; i += TPB) { L.itb_h[i] = 0; L.ipt_h[i] = 0; }
  for (uint32_t i = t; i < 2 * a.smem_keys; i += TPB) stab[i] = 0;
  // shared-memory window of the dense table: [hot_lo, hot_lo + hot_n)
  const uint64_t hot_lo = a.hot_dev ? *a.hot_dev : a.hot_lo;
  const uint32_t hot_n = hot_lo == ~0ull ? 0u : a.smem_keys;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    for (uint32_t it = 0; it < (uint32_t)STAGES && it < my_tiles; ++it) {
      const uint64_t row0 = (wt_begin + it) * WROWS;
      if (row0 < a.tma_rows) {
        mbar_expect_tx(&bars[it], WT * 9);
        tma_load_2d(S.kind[warp][it], &kmap, 0, (int)row0, &bars[it]);
        tma_load_2d(S.pay[warp][it], &pmap, 0, (int)row0, &bars[it]);
      }
    }
  }

  // ---- carry-in at the start of this warp's range: combine the sub-ranges before it ----
  uint32_t cseg = 0, clid = 0, cbyres = 0, cgseq = 0, cgkey = 0;
  uint32_t cso = 0, cgo = 0;  // stream check: a segment / a work-group is open
  unsigned long long c_rd = 0, c_wr = 0, c_br = 0;
  {
    const uint32_t c = blockIdx.x * P1_SUB;  // CTA-wide part: sub-ranges [0, c)
    long long jb = -1, lw = -1, lwe = -1;
    uint64_t s_rd = 0, s_wr = 0, s_br = 0, s_wgb = 0;
    for (uint32_t j = t; j < c; j += TPB) {
      const RangeSum& r = a.ranges[j];
      if (r.last_bnd >= 0) jb = max(jb, (long long)j);
      lw = max(lw, (long long)r.last_wgb);
      lwe = max(lwe, (long long)r.last_wge);
      s_rd += r.n_rd; s_wr += r.n_wr; s_br += r.n_br; s_wgb += r.n_wgb;
    }
    __shared__ unsigned long long red[NWARP][7];
    s_rd = warp_sum(s_rd); s_wr = warp_sum(s_wr); s_br = warp_sum(s_br); s_wgb = warp_sum(s_wgb);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      jb = max(jb, __shfl_xor_sync(0xffffffffu, jb, o));
      lw = max(lw, __shfl_xor_sync(0xffffffffu, lw, o));
      lwe = max(lwe, __shfl_xor_sync(0xffffffffu, lwe, o));
    }
    if (lane == 0) {
      red[warp][0] = s_rd; red[warp][1] = s_wr; red[warp][2] = s_br; red[warp][3] = s_wgb;
      red[warp][4] = (unsigned long long)jb; red[warp][5] = (unsigned long long)lw;
      red[warp][6] = (unsigned long long)lwe;
    }
    __syncthreads();
    jb = -1; lw = -1; lwe = -1; s_rd = s_wr = s_br = s_wgb = 0;
    for (int w = 0; w < NWARP; ++w) {
      s_rd += red[w][0]; s_wr += red[w][1]; s_br += red[w][2]; s_wgb += red[w][3];
      jb = max(jb, (long long)red[w][4]); lw = max(lw, (long long)red[w][5]); lwe = max(lwe, (long long)red[w][6]);
    }
    uint64_t s_in = 0;  // instructions after the last boundary: after(jb) + instrs of later sub-ranges
    // (instr_after = all of a sub-range's instructions when it holds no boundary)
    for (uint32_t j = (uint32_t)(jb + 1) + t; j < c; j += TPB) s_in += a.ranges[j].instr_after;
    s_in = warp_sum(s_in);
    __syncthreads();
    if (lane == 0) red[warp][0] = s_in;
    __syncthreads();
    uint64_t after = 0;
    for (int w = 0; w < NWARP; ++w) after += red[w][0];
    long long lbpos = -1;
    if (jb >= 0) {
      lbpos = a.ranges[jb].last_bnd;
      after += a.ranges[jb].instr_after;
    }
    // warp part: this CTA's sub-ranges before mine, in order
    for (uint32_t j = c; j < c + (uint32_t)warp; ++j) {
      const RangeSum& r = a.ranges[j];
      if (r.last_bnd >= 0) { lbpos = r.last_bnd; after = r.instr_after; }
      else after += r.instr_after;
      if (r.last_wgb >= 0) lw = r.last_wgb;
      if (r.last_wge >= 0) lwe = r.last_wge;
      s_rd += r.n_rd; s_wr += r.n_wr; s_br += r.n_br; s_wgb += r.n_wgb;
    }
    if (lbpos >= 0) {
      clid = (uint32_t)a.payload[lbpos];
      cbyres = a.kind[lbpos] == AIWC_K_WI_RESUME;
      // stream check: a segment is open when the last boundary opened one after the last group event
      cso = (a.kind[lbpos] & 0x20) && lbpos > max(lw, lwe);
    }
    cgo = lw > lwe;
    cseg = (uint32_t)after;
    c_rd = s_rd; c_wr = s_wr; c_br = s_br;
    cgseq = (uint32_t)s_wgb;
    cgkey = lw >= 0 ? (uint32_t)a.payload[lw] : 0u;
  }
  __syncthreads();

  uint32_t oacc[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // opcode bins 0..15, two 16-bit fields each
  uint32_t wacc[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // width bins (bin v = width v + 1)
  uint32_t pres = 0;                                     // slow-path widths 1..16 seen in this presence block
  uint32_t wsnap[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // width counters at the block start
  // widths 1..16 that occurred in presence block `blk` (PRES_TILES warp tiles) of this warp range
  auto record_presence = [&](uint32_t blk) {
    uint32_t bits = pres;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t d = wacc[i] ^ wsnap[i];
      if (d & 0xFFFFu) bits |= 1u << (2 * i);
      if (d >> 16) bits |= 1u << (2 * i + 1);
      wsnap[i] = wacc[i];
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0 && bits) a.width_presence[(uint64_t)gw * a.pres_blocks + blk] = bits;
    pres = 0;
  };
  unsigned long long itb_sum = 0, ipt_sum = 0, flags = 0, max_site = 0;
  unsigned long long amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  uint32_t n_wib = 0, n_bar = 0;  // WI_BEGIN / BARRIER events (metrics.py: work_items, barriers_hit)
  const uint32_t sw = lane & 7, sw2 = sw << 1;
  uint4* const wclose = L.closes[warp];
  uint32_t last_ch = ~0u, last_ch2 = ~0u;  // shard: the last two chunks this lane marked
  // key-block bins: this warp range's segment of the bin buffer and its fill
  constexpr bool CHECK = FEAT & FEAT_CHECK, BINS = DENSE && (FEAT & FEAT_BINS), MARKS = DENSE && (FEAT & FEAT_MARK);
  const unsigned long long zmask = BINS ? *a.bin_zones : 0ull;
  const unsigned long long bin_base0 = c_rd + c_wr;
  uint32_t bfill = 0;
  if (BINS && zmask && lane == 0) a.bin_base[gw] = bin_base0;

  for (uint32_t it = 0; it < my_tiles; ++it) {
    const int s = it % STAGES;
    const uint64_t wt = wt_begin + it;
    const uint64_t tile0 = wt * WT;
    const uint64_t row0 = wt * WROWS;
    const uint64_t* const P = S.pay[warp][s];
    uint8_t* const K = S.kind[warp][s];
    if (row0 < a.tma_rows) mbar_wait(&bars[s], (it / STAGES) & 1);
    const uint64_t e0 = tile0 + 16ull * lane;
    uint32_t w[4];
    if (row0 + lane < a.tma_rows) {
      const uint4 v = *reinterpret_cast<const uint4*>(&K[16 * lane]);
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      // rows beyond the tensor maps (tail of the trace): direct loads, patch smem
      load_kind16(a.kind, e0, n, w);
      *reinterpret_cast<uint4*>(&K[16 * lane]) = make_uint4(w[0], w[1], w[2], w[3]);
      for (int j = 0; j < 16; ++j) {
        const uint64_t e = e0 + j;
        S.pay[warp][s][lane * 16 + ((((j >> 1) ^ sw)) << 1) + (j & 1)] = e < n ? a.payload[e] : 0ull;
      }
    }
    if (row0 + WROWS > a.tma_rows) __syncwarp();  // patched rows are read by other lanes
    // ---- kind bit-planes of my 16 events: plane c bit j = bit c of kind byte j ----
    uint32_t ins16, rd16, wr16, br16, bnd16, p5, p6, p7;
    {
      const uint64_t x0 = transpose8((uint64_t)w[0] | ((uint64_t)w[1] << 32));
      const uint64_t x1 = transpose8((uint64_t)w[2] | ((uint64_t)w[3] << 32));
      const uint32_t a01 = __byte_perm((uint32_t)x0, (uint32_t)x1, 0x5140);
      const uint32_t a23 = __byte_perm((uint32_t)x0, (uint32_t)x1, 0x7362);
      const uint32_t b45 = __byte_perm((uint32_t)(x0 >> 32), (uint32_t)(x1 >> 32), 0x5140);
      const uint32_t b67 = __byte_perm((uint32_t)(x0 >> 32), (uint32_t)(x1 >> 32), 0x7362);
      ins16 = a01 & 0xFFFFu; rd16 = a01 >> 16; wr16 = a23 & 0xFFFFu; br16 = a23 >> 16;
      bnd16 = b45 & 0xFFFFu; p5 = b45 >> 16; p6 = b67 & 0xFFFFu; p7 = b67 >> 16;
    }
    {  // kind bytes outside the columnar alphabet (include/aiwc_b200.h)
      const uint32_t lo4 = ins16 | rd16 | wr16 | br16, hi3 = bnd16 | p5 | p6;
      const uint32_t bad = (ins16 & (rd16 | wr16 | br16)) | (rd16 & (wr16 | br16)) | (wr16 & br16) | (lo4 & hi3) |
                           (p7 & (ins16 | br16)) | (p7 & ~(rd16 | wr16 | hi3)) | (p6 & (bnd16 | p5));
      if (bad) flags |= F_BAD_KIND;
    }
    n_wib += __popc(bnd16 & p5 & ~p7);
    n_bar += __popc(bnd16 & ~p5 & p7);
    const uint32_t close16 = bnd16 & ~p5;          // barrier / wi_end
    const uint32_t wgb16 = p6 & ~p7;               // wg_begin
    const uint32_t rare16 = bnd16 | p5 | p6;       // boundary, group, kernel events
    const int lp = bnd16 ? 31 - __clz(bnd16) : -1;
    const int lw = wgb16 ? 31 - __clz(wgb16) : -1;
    const uint32_t n_in = __popc(ins16);
    const uint32_t after = __popc(ins16 >> (lp + 1));
    // ---- warp scan of 10-bit fields (counts <= 512):
    //      X = instr | branch << 10 | read << 20, Y = write | wgb << 10 | close << 20 ----
    const uint32_t n_rd = __popc(rd16), n_wr = __popc(wr16);
    const uint32_t X = n_in | (__popc(br16) << 10) | (n_rd << 20);
    const uint32_t Y = n_wr | (__popc(wgb16) << 10) | (__popc(close16) << 20);
    uint32_t Xi = X, Yi = Y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ux = __shfl_up_sync(0xffffffffu, Xi, o), uy = __shfl_up_sync(0xffffffffu, Yi, o);
      if (lane >= o) { Xi += ux; Yi += uy; }
    }
    const uint32_t TX = __shfl_sync(0xffffffffu, Xi, 31), TY = __shfl_sync(0xffffffffu, Yi, 31);
    const uint32_t Xex = Xi - X, Yex = Yi - Y;
    const uint32_t ex_in = Xex & 0x3FFu, ex_br = (Xex >> 10) & 0x3FFu, ex_rd = Xex >> 20;
    const uint32_t ex_wr = Yex & 0x3FFu, ex_wgb = (Yex >> 10) & 0x3FFu, ex_cl = Yex >> 20;
    const uint32_t T_br = (TX >> 10) & 0x3FFu, T_rd = TX >> 20, T_wr = TY & 0x3FFu, T_cl = TY >> 20;
    // the last boundary / wg_begin before my row: the nearest lower lane holding one (ballot),
    // its position and (boundary) its count of instructions at positions <= it
    const uint32_t below = (1u << lane) - 1u;
    const uint32_t bl = __ballot_sync(0xffffffffu, bnd16 != 0) & below;
    const uint32_t gl = __ballot_sync(0xffffffffu, wgb16 != 0) & below;
    const uint32_t Lb = bl ? 31u - __clz(bl) : 0u, Lg = gl ? 31u - __clz(gl) : 0u;
    const uint32_t bsrc = __shfl_sync(0xffffffffu, (uint32_t)(lp + 1) | ((ex_in + n_in - after) << 16), Lb);
    const uint32_t gsrc = __shfl_sync(0xffffffffu, (uint32_t)(lw + 1), Lg);
    const uint32_t Pex = bl ? 16u * Lb + (bsrc & 0xFFFFu) : 0u, Qex = gl ? 16u * Lg + gsrc : 0u;
    const uint32_t vsrc = bsrc >> 16;
    // ---- carry-in for this lane ----
    uint32_t seg_in, lid, byres;
    if (Pex) {
      const uint32_t pos = Pex - 1;
      seg_in = ex_in - vsrc;
      lid = (uint32_t)pay_at(P, pos);
      byres = K[pos] == AIWC_K_WI_RESUME;
    } else {
      seg_in = cseg + ex_in; lid = clid; byres = cbyres;
    }
    uint32_t gkey = Qex ? (uint32_t)pay_at(P, Qex - 1) : cgkey;
    uint32_t gseq = cgseq + ex_wgb;
    // ---- stream check, bit-parallel over my row (no per-event branches) ----
    // Segment events (opens / closes) and group events (wg_begin / wg_end) must each
    // alternate; given that, the open / closed state at every position is a parity:
    // the carried state XOR the boundaries up to it.  The state at my row's start is the
    // tile's carried state XOR the parity of all lower lanes' boundaries (one ballot).
    uint32_t so = 0, go = 0;
    if (CHECK) {
      // segment opens: wi_begin, and wi_resume when the per-work-item rules run (a.wi_open)
      const uint32_t ko = bnd16 & p5 & (a.wi_rules ? 0xFFFFu : ~p7);
      const uint32_t kc = bnd16 & ~p5;                           // wi_end / barrier
      const uint32_t gb = wgb16, ge = p6 & p7;                   // wg_begin, wg_end
      const uint32_t kb = p5 & ~bnd16 & ~p6 & ~p7, ke = p5 & ~bnd16 & ~p6 & p7;  // kernel begin / end
      const uint32_t X = bnd16, G = gb | ge;
      so = cso ^ (__popc(__ballot_sync(0xffffffffu, __popc(X) & 1u) & below) & 1u);
      go = cgo ^ (__popc(__ballot_sync(0xffffffffu, __popc(G) & 1u) & below) & 1u);
      // inclusive / exclusive prefix parities (bit j: boundaries at positions <= j / < j)
      uint32_t px = X, pg = G;
      px ^= px << 1; px ^= px << 2; px ^= px << 4; px ^= px << 8;
      pg ^= pg << 1; pg ^= pg << 2; pg ^= pg << 4; pg ^= pg << 8;
      const uint32_t seg_in = ((so ? 0xFFFFu : 0u) ^ px) & 0xFFFFu;          // segment open after position j
      const uint32_t seg_before = seg_in ^ X;                                 // ... before position j
      const uint32_t grp_in = ((go ? 0xFFFFu : 0u) ^ pg) & 0xFFFFu, grp_before = grp_in ^ G;
      const uint32_t metric16 = ins16 | rd16 | wr16 | br16;
      const uint32_t bad =
          (metric16 & ~seg_in) |                  // metric event outside a segment
          (ko & seg_before) | (kc & ~seg_before) |  // segments alternate: open when closed, close when open
          (X & ~grp_before) |                     // work-item events inside a work-group only
          (gb & grp_before) | (ge & ~grp_before) |  // groups alternate
          (G & seg_before) |                      // no group event inside a segment
          (a.wi_rules ? 0u : bnd16 & p7 & ~kc) |  // wi_resume without the per-work-item rules: the full validator's case
          (kb & ~(e0 == 0 ? 1u : 0u)) |           // kernel_begin is event 0 ...
          (ke & ~((n - 1 >= e0 && n - 1 < e0 + 16) ? (1u << (uint32_t)(n - 1 - e0)) : 0u)) |  // ... kernel_end the last
          (ke & grp_before);                      // ... with no work-group open
      if (bad && !(AIWC_ABL & 32)) flags |= F_STREAM;
      // the trace starts with kernel_begin and ends with kernel_end
      if (e0 == 0 && !(kb & 1u)) flags |= F_STREAM;
      if (n - 1 >= e0 && n - 1 < e0 + 16 && !((ke >> (uint32_t)(n - 1 - e0)) & 1u)) flags |= F_STREAM;
      // the next tile's carried state
      const uint32_t all_x = __popc(__ballot_sync(0xffffffffu, __popc(X) & 1u)) & 1u;
      const uint32_t all_g = __popc(__ballot_sync(0xffffffffu, __popc(G) & 1u)) & 1u;
      cso ^= all_x;
      cgo ^= all_g;
    }
    // ordered outputs go straight to their global slots (range offset + exclusive rank)
    uint64_t o_rd = c_rd + ex_rd, o_wr = c_wr + ex_wr;
    const uint64_t o_br = c_br + ex_br;
    uint32_t o_cl = ex_cl;
    // ---- fold my 16 events, one converged loop per event class ----
    // 128 B swizzle: event j of row r sits at u64 index 16 r + (j ^ ((r & 7) << 1))
    const uint64_t* prow = &P[lane * 16];
#define PAY(j) prow[(uint32_t)(j) ^ sw2]
    // instructions: opcode / width bins from bit-planes.  The fast bins take
    // opcode < 16 and width 1..16: min(opcode, 16) and min(width - 1, 16) keep
    // one byte each, bit 4 of those bytes flags the rest, and the low nibbles are
    // transposed into 4 planes each; bin v counts popc(minterm_v & fast).
    uint32_t bad = 0;  // events outside the fast bins (meaningful for instructions only)
    uint32_t op[4], wp[4];
    {
      const uint4* prow4 = reinterpret_cast<const uint4*>(prow);
      uint32_t lo2[8], hi2[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // chunk c = events 2c, 2c + 1
        const uint4 v = prow4[c ^ sw];
        lo2[c] = __byte_perm(min(v.x - 1u, 16u), min(v.z - 1u, 16u), 0x0040);  // width - 1 of events 2c, 2c + 1
        hi2[c] = __byte_perm(min(v.y, 16u), min(v.w, 16u), 0x0040);            // opcode
      }
      uint32_t lw4[4], hw4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lw4[q] = __byte_perm(lo2[2 * q], lo2[2 * q + 1], 0x5410);
        hw4[q] = __byte_perm(hi2[2 * q], hi2[2 * q + 1], 0x5410);
        if (!(AIWC_ABL & 16)) bad |= bit4_nibble(lw4[q] | hw4[q]) << (4 * q);
      }
      uint32_t o23, w23;
      const uint32_t o01 = nibble_planes(hw4[0], hw4[1], hw4[2], hw4[3], o23);
      const uint32_t w01 = nibble_planes(lw4[0], lw4[1], lw4[2], lw4[3], w23);
      op[0] = o01 & 0xFFFFu; op[1] = o01 >> 16; op[2] = o23 & 0xFFFFu; op[3] = o23 >> 16;
      wp[0] = w01 & 0xFFFFu; wp[1] = w01 >> 16; wp[2] = w23 & 0xFFFFu; wp[3] = w23 >> 16;
    }
    if (!(AIWC_ABL & 1)) {
      const uint32_t fast = ins16 & ~bad;
      bin_counts(oacc, op, fast);
      bin_counts(wacc, wp, fast);
    }
    // the rest one by one: opcodes >= 16, widths outside 1..16
    for (uint32_t m = ins16 & bad; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint64_t p = PAY(j);
      const uint32_t opc = (uint32_t)(p >> 32), wd = (uint32_t)p;
      if (opc < a.n_opcodes) atomicAdd(&a.opc_counts[opc], 1ull);
      else flags |= F_BAD_OPCODE;
      if (wd < WIDTH_TABLE) {
        atomicAdd(&a.width_count[wd], 1ull);
        if (wd - 1u < (uint32_t)WBINS) pres |= 1u << (wd - 1);  // first index found after the pass
        else { atomicMin(&a.width_first[wd], (unsigned long long)(e0 + j)); atomicMax(&a.st->max_width, (unsigned long long)wd); }
      } else {
        flags |= F_BAD_WIDTH;
      }
    }
    // memory accesses: dense-table counters (warp-coalesced) or ordered compaction
    if (DENSE && !(AIWC_ABL & 2)) {
      // my accesses go to the warp's list (pre-swizzled smem index | write << 15)
      // at my in-warp exclusive offset ...
      uint16_t* const midx = L.midx[warp];
      uint32_t slot = ex_rd + ex_wr;
      const uint32_t rowb = 16u * lane;
      for (uint32_t m = rd16 | wr16; m; m &= m - 1) {
        const uint32_t j = __ffs(m) - 1;
        midx[slot++] = (uint16_t)((rowb | (j ^ sw2)) | (((wr16 >> j) & 1u) << 15));
      }
      __syncwarp();
      // ... and lane i folds accesses i, i + 32, ... of the warp in stream order, so one
      // RED instruction covers consecutive keys of streaming traces.  An address outside
      // the declared statistics is counted into the sentinel slot n_keys (and flagged).
      const uint32_t n_mem = T_rd + T_wr;
      const uint64_t base = a.am.base, off_max = a.am.off_max;
      const uint32_t k = a.am.k, lmask = (uint32_t)a.am.low_mask, lconst = (uint32_t)a.am.low_const;
      uint32_t inval = 0;
      // the window check and the shard's chunk marks are compiled in only when
      // needed (CTA-uniform branches)
      auto fold = [&](auto with_window, auto with_marks) {
        constexpr bool HOT = decltype(with_window)::value;
        constexpr bool MARK = decltype(with_marks)::value;
        // shard: bit (key >> 10) of the touched-chunk map -- checked only for a chunk
        // neither of this lane's last two marks holds (they persist across tiles: reads
        // and writes of streaming traces alternate between two chunks), and set only
        // when not set yet (a plain load first: the map is small and L1 / L2 resident,
        // same-word REDs are not)
        auto mark = [&](uint64_t key) {
          if (MARK) {
            const uint32_t ch = (uint32_t)(key >> 10);
            if (ch != last_ch && ch != last_ch2) {
              last_ch2 = last_ch;
              last_ch = ch;
              const uint32_t bit = 1u << (ch & 31);
              if (!(a.chunk_bits[ch >> 5] & bit)) atomicOr(&a.chunk_bits[ch >> 5], bit);
            }
          }
        };
        if (a.dense32) {
          uint32_t* const tab = static_cast<uint32_t*>(a.dense);
#pragma unroll 4  // several accesses per lane in flight
          for (uint32_t i = lane; i < n_mem; i += 32) {
            const uint32_t e = midx[i];
            const uint64_t off = P[e & 0x0FFFu] - base;
            const bool v = (off <= off_max) & (((uint32_t)off & lmask) == lconst);
            inval |= !v;
            const uint64_t key = v ? off >> k : a.am.n_keys, rel = key - hot_lo;
            mark(key);
            if (HOT && rel < hot_n) {
              atomicAdd(&stab[((e >> 15) ? hot_n : 0u) + hot_swz((uint32_t)rel)], 1u);
            } else {
              uint32_t* const q = tab + key;
              atomicAdd(q, 1u);
              if (!(AIWC_ABL & 4)) atomicOr(q, E32_READ << (e >> 15));
            }
          }
        } else {
          unsigned long long* const tab = static_cast<unsigned long long*>(a.dense);
#pragma unroll 4  // several accesses per lane in flight
          for (uint32_t i = lane; i < n_mem; i += 32) {
            const uint32_t e = midx[i];
            const uint64_t off = P[e & 0x0FFFu] - base;
            const bool v = (off <= off_max) & (((uint32_t)off & lmask) == lconst);
            inval |= !v;
            const uint64_t key = v ? off >> k : a.am.n_keys, rel = key - hot_lo;
            mark(key);
            if (HOT && rel < hot_n) atomicAdd(&stab[((e >> 15) ? hot_n : 0u) + hot_swz((uint32_t)rel)], 1u);
            else atomicAdd(tab + key, 1ull << (32 * (e >> 15)));
          }
        }
      };
      // key-block bins: whole-warp rounds (a ballot places the appended entries);
      // accesses into a random zone go to the warp's bin segment, the rest as above
      auto fold_bins = [&](auto with_window) {
        constexpr bool HOT = decltype(with_window)::value;
        uint32_t* const seg = a.bin_seg + bin_base0;
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 2
        for (uint32_t b0 = 0; b0 < n_mem; b0 += 32) {
          const uint32_t i = b0 + lane;
          const bool act = i < n_mem;
          const uint32_t e = act ? midx[i] : 0u;
          const uint64_t off = P[e & 0x0FFFu] - base;
          const bool v = act & (off <= off_max) & (((uint32_t)off & lmask) == lconst);
          inval |= act & !v;
          const uint64_t key = v ? off >> k : a.am.n_keys, rel = key - hot_lo;
          const bool hot = HOT && rel < hot_n;
          const bool binned = v && !hot && ((zmask >> min(key >> a.zone_shift, (uint64_t)(ZONES - 1))) & 1ull);
          const uint32_t bm = __ballot_sync(0xffffffffu, binned);
          if (binned) seg[bfill + __popc(bm & lt)] = (uint32_t)key | ((uint32_t)(e >> 15) << 31);
          bfill += __popc(bm);
          if (act && !binned) {
            if (hot) {
              atomicAdd(&stab[((e >> 15) ? hot_n : 0u) + hot_swz((uint32_t)rel)], 1u);
            } else if (a.dense32) {
              uint32_t* const q = static_cast<uint32_t*>(a.dense) + key;
              atomicAdd(q, 1u);
              atomicOr(q, E32_READ << (e >> 15));
            } else {
              atomicAdd(static_cast<unsigned long long*>(a.dense) + key, 1ull << (32 * (e >> 15)));
            }
          }
        }
      };
      if (BINS && zmask) {
        if (hot_n) fold_bins(std::true_type{});
        else fold_bins(std::false_type{});
      } else if (MARKS) {
        if (hot_n) fold(std::true_type{}, std::true_type{});
        else fold(std::false_type{}, std::true_type{});
      } else {
        if (hot_n) fold(std::true_type{}, std::false_type{});
        else fold(std::false_type{}, std::false_type{});
      }
      if (inval) flags |= F_ADDR_HINT;
    }
    for (uint32_t m = DENSE ? 0u : (rd16 | wr16); m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint64_t p = PAY(j);
      const bool isw = (wr16 >> j) & 1u;
      if (isw) a.wr_out[o_wr++] = p;
      else a.rd_out[o_rd++] = p;
      amin = min(amin, (unsigned long long)p); amax = max(amax, (unsigned long long)p);
      aand &= p; aor |= p;
    }
    // branches: ordered records site << 32 | group << 1 | taken; the group is the last
    // wg_begin before the branch in my row, else my carry-in group
    if (STAGE) {
      for (uint32_t m = br16; m; m &= m - 1) {
        const uint32_t j = __ffs(m) - 1;
        const uint64_t p = PAY(j);
        const uint32_t before = wgb16 & ((1u << j) - 1u);
        const uint32_t g = before ? (uint32_t)PAY(31 - __clz(before)) : gkey;
        const uint64_t site = p >> 1;
        flags |= ((site >> 32) ? (unsigned long long)F_BAD_SITE : 0ull) | ((g >> 31) ? (unsigned long long)F_BAD_GROUP : 0ull);
        max_site = max(max_site, (unsigned long long)site);
        a.br_out[o_br + __popc(br16 & ((1u << j) - 1u))] = (site << 32) | ((uint64_t)g << 1) | (p & 1);
      }
    } else if (br16) {
      flags |= F_BAD_KIND;  // the launcher stages whenever branches exist
    }
    // rare events in stream order: segment opens / closes, groups
    const uint64_t klo = (uint64_t)w[0] | ((uint64_t)w[1] << 32), khi = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    int last_b = -1;  // my last boundary position so far
    for (uint32_t m = (AIWC_ABL & 8) ? 0u : rare16; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint32_t kk = (uint32_t)((j < 8 ? klo >> (8 * j) : khi >> (8 * (j - 8))) & 0xFFu);
      const uint64_t p = PAY(j);
      if (CHECK && !(AIWC_ABL & 64)) {  // the payload rules (the sequence rules were checked on the masks above)
        bool bad = false;
        // (an opener's local id range and a wi_begin's duplicate-begin bit are handled at
        // the segment's close, do_close: the masks flag a segment never closed in its group)
        if (kk == AIWC_K_WI_END) {
          bad = p != lid;
        } else if (kk == AIWC_K_WG_BEGIN) {
          bad = (p >> 31) != 0;
        } else if (kk == AIWC_K_WG_END) {
          bad = p != (uint64_t)gkey;
        }
        if (bad) flags |= F_STREAM;
      }
      if (kk & 0x10) {
        if (kk & 0x20) {  // wi_begin / wi_resume opens a segment
          lid = (uint32_t)p; byres = kk >> 7;
        } else {          // barrier / wi_end closes it: instructions since the open
          const uint32_t cl = __popc(ins16 & ((1u << j) - 1u) & (0xFFFFFFFFu << (last_b + 1))) +
                              (last_b < 0 ? seg_in : 0u);
          const uint32_t gz = (gseq & 0x3FFFFFFFu) | ((kk & 0x80u) << 24) | (byres << 30);
          if (gseq >> 30) flags |= F_BAD_GROUP;
          if (o_cl < (uint32_t)WCL_CAP) wclose[o_cl] = make_uint4(cl, lid, gz, 16u * lane + j);
          else do_close(L, a, cl, lid, gz, e0 + j, itb_sum, ipt_sum, flags);
          ++o_cl;
        }
        last_b = (int)j;
      } else if (kk == AIWC_K_WG_BEGIN) {
        ++gseq; gkey = (uint32_t)p;
      } else if (kk != AIWC_K_WG_END && kk != AIWC_K_KERNEL_BEGIN && kk != AIWC_K_KERNEL_END) {
        flags |= F_BAD_KIND;
      }
    }
#undef PAY
    // ---- the next tile's carry-in: lane 31's end state ----
    const uint32_t nseg = __popc(ins16 >> (last_b + 1)) + (last_b < 0 ? seg_in : 0u);
    cseg = __shfl_sync(0xffffffffu, nseg, 31);
    clid = __shfl_sync(0xffffffffu, lid, 31);
    cbyres = __shfl_sync(0xffffffffu, byres, 31);
    cgseq = __shfl_sync(0xffffffffu, gseq, 31);
    cgkey = __shfl_sync(0xffffffffu, gkey, 31);
    c_rd += T_rd; c_wr += T_wr; c_br += T_br;
    __syncwarp();
    // ---- segment closes of the tile, the warp's lanes converged ----
    for (uint32_t i = lane; i < min(T_cl, (uint32_t)WCL_CAP); i += 32) {
      const uint4 c = wclose[i];
      do_close(L, a, c.x, c.y, c.z, tile0 + c.w, itb_sum, ipt_sum, flags);
    }
    __syncwarp();
    // ---- refill this stage (every lane is done with it) ----
    if (lane == 0 && it + STAGES < my_tiles) {
      const uint64_t r2 = (wt + STAGES) * WROWS;
      if (r2 < a.tma_rows) {
        mbar_expect_tx(&bars[s], WT * 9);
        tma_load_2d(S.kind[warp][s], &kmap, 0, (int)r2, &bars[s]);
        tma_load_2d(S.pay[warp][s], &pmap, 0, (int)r2, &bars[s]);
      }
    }
    if ((it + 1) % PRES_TILES == 0) record_presence(it / PRES_TILES);
    if ((it + 1) % ACC_FLUSH_TILES == 0) {
      flush_counts(oacc, wacc, a, lane, flags);
#pragma unroll
      for (int i = 0; i < 8; ++i) wsnap[i] = 0;
    }
  }

  // ---- epilogue: flush CTA-private state ----
  if (BINS && zmask && lane == 0) {
    a.bin_fill[gw] = bfill;
    if (bfill) atomicAdd(&st->bin_total, (unsigned long long)bfill);
  }
  if (my_tiles % PRES_TILES) record_presence((my_tiles - 1) / PRES_TILES);
  flush_counts(oacc, wacc, a, lane, flags);
  __syncthreads();
  if (DENSE && hot_n) {
    for (uint32_t i = t; i < hot_n; i += TPB) {
      const uint32_t r = stab[hot_swz(i)], w = stab[hot_n + hot_swz(i)];
      if (!(r | w) || hot_lo + i >= a.am.n_keys) continue;  // (the sentinel key is not a table key)
      if (a.dense32) {
        uint32_t* const q = static_cast<uint32_t*>(a.dense) + hot_lo + i;
        atomicAdd(q, r + w);
        atomicOr(q, (r ? E32_READ : 0u) | (w ? E32_WRITE : 0u));
      } else {
        atomicAdd(static_cast<unsigned long long*>(a.dense) + hot_lo + i,
                  (unsigned long long)r | ((unsigned long long)w << 32));
      }
    }
  }
  for (int i = t; i < HBINS; i += TPB) {
    if (L.itb_h[i]) atomicAdd(&st->itb_hist[i], (unsigned long long)L.itb_h[i]);
    if (L.ipt_h[i]) atomicAdd(&st->ipt_hist[i], (unsigned long long)L.ipt_h[i]);
  }
  itb_sum = warp_sum(itb_sum);
  ipt_sum = warp_sum(ipt_sum);
  n_wib = warp_sum(n_wib);
  n_bar = warp_sum(n_bar);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    max_site = max(max_site, __shfl_xor_sync(0xffffffffu, max_site, o));
    if (!DENSE) {
      amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
      amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      aand &= __shfl_xor_sync(0xffffffffu, aand, o);
      aor |= __shfl_xor_sync(0xffffffffu, aor, o);
    }
  }
  if (lane == 0) {
    if (itb_sum) atomicAdd(&st->itb_sum, itb_sum);
    if (n_wib) atomicAdd(&st->n_wib, (unsigned long long)n_wib);
    if (n_bar) atomicAdd(&st->n_bar, (unsigned long long)n_bar);
    if (ipt_sum) atomicAdd(&st->ipt_sum, ipt_sum);
    if (flags) atomicOr(&st->flags, flags);
    if (max_site) atomicMax(&st->max_site, max_site);
    if (!DENSE && amin <= amax) {
      atomicMin(&st->addr_min, amin); atomicMax(&st->addr_max, amax);
      atomicAnd(&st->addr_and, aand); atomicOr(&st->addr_or, aor);
    }
  }
}

// ---------------------------------------------------------------------------
// hot-key window choice: one CTA samples HS_SAMPLES events at hashed positions,
// counts the 1024-key blocks of the sampled memory accesses in a shared hash
// table and elects the most frequent block when it carries >= 1/64 of them.
// Keys of that block are then counted in shared memory by every ingest CTA
// (contended same-address REDs become one add per key per CTA).
// ---------------------------------------------------------------------------
constexpr int HS_T = 1024, HS_SAMPLES = 4096, HS_SLOTS = 4096;

__global__ void __launch_bounds__(HS_T) hot_sample_kernel(const uint8_t* __restrict__ kind,
                                                          const uint64_t* __restrict__ payload, uint64_t n,
                                                          AddrMap am, unsigned long long* hot_out) {
  __shared__ uint32_t hk[HS_SLOTS], hc[HS_SLOTS];
  __shared__ unsigned long long red[HS_T / 32];
  __shared__ uint32_t rmem[HS_T / 32];
  const int t = threadIdx.x;
  for (int i = t; i < HS_SLOTS; i += HS_T) { hk[i] = ~0u; hc[i] = 0; }
  __syncthreads();
  uint32_t nmem = 0;
  constexpr int PER = HS_SAMPLES / HS_T;
  uint64_t pos[PER], pv[PER];
  uint8_t kk[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    uint64_t x = (uint64_t)(t * PER + j) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    x = (x ^ (x >> 31)) * 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    pos[j] = x % n;
  }
  // all loads in flight at once (kind and payload independently): two memory round trips
#pragma unroll
  for (int j = 0; j < PER; ++j) { kk[j] = kind[pos[j]]; pv[j] = payload[pos[j]]; }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!is_mem(kk[j])) continue;
    const uint64_t off = pv[j] - am.base;
    if (off > am.off_max || (off & am.low_mask) != am.low_const) continue;
    const uint32_t blk = (uint32_t)((off >> am.k) >> 10);
    ++nmem;
    uint32_t h = (blk * 2654435761u) >> 20;  // 12-bit slot
    for (int probe = 0; probe < 64; ++probe, h = (h + 1) & (HS_SLOTS - 1)) {
      const uint32_t old = atomicCAS(&hk[h], ~0u, blk);
      if (old == ~0u || old == blk) { atomicAdd(&hc[h], 1u); break; }
    }
  }
  __syncthreads();
  unsigned long long best = 0;  // count << 32 | block
  for (int i = t; i < HS_SLOTS; i += HS_T)
    if (hc[i]) best = max(best, ((unsigned long long)hc[i] << 32) | hk[i]);
  nmem = warp_sum(nmem);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((t & 31) == 0) { red[t >> 5] = best; rmem[t >> 5] = nmem; }
  __syncthreads();
  if (t == 0) {
    unsigned long long b = 0;
    uint32_t m = 0;
    for (int w = 0; w < HS_T / 32; ++w) { b = max(b, red[w]); m += rmem[w]; }
    const uint32_t cnt = (uint32_t)(b >> 32);
    *hot_out = (cnt >= 16 && 64ull * cnt >= m) ? (unsigned long long)(uint32_t)b << 10 : ~0ull;
  }
}

void launch_hot_sample(const uint8_t* kind, const uint64_t* payload, uint64_t n, const AddrMap& am,
                       unsigned long long* hot_out, cudaStream_t s) {
  hot_sample_kernel<<<1, HS_T, 0, s>>>(kind, payload, n, am, hot_out);
}

template <bool DENSE, bool STAGE, int FEAT>
static cudaError_t launch_variant(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap,
                                  uint32_t n_ctas, cudaStream_t s) {
  const size_t smem = sizeof(StageSmem) + 1024 + 8ull * a.smem_keys;
  cudaError_t e = set_smem_once(ingest_kernel<DENSE, STAGE, FEAT>, (int)smem);
  if (e != cudaSuccess) return e;
  ingest_kernel<DENSE, STAGE, FEAT><<<n_ctas, TPB, smem, s>>>(a, kmap, pmap);
  return cudaGetLastError();
}

template <bool DENSE, bool STAGE>
static cudaError_t launch_feat(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap, uint32_t n_ctas,
                               cudaStream_t s) {
  const int feat = (a.check ? FEAT_CHECK : 0) | (DENSE && a.bin_zones ? FEAT_BINS : 0) |
                   (DENSE && a.chunk_bits ? FEAT_MARK : 0);
  switch (feat) {
    case 0: return launch_variant<DENSE, STAGE, 0>(a, kmap, pmap, n_ctas, s);
    case FEAT_CHECK: return launch_variant<DENSE, STAGE, FEAT_CHECK>(a, kmap, pmap, n_ctas, s);
    case FEAT_BINS: return launch_variant<DENSE, STAGE, FEAT_BINS>(a, kmap, pmap, n_ctas, s);
    case FEAT_BINS | FEAT_CHECK: return launch_variant<DENSE, STAGE, FEAT_BINS | FEAT_CHECK>(a, kmap, pmap, n_ctas, s);
    case FEAT_MARK: return launch_variant<DENSE, STAGE, FEAT_MARK>(a, kmap, pmap, n_ctas, s);
    case FEAT_MARK | FEAT_CHECK: return launch_variant<DENSE, STAGE, FEAT_MARK | FEAT_CHECK>(a, kmap, pmap, n_ctas, s);
    default: return cudaErrorInvalidValue;  // bins and marks never combine (a shard does not bin)
  }
}

cudaError_t launch_ingest(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap, uint32_t n_ctas,
                          bool dense, bool stage, cudaStream_t s) {
  if (dense) return stage ? launch_feat<true, true>(a, kmap, pmap, n_ctas, s)
                          : launch_feat<true, false>(a, kmap, pmap, n_ctas, s);
  return a.check ? launch_variant<false, true, FEAT_CHECK>(a, kmap, pmap, n_ctas, s)
                 : launch_variant<false, true, 0>(a, kmap, pmap, n_ctas, s);
}

}  // namespace aiwc
