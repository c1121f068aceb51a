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
//          consecutive events.  A block scan over per-thread kind summaries
//          gives every thread its exact carry-in (segment count, work-item,
//          group, output offsets); then each thread folds its 16 events:
//          opcode/width histograms (lane-private u16 smem bins), memory
//          addresses (dense-table RED.ADD or ordered compaction), and -- on
//          the rare path -- ITB/IPT values (smem histograms + exact overflow
//          lists), per-work-item IPT slots and ordered branch records.
#include "aiwc_internal.cuh"

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

__device__ __forceinline__ uint32_t m_wgb(uint32_t w) { return w & ~(w >> 1) & 0x40404040u; }

// bit 0 of each byte of four words -> 16-bit mask in event order (byte b of
// word i -> bit 4i + b).  The multiply by 0x01020408 moves byte b's bit 0 to
// bit 24 + b without carries.
__device__ __forceinline__ uint32_t nib4(uint32_t x) { return ((x & 0x01010101u) * 0x01020408u) >> 24; }
__device__ __forceinline__ uint32_t gather16(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return nib4(a) | (nib4(b) << 4) | (nib4(c) << 8) | (nib4(d) << 12);
}

// per-class counts of 16 kind bytes.  Nibble packing: L holds bits 0..3
// (instr, read, write, branch) of two words, H bits 4..7 (boundary, open,
// group, variant); each class is then one masked popcount per packed word.
struct KindCounts {
  uint32_t instr = 0, rd = 0, wr = 0, br = 0, bnd = 0, wgb = 0, bres = 0, wib = 0, bar = 0;
  __device__ __forceinline__ void add(const uint32_t w[4]) {
    const uint32_t L0 = (w[0] & 0x0F0F0F0Fu) | ((w[1] & 0x0F0F0F0Fu) << 4);
    const uint32_t L1 = (w[2] & 0x0F0F0F0Fu) | ((w[3] & 0x0F0F0F0Fu) << 4);
    const uint32_t H0 = ((w[0] >> 4) & 0x0F0F0F0Fu) | (w[1] & 0xF0F0F0F0u);
    const uint32_t H1 = ((w[2] >> 4) & 0x0F0F0F0Fu) | (w[3] & 0xF0F0F0F0u);
    instr += __popc(L0 & 0x11111111u) + __popc(L1 & 0x11111111u);
    rd += __popc(L0 & 0x22222222u) + __popc(L1 & 0x22222222u);
    wr += __popc(L0 & 0x44444444u) + __popc(L1 & 0x44444444u);
    br += __popc(L0 & 0x88888888u) + __popc(L1 & 0x88888888u);
    bnd += __popc(H0 & 0x11111111u) + __popc(H1 & 0x11111111u);
    wgb += __popc(H0 & ~(H0 >> 1) & 0x44444444u) + __popc(H1 & ~(H1 >> 1) & 0x44444444u);
    bres += __popc(H0 & (H0 >> 3) & 0x11111111u) + __popc(H1 & (H1 >> 3) & 0x11111111u);
    wib += __popc(H0 & (H0 >> 1) & ~(H0 >> 3) & 0x11111111u) + __popc(H1 & (H1 >> 1) & ~(H1 >> 3) & 0x11111111u);
    bar += __popc(H0 & ~(H0 >> 1) & (H0 >> 3) & 0x11111111u) + __popc(H1 & ~(H1 >> 1) & (H1 >> 3) & 0x11111111u);
  }
};

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
  long long last_bnd = -1, last_wgb = -1;
  unsigned long long amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  constexpr int U = 4;  // 16-byte loads in flight per thread
  for (uint64_t base = rb + 16ull * U * t; base < re; base += 16ull * U * P1_THREADS) {
    uint32_t w[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) load_kind16(kind, base + 16 * u, re, w[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      kc.add(w[u]);
      const uint64_t e0 = base + 16 * u;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t bm = w[u][i] & 0x10101010u, gm = m_wgb(w[u][i]);
        if (bm) last_bnd = (long long)(e0 + 4 * i + ((31 - __clz(bm)) >> 3));
        if (gm) last_wgb = (long long)(e0 + 4 * i + ((31 - __clz(gm)) >> 3));
        if (with_stats) {
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
  // block reduction
  constexpr int NW = P1_THREADS / 32;
  __shared__ uint32_t s_cnt[NW][9];
  __shared__ long long s_pos[NW][2];
  __shared__ unsigned long long s_addr[NW][4];
  __shared__ long long s_lb;
  uint32_t v[9] = {kc.instr, kc.rd, kc.wr, kc.br, kc.bnd, kc.wgb, kc.bres, kc.wib, kc.bar};
  const int lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int i = 0; i < 9; ++i) v[i] = warp_sum(v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    last_bnd = max(last_bnd, __shfl_xor_sync(0xffffffffu, last_bnd, o));
    last_wgb = max(last_wgb, __shfl_xor_sync(0xffffffffu, last_wgb, o));
    if (with_stats) {
      amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
      amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      aand &= __shfl_xor_sync(0xffffffffu, aand, o);
      aor |= __shfl_xor_sync(0xffffffffu, aor, o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 9; ++i) s_cnt[warp][i] = v[i];
    s_pos[warp][0] = last_bnd; s_pos[warp][1] = last_wgb;
    s_addr[warp][0] = amin; s_addr[warp][1] = amax; s_addr[warp][2] = aand; s_addr[warp][3] = aor;
  }
  __syncthreads();
  if (t == 0) {
    RangeSum r{};
    uint32_t tot[9] = {0};
    long long lb = -1, lw = -1;
    unsigned long long mn = ~0ull, mx = 0, an = ~0ull, o = 0;
    for (int w = 0; w < NW; ++w) {
      for (int i = 0; i < 9; ++i) tot[i] += s_cnt[w][i];
      lb = max(lb, s_pos[w][0]); lw = max(lw, s_pos[w][1]);
      mn = min(mn, s_addr[w][0]); mx = max(mx, s_addr[w][1]); an &= s_addr[w][2]; o |= s_addr[w][3];
    }
    r.n_instr = tot[0]; r.n_rd = tot[1]; r.n_wr = tot[2]; r.n_br = tot[3]; r.n_bnd = tot[4];
    r.n_wgb = tot[5]; r.n_bres = tot[6]; r.n_wib = tot[7]; r.n_bar = tot[8];
    r.last_bnd = lb; r.last_wgb = lw;
    out[blockIdx.x] = r;
    s_lb = lb;
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
                  bool with_stats, RangeSum* out, DevState* st, cudaStream_t s) {
  pass1_kernel<<<n_ranges * P1_SUB, P1_THREADS, 0, s>>>(kind, payload, n, tiles_per_cta, with_stats, out, st);
}

// ---------------------------------------------------------------------------
// main ingest pass
// ---------------------------------------------------------------------------
constexpr int BND_CAP = 512;  // close records buffered per tile (overflow is processed inline)

struct IngestSmem {
  uint64_t pay[STAGES][TILE];        // 128 B-swizzled payload rows (TMA); 1024 B aligned
  uint8_t kind[STAGES][TILE];
  uint16_t opc_priv[OBINS][TPB];     // lane-private opcode counts (flushed before they can wrap)
  uint16_t wid_priv[WBINS][TPB];     // lane-private width counts (width 1..16)
  uint32_t itb_h[HBINS];
  uint32_t ipt_h[HBINS];
  unsigned long long wfirst[WBINS];
  uint4 closes[BND_CAP];             // segment closes of the tile: (seg, lid, gseq | bar << 31 | byres << 30)
  uint32_t ws[TPB / 32][6];
  uint32_t vpos[TPB];
  uint32_t nc[5];
  uint64_t bar[STAGES];
  uint64_t stage_out[1];             // TILE entries when the kernel stages compaction output
};
constexpr uint32_t PRIV_FLUSH_TILES = 65535 / EPT;  // u16 bins take at most EPT increments per tile

__device__ __forceinline__ uint64_t pay_at(const uint64_t* pay, uint32_t pos) {
  const uint32_t row = pos >> 4, j = pos & 15;
  return pay[row * 16 + ((((j >> 1) ^ (row & 7))) << 1) + (j & 1)];
}

// One segment close (metrics.py:156-174): ITB sample (barrier always, wi_end when
// non-empty); IPT either straight to the histogram (work-item never crossed a
// barrier) or accumulated in the work-item's lifetime slot.
__device__ __forceinline__ void do_close(IngestSmem& S, const IngestArgs& a, uint32_t seg, uint32_t lid, uint32_t gz,
                                         unsigned long long& itb_sum, unsigned long long& ipt_sum,
                                         unsigned long long& flags) {
  const bool bar = gz >> 31, byres = (gz >> 30) & 1u;
  const uint32_t gseq = gz & 0x3FFFFFFFu;
  if (bar || seg) {
    if (seg < (uint32_t)HBINS) atomicAdd(&S.itb_h[seg], 1u);
    else a.itb_ovf[atomicAdd(&a.st->itb_ovf_n, 1ull)] = seg;
    itb_sum += seg;
  }
  if (bar || byres) {
    const uint64_t slot = (uint64_t)(gseq - 1) * a.local_volume + lid;
    if (gseq == 0 || slot >= a.ipt_tab_len) flags |= F_SLOT_RANGE;
    else atomicAdd(&a.ipt_tab[slot], (unsigned long long)seg + (bar ? 0ull : IPT_END_FLAG));
  } else {
    if (seg < (uint32_t)HBINS) atomicAdd(&S.ipt_h[seg], 1u);
    else a.ipt_ovf[atomicAdd(&a.st->ipt_ovf_n, 1ull)] = seg;
    ipt_sum += seg;
  }
}

__device__ __forceinline__ void flush_private(IngestSmem& S, const IngestArgs& a, int t) {
  __syncthreads();
  if (t < OBINS) {
    unsigned long long sum = 0;
    for (int i = 0; i < TPB; ++i) { sum += S.opc_priv[t][i]; S.opc_priv[t][i] = 0; }
    if (sum) atomicAdd(&a.opc_counts[t], sum);
  } else if (t >= 32 && t < 32 + WBINS) {
    const int b = t - 32;
    unsigned long long sum = 0;
    for (int i = 0; i < TPB; ++i) { sum += S.wid_priv[b][i]; S.wid_priv[b][i] = 0; }
    if (sum) atomicAdd(&a.width_count[b + 1], sum);
  }
  __syncthreads();
}

template <bool DENSE, bool STAGE>
__global__ void __launch_bounds__(TPB, STAGE ? 1 : 2)
    ingest_kernel(const IngestArgs a, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap pmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  IngestSmem& S = *reinterpret_cast<IngestSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t n = a.n;
  const uint64_t n_tiles_total = (n + TILE - 1) / TILE;
  const uint64_t tile_begin = (uint64_t)blockIdx.x * a.tiles_per_cta;
  if (tile_begin >= n_tiles_total) return;
  const uint32_t my_tiles = (uint32_t)min((uint64_t)a.tiles_per_cta, n_tiles_total - tile_begin);
  DevState* st = a.st;

  // ---- prologue: smem init + TMA ring fill ----
  for (int i = t; i < OBINS * TPB; i += TPB) (&S.opc_priv[0][0])[i] = 0;
  for (int i = t; i < WBINS * TPB; i += TPB) (&S.wid_priv[0][0])[i] = 0;
  for (int i = t; i < HBINS; i += TPB) { S.itb_h[i] = 0; S.ipt_h[i] = 0; }
  if (t < WBINS) S.wfirst[t] = ~0ull;
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&S.bar[s], 1);
    fence_barrier_init();
    for (uint32_t it = 0; it < (uint32_t)STAGES && it < my_tiles; ++it) {
      const uint64_t row0 = (tile_begin + it) * (TILE / 16);
      if (row0 < a.tma_rows) {
        mbar_expect_tx(&S.bar[it], TILE * 9);
        tma_load_2d(S.kind[it], &kmap, 0, (int)row0, &S.bar[it]);
        tma_load_2d(S.pay[it], &pmap, 0, (int)row0, &S.bar[it]);
      }
    }
  }

  // ---- carry-in at the start of this CTA's range: combine the sub-ranges before it ----
  uint32_t cseg, clid = 0, cbyres = 0, cgseq = 0, cgkey = 0;
  unsigned long long c_rd = 0, c_wr = 0, c_br = 0;
  {
    const uint32_t c = blockIdx.x * P1_SUB;
    long long jb = -1, lw = -1;
    uint64_t s_rd = 0, s_wr = 0, s_br = 0, s_wgb = 0;
    for (uint32_t j = t; j < c; j += TPB) {
      const RangeSum& r = a.ranges[j];
      if (r.last_bnd >= 0) jb = max(jb, (long long)j);
      lw = max(lw, (long long)r.last_wgb);
      s_rd += r.n_rd; s_wr += r.n_wr; s_br += r.n_br; s_wgb += r.n_wgb;
    }
    __shared__ unsigned long long red[TPB / 32][6];
    s_rd = warp_sum(s_rd); s_wr = warp_sum(s_wr); s_br = warp_sum(s_br); s_wgb = warp_sum(s_wgb);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      jb = max(jb, __shfl_xor_sync(0xffffffffu, jb, o));
      lw = max(lw, __shfl_xor_sync(0xffffffffu, lw, o));
    }
    if (lane == 0) {
      red[warp][0] = s_rd; red[warp][1] = s_wr; red[warp][2] = s_br; red[warp][3] = s_wgb;
      red[warp][4] = (unsigned long long)jb; red[warp][5] = (unsigned long long)lw;
    }
    __syncthreads();
    jb = -1; lw = -1; s_rd = s_wr = s_br = s_wgb = 0;
    for (int w = 0; w < TPB / 32; ++w) {
      s_rd += red[w][0]; s_wr += red[w][1]; s_br += red[w][2]; s_wgb += red[w][3];
      jb = max(jb, (long long)red[w][4]); lw = max(lw, (long long)red[w][5]);
    }
    uint64_t s_in = 0;  // instructions after the last boundary: after(jb) + instrs of later sub-ranges
    for (uint32_t j = (uint32_t)(jb + 1) + t; j < c; j += TPB) s_in += a.ranges[j].n_instr;
    s_in = warp_sum(s_in);
    __syncthreads();
    if (lane == 0) red[warp][0] = s_in;
    __syncthreads();
    uint64_t after = 0;
    for (int w = 0; w < TPB / 32; ++w) after += red[w][0];
    if (jb >= 0) {
      const long long lbpos = a.ranges[jb].last_bnd;
      after += a.ranges[jb].instr_after;
      clid = (uint32_t)a.payload[lbpos];
      cbyres = a.kind[lbpos] == AIWC_K_WI_RESUME;
    }
    cseg = (uint32_t)after;
    c_rd = s_rd; c_wr = s_wr; c_br = s_br;
    cgseq = (uint32_t)s_wgb;
    cgkey = lw >= 0 ? (uint32_t)a.payload[lw] : 0u;
  }
  __syncthreads();

  uint32_t seen_w = 0;  // widths 1..16 already first-indexed by this thread
  unsigned long long itb_sum = 0, ipt_sum = 0, flags = 0, max_site = 0;
  unsigned long long amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  uint16_t* const opc_col = &S.opc_priv[0][t];
  uint16_t* const wid_col = &S.wid_priv[0][t];

  for (uint32_t it = 0; it < my_tiles; ++it) {
    const int s = it % STAGES;
    const uint64_t tile0 = (tile_begin + it) * TILE;
    const uint64_t row0 = tile0 / 16;
    if (row0 < a.tma_rows) mbar_wait(&S.bar[s], (it / STAGES) & 1);
    const uint64_t e0 = tile0 + 16ull * t;
    uint32_t w[4];
    if (row0 + t < a.tma_rows) {
      const uint4 v = *reinterpret_cast<const uint4*>(&S.kind[s][16 * t]);
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      // rows beyond the tensor maps (tail of the trace): direct loads, patch smem
      load_kind16(a.kind, e0, n, w);
      *reinterpret_cast<uint4*>(&S.kind[s][16 * t]) = make_uint4(w[0], w[1], w[2], w[3]);
      for (int j = 0; j < 16; ++j) {
        const uint64_t e = e0 + j;
        S.pay[s][t * 16 + ((((j >> 1) ^ (t & 7))) << 1) + (j & 1)] = e < n ? a.payload[e] : 0ull;
      }
    }
    // ---- per-thread class masks: bit j = event j of my 16 is in the class ----
    const uint32_t ins16 = gather16(w[0], w[1], w[2], w[3]);
    const uint32_t rd16 = gather16(w[0] >> 1, w[1] >> 1, w[2] >> 1, w[3] >> 1);
    const uint32_t wr16 = gather16(w[0] >> 2, w[1] >> 2, w[2] >> 2, w[3] >> 2);
    const uint32_t br16 = gather16(w[0] >> 3, w[1] >> 3, w[2] >> 3, w[3] >> 3);
    const uint32_t bnd16 = gather16(w[0] >> 4, w[1] >> 4, w[2] >> 4, w[3] >> 4);
    const uint32_t open16 = bnd16 & gather16(w[0] >> 5, w[1] >> 5, w[2] >> 5, w[3] >> 5);
    const uint32_t wgb16 = gather16(m_wgb(w[0]) >> 6, m_wgb(w[1]) >> 6, m_wgb(w[2]) >> 6, m_wgb(w[3]) >> 6);
    // rare: branch, boundary, group and kernel events (bits 3..6)
    const uint32_t rare16 = gather16((w[0] >> 3) | (w[0] >> 4) | (w[0] >> 5) | (w[0] >> 6),
                                     (w[1] >> 3) | (w[1] >> 4) | (w[1] >> 5) | (w[1] >> 6),
                                     (w[2] >> 3) | (w[2] >> 4) | (w[2] >> 5) | (w[2] >> 6),
                                     (w[3] >> 3) | (w[3] >> 4) | (w[3] >> 5) | (w[3] >> 6));
    const uint32_t n_in = __popc(ins16), n_rd = __popc(rd16), n_wr = __popc(wr16), n_br = __popc(br16);
    const uint32_t n_wg = __popc(wgb16), n_cl = __popc(bnd16 & ~open16);
    const int lp = bnd16 ? 31 - __clz(bnd16) : -1;
    const int lw = wgb16 ? 31 - __clz(wgb16) : -1;
    const uint32_t after = __popc(ins16 >> (lp + 1));
    // ---- block scan ----
    const uint32_t A = n_in | (n_br << 16), B = n_rd | (n_wr << 16), C = n_wg | (n_cl << 16);
    const uint32_t P = lp >= 0 ? (uint32_t)(16 * t + lp + 1) : 0u;
    const uint32_t Q = lw >= 0 ? (uint32_t)(16 * t + lw + 1) : 0u;
    const uint32_t Ai = warp_incl_sum(A), Bi = warp_incl_sum(B), Ci = warp_incl_sum(C);
    const uint32_t Pi = warp_incl_max(P), Qi = warp_incl_max(Q);
    if (lane == 31) { S.ws[warp][0] = Ai; S.ws[warp][1] = Bi; S.ws[warp][2] = Ci; S.ws[warp][3] = Pi; S.ws[warp][4] = Qi; }
    __syncthreads();
    uint32_t Ap = 0, Bp = 0, Cp = 0, Pp = 0, Qp = 0, TA = 0, TB = 0, TC = 0;
#pragma unroll
    for (int q = 0; q < TPB / 32; ++q) {
      const uint32_t a0 = S.ws[q][0], b0 = S.ws[q][1], c0 = S.ws[q][2];
      if (q < warp) { Ap += a0; Bp += b0; Cp += c0; Pp = max(Pp, S.ws[q][3]); Qp = max(Qp, S.ws[q][4]); }
      TA += a0; TB += b0; TC += c0;
    }
    uint32_t Pe = __shfl_up_sync(0xffffffffu, Pi, 1), Qe = __shfl_up_sync(0xffffffffu, Qi, 1);
    if (lane == 0) { Pe = 0; Qe = 0; }
    const uint32_t Aex = Ap + Ai - A, Bex = Bp + Bi - B, Cex = Cp + Ci - C;
    const uint32_t Pex = max(Pp, Pe), Qex = max(Qp, Qe);
    const uint32_t ex_in = Aex & 0xFFFFu, ex_br = Aex >> 16, ex_rd = Bex & 0xFFFFu, ex_wr = Bex >> 16;
    const uint32_t T_rd = TB & 0xFFFFu, T_wr = TB >> 16, T_br = TA >> 16;
    S.vpos[t] = ex_in + n_in - after;  // instructions in the tile at positions <= my last boundary
    __syncthreads();
    // ---- carry-in for this thread ----
    uint32_t seg, lid, byres;
    if (Pex) {
      const uint32_t pos = Pex - 1;
      seg = ex_in - S.vpos[pos >> 4];
      lid = (uint32_t)pay_at(S.pay[s], pos);
      byres = S.kind[s][pos] == AIWC_K_WI_RESUME;
    } else {
      seg = cseg + ex_in; lid = clid; byres = cbyres;
    }
    uint32_t gkey = Qex ? (uint32_t)pay_at(S.pay[s], Qex - 1) : cgkey;
    uint32_t gseq = cgseq + (Cex & 0xFFFFu);
    uint32_t o_rd = ex_rd, o_wr = T_rd + ex_wr;
    uint32_t o_br = (DENSE ? 0u : T_rd + T_wr) + ex_br;
    uint32_t o_cl = Cex >> 16;
    const uint32_t T_cl = TC >> 16;
    // ---- fold my 16 events, one converged loop per event class ----
    const uint64_t* prow = &S.pay[s][t * 16];
    const uint32_t sw = t & 7;
#define PAY(j) prow[((((uint32_t)(j) >> 1) ^ sw) << 1) | ((uint32_t)(j) & 1u)]
    // instructions: opcode / width histograms
    for (uint32_t m = ins16; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint64_t p = PAY(j);
      const uint32_t opc = (uint32_t)(p >> 32), wd = (uint32_t)p;
      if (opc < OBINS) ++opc_col[opc * TPB];
      else if (opc < a.n_opcodes) atomicAdd(&a.opc_counts[opc], 1ull);
      else flags |= F_BAD_OPCODE;
      if (wd - 1u < (uint32_t)WBINS) {
        ++wid_col[(wd - 1) * TPB];
        if (!((seen_w >> (wd - 1)) & 1u)) {
          seen_w |= 1u << (wd - 1);
          atomicMin(&S.wfirst[wd - 1], (unsigned long long)(e0 + j));
        }
      } else if (wd < WIDTH_TABLE) {
        atomicAdd(&a.width_count[wd], 1ull);
        atomicMin(&a.width_first[wd], (unsigned long long)(e0 + j));
      } else {
        flags |= F_BAD_WIDTH;
      }
    }
    // memory accesses: dense-table counters or compaction
    for (uint32_t m = rd16 | wr16; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint64_t p = PAY(j);
      const bool isw = (wr16 >> j) & 1u;
      if (DENSE) {
        const uint64_t off = p - a.am.base;
        const uint64_t key = off >> a.am.k;
        if (p < a.am.base || (off & a.am.low_mask) != a.am.low_const || key >= a.am.n_keys) flags |= F_ADDR_HINT;
        else atomicAdd(&a.dense[key], isw ? (1ull << 32) : 1ull);
      } else {
        S.stage_out[isw ? o_wr++ : o_rd++] = p;
        amin = min(amin, (unsigned long long)p); amax = max(amax, (unsigned long long)p);
        aand &= p; aor |= p;
      }
    }
    // rare events in stream order: segment opens / closes, branches, groups
    const uint64_t klo = (uint64_t)w[0] | ((uint64_t)w[1] << 32), khi = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    const uint32_t seg_in = seg;
    int last_b = -1;  // my last boundary position so far
    for (uint32_t m = rare16; m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint32_t k = (uint32_t)((j < 8 ? klo >> (8 * j) : khi >> (8 * (j - 8))) & 0xFFu);
      const uint64_t p = PAY(j);
      if (k == AIWC_K_BRANCH) {
        const uint64_t site = p >> 1;
        if (site >> 32) flags |= F_BAD_SITE;
        if (gkey >> 31) flags |= F_BAD_GROUP;
        max_site = max(max_site, (unsigned long long)site);
        if (STAGE) S.stage_out[o_br++] = (site << 32) | ((uint64_t)gkey << 1) | (p & 1);
        else flags |= F_BAD_KIND;  // the launcher stages whenever branches exist
      } else if (k & 0x10) {
        if (k & 0x20) {  // wi_begin / wi_resume opens a segment
          lid = (uint32_t)p; byres = k >> 7;
        } else {         // barrier / wi_end closes it: instructions since the open
          const uint32_t cl = __popc(ins16 & ((1u << j) - 1u) & (0xFFFFFFFFu << (last_b + 1))) +
                              (last_b < 0 ? seg_in : 0u);
          const uint32_t gz = (gseq & 0x3FFFFFFFu) | ((k & 0x80u) << 24) | (byres << 30);
          if (gseq >> 30) flags |= F_BAD_GROUP;
          if (o_cl < (uint32_t)BND_CAP) S.closes[o_cl] = make_uint4(cl, lid, gz, 0u);
          else do_close(S, a, cl, lid, gz, itb_sum, ipt_sum, flags);
          ++o_cl;
        }
        last_b = (int)j;
      } else if (k == AIWC_K_WG_BEGIN) {
        ++gseq; gkey = (uint32_t)p;
      } else if (k != AIWC_K_WG_END && k != AIWC_K_KERNEL_BEGIN && k != AIWC_K_KERNEL_END) {
        flags |= F_BAD_KIND;
      }
    }
#undef PAY
    seg = __popc(ins16 >> (last_b + 1)) + (last_b < 0 ? seg_in : 0u);
    if (t == TPB - 1) { S.nc[0] = seg; S.nc[1] = lid; S.nc[2] = byres; S.nc[3] = gseq; S.nc[4] = gkey; }
    __syncthreads();
    // ---- segment closes of the tile, all threads converged ----
    for (uint32_t i = t; i < min(T_cl, (uint32_t)BND_CAP); i += TPB) {
      const uint4 c = S.closes[i];
      do_close(S, a, c.x, c.y, c.z, itb_sum, ipt_sum, flags);
    }
    // ---- flush ordered compaction ----
    if (STAGE) {
      if (!DENSE) {
        for (uint32_t i = t; i < T_rd; i += TPB) a.rd_out[c_rd + i] = S.stage_out[i];
        for (uint32_t i = t; i < T_wr; i += TPB) a.wr_out[c_wr + i] = S.stage_out[T_rd + i];
      }
      const uint32_t bb = DENSE ? 0u : T_rd + T_wr;
      for (uint32_t i = t; i < T_br; i += TPB) a.br_out[c_br + i] = S.stage_out[bb + i];
    }
    cseg = S.nc[0]; clid = S.nc[1]; cbyres = S.nc[2]; cgseq = S.nc[3]; cgkey = S.nc[4];
    c_rd += T_rd; c_wr += T_wr; c_br += T_br;
    // ---- refill this stage ----
    if (t == 0 && it + STAGES < my_tiles) {
      const uint64_t r2 = (tile_begin + it + STAGES) * (TILE / 16);
      if (r2 < a.tma_rows) {
        mbar_expect_tx(&S.bar[s], TILE * 9);
        tma_load_2d(S.kind[s], &kmap, 0, (int)r2, &S.bar[s]);
        tma_load_2d(S.pay[s], &pmap, 0, (int)r2, &S.bar[s]);
      }
    }
    if ((it + 1) % PRIV_FLUSH_TILES == 0) flush_private(S, a, t);
  }

  // ---- epilogue: flush CTA-private state ----
  flush_private(S, a, t);
  if (t >= 32 && t < 32 + WBINS && S.wfirst[t - 32] != ~0ull) atomicMin(&a.width_first[t - 32 + 1], S.wfirst[t - 32]);
  for (int i = t; i < HBINS; i += TPB) {
    if (S.itb_h[i]) atomicAdd(&st->itb_hist[i], (unsigned long long)S.itb_h[i]);
    if (S.ipt_h[i]) atomicAdd(&st->ipt_hist[i], (unsigned long long)S.ipt_h[i]);
  }
  itb_sum = warp_sum(itb_sum);
  ipt_sum = warp_sum(ipt_sum);
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
    if (ipt_sum) atomicAdd(&st->ipt_sum, ipt_sum);
    if (flags) atomicOr(&st->flags, flags);
    if (max_site) atomicMax(&st->max_site, max_site);
    if (!DENSE && amin <= amax) {
      atomicMin(&st->addr_min, amin); atomicMax(&st->addr_max, amax);
      atomicAnd(&st->addr_and, aand); atomicOr(&st->addr_or, aor);
    }
  }
}

template <bool DENSE, bool STAGE>
static cudaError_t launch_variant(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap,
                                  uint32_t n_ctas, cudaStream_t s) {
  const size_t smem = sizeof(IngestSmem) + (STAGE ? (TILE - 1) * sizeof(uint64_t) : 0) + 1024;
  cudaError_t e = cudaFuncSetAttribute(ingest_kernel<DENSE, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  ingest_kernel<DENSE, STAGE><<<n_ctas, TPB, smem, s>>>(a, kmap, pmap);
  return cudaGetLastError();
}

cudaError_t launch_ingest(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap, uint32_t n_ctas,
                          bool dense, bool stage, cudaStream_t s) {
  if (dense) return stage ? launch_variant<true, true>(a, kmap, pmap, n_ctas, s)
                          : launch_variant<true, false>(a, kmap, pmap, n_ctas, s);
  return launch_variant<false, true>(a, kmap, pmap, n_ctas, s);
}

}  // namespace aiwc
