// aiwc_ingest.cu -- the streaming pass over the columnar trace.
//
// Replaces the per-event dispatch loop of the reference's consume()
// (pkg/src/aiwc/metrics.py:125-180).  Two launches:
//
//  pass1   one CTA per contiguous event range; reads ONLY the kind bytes
//          (16 per thread per step, SWAR bit-tests) and writes a RangeSum:
//          per-class counts, the last work-item boundary / work-group begin
//          and the instructions after the last boundary.  That is all the
//          sequential state (open segment length, open work-item, group) the
//          next pass needs at its range start.
//  ingest  the same ranges, one persistent 256-thread CTA per SM.  Tiles of
//          4096 events arrive by TMA (kind rows + payload rows with 128 B
//          swizzle) through a 3-stage mbarrier ring; each thread owns 16
//          consecutive events.  A block scan over per-thread kind summaries
//          gives every thread its exact carry-in (segment count, work-item,
//          group, output offsets), then each thread folds its 16 events:
//          opcode/width histograms (lane-private smem bins), ITB/IPT values
//          (smem histograms + exact overflow lists), per-work-item IPT slots,
//          memory addresses (dense table RED.ADD or compaction) and branch
//          records (ordered compaction).
#include "aiwc_internal.cuh"

namespace aiwc {

// ---------------------------------------------------------------------------
// pass 1
// ---------------------------------------------------------------------------
constexpr int P1_THREADS = 512;

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

// SWAR class masks over 4 kind bytes
__device__ __forceinline__ uint32_t m_wgb(uint32_t w) { return w & ~(w >> 1) & 0x40404040u; }
// each test is evaluated at one bit position of the byte; shifts never reach
// across a byte boundary at that position
__device__ __forceinline__ uint32_t m_wib(uint32_t w) {  // 0x30: bit4 & bit5 & !bit7, at bit5
  return (w & (w << 1) & ~(w >> 2)) & 0x20202020u;
}
__device__ __forceinline__ uint32_t m_wir(uint32_t w) {  // 0xB0: bit4 & bit5 & bit7, at bit4
  return (w & (w >> 1) & (w >> 3)) & 0x10101010u;
}
__device__ __forceinline__ uint32_t m_wie(uint32_t w) {  // 0x10: bit4 & !bit5 & !bit7
  return (w & ~(w >> 1) & ~(w >> 3)) & 0x10101010u;
}
__device__ __forceinline__ uint32_t m_bar(uint32_t w) {  // 0x90: bit4 & !bit5 & bit7
  return (w & ~(w >> 1) & (w >> 3)) & 0x10101010u;
}

__global__ void __launch_bounds__(P1_THREADS) pass1_kernel(const uint8_t* __restrict__ kind,
                                                           const uint64_t* __restrict__ payload, uint64_t n,
                                                           uint32_t tiles_per_cta, bool with_stats,
                                                           RangeSum* __restrict__ out, DevState* st) {
  const uint64_t rb = (uint64_t)blockIdx.x * tiles_per_cta * TILE;
  const uint64_t re = min(n, rb + (uint64_t)tiles_per_cta * TILE);
  const int t = threadIdx.x;
  uint32_t c_instr = 0, c_rd = 0, c_wr = 0, c_br = 0, c_wgb = 0, c_wib = 0, c_wir = 0, c_wie = 0, c_bar = 0,
           c_ev = 0;
  long long last_bnd = -1, last_wgb = -1;
  unsigned long long amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  for (uint64_t e0 = rb + 16ull * t; e0 < re; e0 += 16ull * P1_THREADS) {
    uint32_t w[4];
    load_kind16(kind, e0, re, w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t x = w[i];
      c_instr += __popc(x & 0x01010101u);
      c_rd += __popc(x & 0x02020202u);
      c_wr += __popc(x & 0x04040404u);
      c_br += __popc(x & 0x08080808u);
      c_wgb += __popc(m_wgb(x));
      c_wib += __popc(m_wib(x));
      c_wir += __popc(m_wir(x));
      c_wie += __popc(m_wie(x));
      c_bar += __popc(m_bar(x));
      c_ev += __popc(((x | (x >> 1) | (x >> 2) | (x >> 3) | (x >> 4) | (x >> 5) | (x >> 6) | (x >> 7)) & 0x01010101u));
      const uint32_t bm = x & 0x10101010u;
      if (bm) last_bnd = (long long)(e0 + 4 * i + ((31 - __clz(bm)) >> 3));
      const uint32_t gm = m_wgb(x);
      if (gm) last_wgb = (long long)(e0 + 4 * i + ((31 - __clz(gm)) >> 3));
      if (with_stats) {
        uint32_t mm = x & 0x06060606u;
        while (mm) {
          const int b = (__ffs(mm) - 1) >> 3;
          mm &= ~(0xFFu << (8 * b));
          const unsigned long long ad = payload[e0 + 4 * i + b];
          amin = min(amin, ad); amax = max(amax, ad); aand &= ad; aor |= ad;
        }
      }
    }
  }
  // block reduction
  __shared__ uint32_t s_cnt[P1_THREADS / 32][10];
  __shared__ long long s_pos[P1_THREADS / 32][2];
  __shared__ unsigned long long s_addr[P1_THREADS / 32][4];
  __shared__ long long s_lb;
  uint32_t v[10] = {c_instr, c_rd, c_wr, c_br, c_wgb, c_wib, c_wir, c_wie, c_bar, c_ev};
  const int lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int i = 0; i < 10; ++i) v[i] = warp_sum(v[i]);
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
    for (int i = 0; i < 10; ++i) s_cnt[warp][i] = v[i];
    s_pos[warp][0] = last_bnd; s_pos[warp][1] = last_wgb;
    s_addr[warp][0] = amin; s_addr[warp][1] = amax; s_addr[warp][2] = aand; s_addr[warp][3] = aor;
  }
  __syncthreads();
  if (t == 0) {
    RangeSum r{};
    uint32_t tot[10] = {0};
    long long lb = -1, lw = -1;
    unsigned long long mn = ~0ull, mx = 0, an = ~0ull, o = 0;
    for (int w = 0; w < P1_THREADS / 32; ++w) {
      for (int i = 0; i < 10; ++i) tot[i] += s_cnt[w][i];
      lb = max(lb, s_pos[w][0]); lw = max(lw, s_pos[w][1]);
      mn = min(mn, s_addr[w][0]); mx = max(mx, s_addr[w][1]); an &= s_addr[w][2]; o |= s_addr[w][3];
    }
    r.n_instr = tot[0]; r.n_rd = tot[1]; r.n_wr = tot[2]; r.n_br = tot[3]; r.n_wgb = tot[4];
    r.n_wib = tot[5]; r.n_wir = tot[6]; r.n_wie = tot[7]; r.n_bar = tot[8];
    r.n_other = tot[9];  // events with a non-zero kind byte
    r.last_bnd = lb; r.last_wgb = lw;
    out[blockIdx.x] = r;
    s_lb = lb;
    if (with_stats && tot[1] + tot[2] > 0) {
      atomicMin(&st->addr_min, mn); atomicMax(&st->addr_max, mx);
      atomicAnd(&st->addr_and, an); atomicOr(&st->addr_or, o);
    }
  }
  __syncthreads();
  // instructions strictly after the range's last boundary
  const long long lb = s_lb;
  uint32_t after = 0;
  const uint64_t start = lb < 0 ? rb : ((uint64_t)lb & ~15ull);
  for (uint64_t e0 = rb + 16ull * t; e0 < re; e0 += 16ull * P1_THREADS) {
    if (e0 + 16 <= start) continue;
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
  __shared__ uint32_t s_after[P1_THREADS / 32];
  if (lane == 0) s_after[warp] = after;
  __syncthreads();
  if (t == 0) {
    uint32_t a = 0;
    for (int w = 0; w < P1_THREADS / 32; ++w) a += s_after[w];
    out[blockIdx.x].instr_after = a;
  }
}

void launch_pass1(const uint8_t* kind, const uint64_t* payload, uint64_t n, uint32_t n_ranges, uint32_t tiles_per_cta,
                  bool with_stats, RangeSum* out, DevState* st, cudaStream_t s) {
  pass1_kernel<<<n_ranges, P1_THREADS, 0, s>>>(kind, payload, n, tiles_per_cta, with_stats, out, st);
}

// ---------------------------------------------------------------------------
// main ingest pass
// ---------------------------------------------------------------------------
struct IngestSmem {
  uint64_t pay[STAGES][TILE];        // 128 B-swizzled payload rows (TMA); must be 1024 B aligned
  uint8_t kind[STAGES][TILE];
  uint64_t stage_out[TILE];          // ordered compaction staging (reads | writes | branches)
  uint32_t opc_priv[OBINS][TPB];     // lane-private opcode counts
  uint32_t wid_priv[WBINS][TPB];     // lane-private width counts (width 1..16)
  uint32_t itb_h[HBINS];
  uint32_t ipt_h[HBINS];
  unsigned long long wfirst[WBINS];
  uint32_t ws[TPB / 32][5];
  uint32_t vpos[TPB];
  uint32_t nc[5];
  long long pre_lb;
  uint32_t pre_after;
  uint64_t bar[STAGES];
};

__device__ __forceinline__ uint64_t pay_at(const uint64_t* pay, uint32_t pos) {
  const uint32_t row = pos >> 4, j = pos & 15;
  return pay[row * 16 + ((((j >> 1) ^ (row & 7))) << 1) + (j & 1)];
}

template <bool DENSE>
__global__ void __launch_bounds__(TPB, 1)
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

  // ---- carry-in at the start of this CTA's range (combine earlier ranges) ----
  // counts: sum over ranges < c; last boundary: range jb = max j with a boundary
  uint32_t cseg, clid = 0, cbyres = 0, cgseq = 0, cgkey = 0;
  unsigned long long c_rd = 0, c_wr = 0, c_br = 0;
  {
    const uint32_t c = blockIdx.x;
    long long jb = -1, lw = -1;
    uint64_t s_rd = 0, s_wr = 0, s_br = 0, s_wgb = 0;
    for (uint32_t j = t; j < c; j += TPB) {
      const RangeSum& r = a.ranges[j];
      if (r.last_bnd >= 0) jb = max(jb, (long long)j);
      lw = max(lw, (long long)r.last_wgb);
      s_rd += r.n_rd; s_wr += r.n_wr; s_br += r.n_br; s_wgb += r.n_wgb;
    }
    // block reduce (sum / max)
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
    // instructions after the last boundary: after(jb) + instrs of ranges jb+1..c-1
    uint64_t s_in = 0;
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
      const uint32_t kb = a.kind[lbpos];
      clid = (uint32_t)a.payload[lbpos];
      cbyres = kb == AIWC_K_WI_RESUME;
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
    // ---- per-thread kind summary ----
    uint32_t n_in = 0, n_rd = 0, n_wr = 0, n_br = 0, n_wg = 0;
    int lp = -1, lw = -1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t x = w[i];
      n_in += __popc(x & 0x01010101u);
      n_rd += __popc(x & 0x02020202u);
      n_wr += __popc(x & 0x04040404u);
      n_br += __popc(x & 0x08080808u);
      const uint32_t gm = m_wgb(x);
      n_wg += __popc(gm);
      const uint32_t bm = x & 0x10101010u;
      if (bm) lp = 4 * i + ((31 - __clz(bm)) >> 3);
      if (gm) lw = 4 * i + ((31 - __clz(gm)) >> 3);
    }
    uint32_t after = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x = w[i] & 0x01010101u;
      const int p0 = 4 * i;
      if (p0 + 3 <= lp) x = 0;
      else if (p0 <= lp) x &= 0xFFFFFFFFu << (8 * (lp - p0 + 1));
      after += __popc(x);
    }
    // ---- block scan ----
    const uint32_t A = n_in | (n_br << 16), B = n_rd | (n_wr << 16), C = n_wg;
    const uint32_t P = lp >= 0 ? (uint32_t)(16 * t + lp + 1) : 0u;
    const uint32_t Q = lw >= 0 ? (uint32_t)(16 * t + lw + 1) : 0u;
    const uint32_t Ai = warp_incl_sum(A), Bi = warp_incl_sum(B), Ci = warp_incl_sum(C);
    const uint32_t Pi = warp_incl_max(P), Qi = warp_incl_max(Q);
    if (lane == 31) { S.ws[warp][0] = Ai; S.ws[warp][1] = Bi; S.ws[warp][2] = Ci; S.ws[warp][3] = Pi; S.ws[warp][4] = Qi; }
    __syncthreads();
    uint32_t Ap = 0, Bp = 0, Cp = 0, Pp = 0, Qp = 0, TA = 0, TB = 0;
#pragma unroll
    for (int q = 0; q < TPB / 32; ++q) {
      const uint32_t a0 = S.ws[q][0], b0 = S.ws[q][1];
      if (q < warp) { Ap += a0; Bp += b0; Cp += S.ws[q][2]; Pp = max(Pp, S.ws[q][3]); Qp = max(Qp, S.ws[q][4]); }
      TA += a0; TB += b0;
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
    uint32_t gseq = cgseq + Cex;
    uint32_t o_rd = ex_rd, o_wr = T_rd + ex_wr;
    uint32_t o_br = (DENSE ? 0u : T_rd + T_wr) + ex_br;
    // ---- fold my 16 events ----
    const uint64_t* prow = &S.pay[s][t * 16];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const uint4 pv = *reinterpret_cast<const uint4*>(prow + (((jj ^ (t & 7))) << 1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jj + h;
        const uint32_t k = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const uint64_t p = h ? (((uint64_t)pv.w << 32) | pv.z) : (((uint64_t)pv.y << 32) | pv.x);
        if (k == AIWC_K_INSTR) {
          ++seg;
          const uint32_t opc = (uint32_t)(p >> 32), wd = (uint32_t)p;
          if (opc < OBINS) ++S.opc_priv[opc][t];
          else if (opc < a.n_opcodes) atomicAdd(&a.opc_counts[opc], 1ull);
          else flags |= F_BAD_OPCODE;
          if (wd - 1u < (uint32_t)WBINS) {
            ++S.wid_priv[wd - 1][t];
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
        } else if (is_mem(k)) {
          if (DENSE) {
            const uint64_t off = p - a.am.base;
            const uint64_t key = off >> a.am.k;
            if (p < a.am.base || p > a.am.hi || (off & a.am.low_mask) != a.am.low_const || key >= a.am.n_keys) {
              flags |= F_ADDR_HINT;
            } else {
              atomicAdd(&a.dense[key], (k & 0x04) ? (1ull << 32) : 1ull);
            }
          } else {
            if (k & 0x02) S.stage_out[o_rd++] = p; else S.stage_out[o_wr++] = p;
            amin = min(amin, (unsigned long long)p); amax = max(amax, (unsigned long long)p);
            aand &= p; aor |= p;
          }
        } else if (k == AIWC_K_BRANCH) {
          const uint64_t site = p >> 1;
          if (site >> 32) flags |= F_BAD_SITE;
          if (gkey >> 31) flags |= F_BAD_GROUP;
          max_site = max(max_site, (unsigned long long)site);
          S.stage_out[o_br++] = (site << 32) | ((uint64_t)gkey << 1) | (p & 1);
        } else if (k & 0x10) {
          if (k & 0x20) {  // wi_begin / wi_resume: open a segment
            lid = (uint32_t)p; byres = k >> 7; seg = 0;
          } else {         // barrier (always sampled) / wi_end (sampled when non-empty)
            const bool bar = k & 0x80;
            if (bar || seg) {
              if (seg < (uint32_t)HBINS) atomicAdd(&S.itb_h[seg], 1u);
              else a.itb_ovf[atomicAdd(&st->itb_ovf_n, 1ull)] = seg;
              itb_sum += seg;
            }
            const uint64_t slot = (uint64_t)(gseq - 1) * a.local_volume + lid;
            if (bar || byres) {
              if (gseq == 0 || slot >= a.ipt_tab_len) flags |= F_SLOT_RANGE;
              else atomicAdd(&a.ipt_tab[slot], (unsigned long long)seg + (bar ? 0ull : IPT_END_FLAG));
            } else {
              if (seg < (uint32_t)HBINS) atomicAdd(&S.ipt_h[seg], 1u);
              else a.ipt_ovf[atomicAdd(&st->ipt_ovf_n, 1ull)] = seg;
              ipt_sum += seg;
            }
            seg = 0;
          }
        } else if (k == AIWC_K_WG_BEGIN) {
          ++gseq; gkey = (uint32_t)p;
        } else if (k != AIWC_K_PAD && k != AIWC_K_WG_END && k != AIWC_K_KERNEL_BEGIN && k != AIWC_K_KERNEL_END) {
          flags |= F_BAD_KIND;
        }
      }
    }
    if (t == TPB - 1) { S.nc[0] = seg; S.nc[1] = lid; S.nc[2] = byres; S.nc[3] = gseq; S.nc[4] = gkey; }
    __syncthreads();
    // ---- flush ordered compaction ----
    if (!DENSE) {
      for (uint32_t i = t; i < T_rd; i += TPB) a.rd_out[c_rd + i] = S.stage_out[i];
      for (uint32_t i = t; i < T_wr; i += TPB) a.wr_out[c_wr + i] = S.stage_out[T_rd + i];
    }
    const uint32_t bb = DENSE ? 0u : T_rd + T_wr;
    for (uint32_t i = t; i < T_br; i += TPB) a.br_out[c_br + i] = S.stage_out[bb + i];
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
  }

  // ---- epilogue: flush CTA-private state ----
  __syncthreads();
  if (t < OBINS) {
    unsigned long long sum = 0;
    for (int i = 0; i < TPB; ++i) sum += S.opc_priv[t][i];
    if (sum) atomicAdd(&a.opc_counts[t], sum);
  } else if (t >= 32 && t < 32 + WBINS) {
    const int b = t - 32;
    unsigned long long sum = 0;
    for (int i = 0; i < TPB; ++i) sum += S.wid_priv[b][i];
    if (sum) {
      atomicAdd(&a.width_count[b + 1], sum);
      atomicMin(&a.width_first[b + 1], S.wfirst[b]);
    }
  }
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

cudaError_t launch_ingest(const IngestArgs& a, const CUtensorMap& kmap, const CUtensorMap& pmap, uint32_t n_ctas,
                          bool dense, cudaStream_t s) {
  const size_t smem = sizeof(IngestSmem) + 1024;
  cudaError_t e;
  if (dense) {
    e = cudaFuncSetAttribute(ingest_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ingest_kernel<true><<<n_ctas, TPB, smem, s>>>(a, kmap, pmap);
  } else {
    e = cudaFuncSetAttribute(ingest_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ingest_kernel<false><<<n_ctas, TPB, smem, s>>>(a, kmap, pmap);
  }
  return cudaGetLastError();
}

}  // namespace aiwc
