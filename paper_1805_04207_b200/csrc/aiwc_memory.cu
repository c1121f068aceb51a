// aiwc_memory.cu -- memory footprint, 90% footprint and LSB-skip entropy.
//
// Replaces finalize's merged address Counter (pkg/src/aiwc/metrics.py:308-321)
// and entropy.shannon_entropy / local_entropy / coverage_count
// (pkg/src/aiwc/entropy.py:20-66).
//
// Both paths reduce to per-level COUNT-OF-COUNTS histograms: the entropy
// -sum p log2 p (p = c / M) and the coverage count depend only on the multiset
// of bin counts, so counts < CBINS are histogrammed exactly (integers) and the
// rare larger counts contribute their fp64 term directly (plus, for level 0,
// their exact value for the coverage walk).  Level n groups addresses by
// addr >> n; keys are (addr - base) >> k with base 1024-aligned, so level n is
// key >> max(0, n - k) and aligned blocks of 2^(10-k) keys hold every group.
//
//  dense path  keys index a table (r | w << 32 per key) filled by the ingest
//              pass; one coalesced sweep computes unique reads / writes /
//              footprint and all eleven levels (in-thread sums, warp shuffles,
//              then smem across warps).
//  sparse path addresses were compacted by the ingest pass; radix sort of the
//              varying key bits + run-length reduction gives the unique
//              (key, r, w) list, then each level is a run-length reduction of
//              the previous one.
#include <math.h>

#include <algorithm>

#include "aiwc_util.cuh"

namespace aiwc {

__device__ __forceinline__ double plogp(unsigned long long c, double m) {
  const double p = (double)c / m;
  return p * log2(p);
}

constexpr int DS_T = 128;  // threads per count-statistics CTA

// ---------------------------------------------------------------------------
// count statistics over a compact count array (sparse path, one level)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(DS_T) count_stats_kernel(const unsigned long long* __restrict__ ca,
                                                           const unsigned long long* __restrict__ cb, uint64_t n,
                                                           int level, double m, DevState* st, double* partials,
                                                           uint32_t n_parts, unsigned long long* lvl0_ovf) {
  __shared__ uint32_t h[CBINS];
  __shared__ double red[DS_T / 32];
  for (int i = threadIdx.x; i < CBINS; i += DS_T) h[i] = 0;
  __syncthreads();
  double part = 0.0;
  unsigned long long ur = 0, uw = 0;
  uint32_t cur = 0, run = 0;  // equal consecutive small counts of this thread: one atomic per run
  // a few CTAs walk the whole array: UNR elements per thread in flight
  constexpr int UNR = 8;
  const uint64_t G = (uint64_t)gridDim.x * DS_T;
  for (uint64_t i0 = (uint64_t)blockIdx.x * DS_T + threadIdx.x; i0 < n; i0 += UNR * G) {
    unsigned long long cv[UNR], wv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t i = i0 + u * G;
      cv[u] = i < n ? ca[i] : 0ull;
      wv[u] = (cb && i < n) ? cb[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      unsigned long long c = cv[u];
      if (cb) {
        const unsigned long long w = wv[u];
        ur += c != 0; uw += w != 0;
        c += w;
      }
      if (c == 0) continue;
      if (c < (unsigned long long)CBINS) {
        if ((uint32_t)c == cur) {
          ++run;
        } else {
          if (run) atomicAdd(&h[cur], run);
          cur = (uint32_t)c;
          run = 1;
        }
      } else {
        part += plogp(c, m);
        if (level == 0) lvl0_ovf[atomicAdd(&st->lvl0_ovf_n, 1ull)] = c;
      }
    }
  }
  if (run) atomicAdd(&h[cur], run);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  ur = warp_sum(ur); uw = warp_sum(uw);
  if (lane == 0) {
    red[warp] = part;
    if (ur) atomicAdd(&st->unique_r, ur);
    if (uw) atomicAdd(&st->unique_w, uw);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < DS_T / 32; ++w) v += red[w];
    partials[level * n_parts + blockIdx.x] = v;
  }
  for (int i = threadIdx.x; i < CBINS; i += DS_T) {
    if (h[i]) {
      if (level == 0) atomicAdd(&st->cnt_hist0[i], (unsigned long long)h[i]);
      else atomicAdd(&st->cnt_hist[level][i], (unsigned long long)h[i]);
    }
  }
}

size_t sparse_scratch_bytes(uint64_t m) {
  // keys, tmp, 2 level-key buffers, r, w, 2 level-count buffers + sort/RLE scratch
  return m * 8 * 8 + radix_hist_bytes(m) + rle_scratch_elems(m) * 4 + 4096;
}

// key packing: (((addr - base) >> k) << 1) | is_write  when it fits 64 bits
__global__ void pack_keys_kernel(const uint64_t* __restrict__ src, uint64_t n, uint64_t base, uint32_t k,
                                 uint64_t flag, uint64_t* __restrict__ dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (((src[i] - base) >> k) << 1) | flag;
}

__global__ void shift_copy_kernel(const uint64_t* __restrict__ src, uint64_t n, int sh, uint64_t* __restrict__ dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] >> sh;
}

// ---------------------------------------------------------------------------
// every level >= 1 in ONE sweep over the sorted unique keys (sparse path)
// ---------------------------------------------------------------------------
// Level j groups keys by key >> j; the groups of every level lie inside one group
// of the top level (key >> (nlev - 1)), so each warp takes whole top-level groups
// (its nominal range moved forward to a top-level boundary) and walks them 32
// keys at a time: per level, a head flag (key >> j differs from the previous
// key's), a segmented warp scan of the counts, and every group that ends inside
// the tile goes to that level's count-of-counts histogram (or, >= CBINS, its fp64
// term); the group still open at the tile's end carries to the next tile.
constexpr int LV_T = 256, LV_W = LV_T / 32;

__global__ void __launch_bounds__(LV_T) levels_kernel(const uint64_t* __restrict__ key,
                                                      const unsigned long long* __restrict__ cr,
                                                      const unsigned long long* __restrict__ cw, uint64_t n,
                                                      int nlev, double m, DevState* st, double* partials,
                                                      uint32_t n_parts) {
  extern __shared__ uint32_t lh[];  // [nlev - 1][CBINS]
  __shared__ double red[LV_W][NLEVELS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (nlev - 1) * CBINS; i += LV_T) lh[i] = 0;
  __syncthreads();
  const int top = nlev - 1;
  const uint64_t W = (uint64_t)gridDim.x * LV_W, gw = (uint64_t)blockIdx.x * LV_W + warp;
  // a top-level boundary at or after position p (n if none)
  auto boundary = [&](uint64_t p) -> uint64_t {
    if (p == 0 || p >= n) return p >= n ? n : 0;
    for (uint64_t q = p; q < n; q += 32) {
      const uint64_t i = q + lane;
      const bool h = i < n && (key[i] >> top) != (key[i - 1] >> top);
      const uint32_t b = __ballot_sync(0xffffffffu, h);
      if (b) return q + (__ffs(b) - 1);
    }
    return n;
  };
  const uint64_t lo = boundary(n * gw / W), hi = boundary(n * (gw + 1) / W);
  double part[NLEVELS];
#pragma unroll
  for (int j = 0; j < NLEVELS; ++j) part[j] = 0.0;
  unsigned long long csum[NLEVELS];   // open group's sum carried from the previous tile (per level)
  uint64_t ckey = 0;                  // previous tile's last key
#pragma unroll
  for (int j = 0; j < NLEVELS; ++j) csum[j] = 0;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint64_t t0 = lo; t0 < hi; t0 += 32) {
    const uint64_t i = t0 + lane;
    const bool act = i < hi;
    const uint64_t kk = act ? key[i] : 0ull;
    const unsigned long long c = act ? cr[i] + cw[i] : 0ull;
    uint64_t pk = __shfl_up_sync(0xffffffffu, kk, 1);
    if (lane == 0) pk = ckey;
    const uint32_t nact = __ballot_sync(0xffffffffu, act);
    const int last = 31 - __clz(nact);
#pragma unroll
    for (int j = 1; j < NLEVELS; ++j) {
      if (j >= nlev) break;
      const bool head = act && ((kk >> j) != (pk >> j) || (i == lo));
      const uint32_t hm = __ballot_sync(0xffffffffu, head);
      // a head at the tile's first key closes the group carried from the previous tile
      if (lane == 0 && t0 != lo && (hm & 1u)) {
        const unsigned long long g = csum[j];
        if (g < (unsigned long long)CBINS) atomicAdd(&lh[(j - 1) * CBINS + (uint32_t)g], 1u);
        else part[j] += plogp(g, m);
      }
      // segmented inclusive scan: sum over my segment up to me
      unsigned long long v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
        // add when no head in (lane - o, lane]
        const uint32_t win = (lane >= o) ? (((1u << lane) << 1) - (1u << (lane - o + 1))) : 0u;
        if (lane >= o && !(hm & win)) v += u;
      }
      // the tile's first segment continues the carried group (no head before me)
      if (!(hm & (lt | (1u << lane)))) v += csum[j];
      // my group ends here when the next position is a head, or past the tile (flushed next tile / at the end)
      const bool next_head = (hm >> (lane + 1)) & 1u;
      const bool ends = act && lane < last && next_head;
      if (ends) {
        if (v < (unsigned long long)CBINS) atomicAdd(&lh[(j - 1) * CBINS + (uint32_t)v], 1u);
        else part[j] += plogp(v, m);
      }
      csum[j] = __shfl_sync(0xffffffffu, v, last);
    }
    ckey = __shfl_sync(0xffffffffu, kk, last);
  }
  // the groups open at the warp range's end are complete (ranges end on top-level boundaries)
  if (lo < hi && lane == 0) {
    for (int j = 1; j < nlev; ++j) {
      const unsigned long long v = csum[j];
      if (v < (unsigned long long)CBINS) atomicAdd(&lh[(j - 1) * CBINS + (uint32_t)v], 1u);
      else part[j] += plogp(v, m);
    }
  }
#pragma unroll
  for (int j = 1; j < NLEVELS; ++j) {
    double x = part[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][j] = x;
  }
  __syncthreads();
  if (threadIdx.x >= 1 && threadIdx.x < nlev) {
    double x = 0.0;
    for (int w = 0; w < LV_W; ++w) x += red[w][threadIdx.x];
    partials[threadIdx.x * n_parts + blockIdx.x] = x;
  }
  for (int i = threadIdx.x; i < (nlev - 1) * CBINS; i += LV_T)
    if (lh[i]) atomicAdd(&st->cnt_hist[1 + i / CBINS][i % CBINS], (unsigned long long)lh[i]);
}

static int bitwidth(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

static void set_u64(unsigned long long* dst, unsigned long long v, cudaStream_t s) {
  // pageable H2D: the value is staged before cudaMemcpyAsync returns
  cudaMemcpyAsync(dst, &v, 8, cudaMemcpyHostToDevice, s);
}

int sparse_memory_stats(const uint64_t* rd, uint64_t n_rd, const uint64_t* wr, uint64_t n_wr, AddrMap am,
                        uint64_t total_m, DevState* st, double* partials, uint32_t n_parts, uint64_t* lvl0_ovf,
                        void* scratch, size_t scratch_bytes, cudaStream_t s) {
  int kernels = 0;
  const uint64_t m = n_rd + n_wr;
  if (m == 0) return 0;
  (void)scratch_bytes;
  uint64_t* keys = reinterpret_cast<uint64_t*>(scratch);
  uint64_t* tmp = keys + m;
  uint64_t* lkey[2] = {tmp + m, tmp + 2 * m};
  unsigned long long* ur = reinterpret_cast<unsigned long long*>(tmp + 3 * m);
  unsigned long long* uw = ur + m;
  unsigned long long* lcnt[2] = {uw + m, uw + 2 * m};
  uint32_t* hist = reinterpret_cast<uint32_t*>(uw + 3 * m);
  uint32_t* rscr = hist + radix_hist_bytes(m) / 4;
  unsigned long long* ovf = reinterpret_cast<unsigned long long*>(lvl0_ovf);
  const double dm = (double)total_m;
  const int kbits = bitwidth((am.hi - am.base) >> am.k);
  const uint32_t blocks = (uint32_t)std::min<uint64_t>((m + 255) / 256, 148 * 8);
  uint64_t U;
  int nlev;
  if (kbits <= 63) {
    // one sort of tagged keys: (((addr - base) >> k) << 1) | is_write
    pack_keys_kernel<<<blocks, 256, 0, s>>>(rd, n_rd, am.base, am.k, 0, keys);
    pack_keys_kernel<<<blocks, 256, 0, s>>>(wr, n_wr, am.base, am.k, 1, keys + n_rd);
    kernels += 2;
    radix_sort_u64(keys, tmp, m, 0, kbits + 1, hist, s, &kernels);
    U = rle_reduce(keys, nullptr, m, 1, RLE_RW, lkey[1], ur, uw, rscr, s, &kernels);
    count_stats_kernel<<<n_parts, DS_T, 0, s>>>(ur, uw, U, 0, dm, st, partials, n_parts, ovf);
    ++kernels;
    nlev = am.k >= 10 ? 1 : 11 - (int)am.k;
    set_u64(&st->footprint, U, s);
    if (nlev > 1) {  // every other level in one sweep over the unique keys
      const size_t smem = (size_t)(nlev - 1) * CBINS * 4;
      set_smem_once(levels_kernel, (int)smem);
      levels_kernel<<<n_parts, LV_T, smem, s>>>(lkey[1], ur, uw, U, nlev, dm, st, partials, n_parts);
      ++kernels;
    }
    return kernels;
  } else {
    // all 64 key bits significant: untagged sorts (reads, writes, all) of raw addresses
    cudaMemcpyAsync(keys, rd, n_rd * 8, cudaMemcpyDeviceToDevice, s);
    radix_sort_u64(keys, tmp, n_rd, 0, 64, hist, s, &kernels);
    set_u64(&st->unique_r, rle_reduce(keys, nullptr, n_rd, 0, RLE_ONES, lkey[0], lcnt[0], nullptr, rscr, s, &kernels), s);
    cudaMemcpyAsync(keys, wr, n_wr * 8, cudaMemcpyDeviceToDevice, s);
    radix_sort_u64(keys, tmp, n_wr, 0, 64, hist, s, &kernels);
    set_u64(&st->unique_w, rle_reduce(keys, nullptr, n_wr, 0, RLE_ONES, lkey[0], lcnt[0], nullptr, rscr, s, &kernels), s);
    cudaMemcpyAsync(keys, rd, n_rd * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(keys + n_rd, wr, n_wr * 8, cudaMemcpyDeviceToDevice, s);
    radix_sort_u64(keys, tmp, m, 0, 64, hist, s, &kernels);
    U = rle_reduce(keys, nullptr, m, 0, RLE_ONES, lkey[0], lcnt[0], nullptr, rscr, s, &kernels);
    count_stats_kernel<<<n_parts, DS_T, 0, s>>>(lcnt[0], nullptr, U, 0, dm, st, partials, n_parts, ovf);
    ++kernels;
    nlev = 11;  // raw addresses: level n is key >> n
  }
  set_u64(&st->footprint, U, s);
  int ci = 0;
  uint64_t cn = U;
  for (int j = 1; j < nlev; ++j) {
    const int co = 1 - ci;
    const uint64_t nn = rle_reduce(lkey[ci], lcnt[ci], cn, 1, RLE_SUM, lkey[co], lcnt[co], nullptr, rscr, s, &kernels);
    count_stats_kernel<<<n_parts, DS_T, 0, s>>>(lcnt[co], nullptr, nn, j, dm, st, partials, n_parts, nullptr);
    ++kernels;
    ci = co; cn = nn;
  }
  return kernels;
}

// ---------------------------------------------------------------------------
// entropy finishing: -(sum_c H[c] * p log2 p + big-count partials) per level
// ---------------------------------------------------------------------------
constexpr int EF_T = 1024;

// one CTA per level j: -(sum over the count-of-counts histogram and the big-count
// partials); report level n (0..10) reads level j(n) = raw ? n : max(0, n - k)
__global__ void __launch_bounds__(EF_T) entropy_finish_kernel(DevState* st, const double* partials,
                                                              uint32_t n_parts, double m, int nlev, int k,
                                                              int raw_levels) {
  __shared__ double red[EF_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x;
  const unsigned long long* H = j == 0 ? st->cnt_hist0 : st->cnt_hist[j];
  double v = 0.0;
  for (int c = threadIdx.x; c < CBINS; c += EF_T) {
    const unsigned long long h = H[c];
    if (h && c) v += (double)h * plogp((unsigned long long)c, m);
  }
  for (uint32_t b = threadIdx.x; b < n_parts; b += EF_T) v += partials[j * n_parts + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x < NLEVELS) {
    double tsum = 0.0;
    for (int w = 0; w < EF_T / 32; ++w) tsum += red[w];
    const int n = threadIdx.x;
    int jn = raw_levels ? n : (n <= k ? 0 : n - k);
    if (jn >= nlev) jn = nlev - 1;
    if (jn == j) st->entropy[n] = -tsum;
  }
}

void launch_entropy_finish(DevState* st, const double* partials, uint32_t n_parts, uint64_t total_m, uint32_t k,
                           cudaStream_t s) {
  // k == 64 marks the raw-address sparse path (levels are n directly)
  const bool raw = k == 64;
  const int nlev = raw ? 11 : (k >= 10 ? 1 : 11 - (int)k);
  entropy_finish_kernel<<<nlev, EF_T, 0, s>>>(st, partials, n_parts, (double)total_m, nlev, raw ? 0 : (int)k, raw);
}

// ---------------------------------------------------------------------------
// IPT of work-items that crossed a barrier (per-lifetime slot table)
// ---------------------------------------------------------------------------
__global__ void ipt_table_kernel(const unsigned long long* __restrict__ tab, uint64_t len, DevState* st,
                                 uint32_t* ipt_ovf) {
  __shared__ uint32_t h[HBINS];
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned long long sum = 0, cnt = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long e = tab[i];
    if (!(e & IPT_END_FLAG)) continue;
    const unsigned long long v = e & ~IPT_END_FLAG;
    ++cnt; sum += v;
    if (v < HBINS) atomicAdd(&h[v], 1u);
    else ipt_ovf[atomicAdd(&st->ipt_ovf_n, 1ull)] = (uint32_t)v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x)
    if (h[i]) atomicAdd(&st->ipt_hist[i], (unsigned long long)h[i]);
  sum = warp_sum(sum); cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(&st->ipt_sum, sum);
    atomicAdd(&st->ipt_tab_n, cnt);
  }
}

void launch_ipt_table(const unsigned long long* tab, uint64_t len, DevState* st, uint32_t* ipt_ovf, cudaStream_t s) {
  const uint32_t blocks = (uint32_t)std::min<uint64_t>((len + 255) / 256, 148 * 4);
  ipt_table_kernel<<<blocks, 256, 0, s>>>(tab, len, st, ipt_ovf);
}

// ---------------------------------------------------------------------------
// width Counter in first-appearance order (metrics.py:136, :298-306)
// ---------------------------------------------------------------------------
// First index of each width 1..16 (first-appearance order of simd widths,
// reference Counter insertion order).  The ingest pass left one presence word per
// (range, unit of PRES_TILES tiles) with bit w-1 set when width w occurs there
// (ranges are contiguous and in order, so (range, unit) order is stream order).
// width_unit_kernel: the first unit holding each width (all presence words read
// in parallel); width_pos_kernel: one block per (width, tile of that unit) finds
// the first matching instruction.
__global__ void __launch_bounds__(256) width_unit_kernel(const uint32_t* __restrict__ presence, uint64_t n_units,
                                                         unsigned long long* __restrict__ unit_first) {
  __shared__ unsigned long long s_min[WBINS];
  if (threadIdx.x < WBINS) s_min[threadIdx.x] = ~0ull;
  __syncthreads();
  uint32_t seen = 0;  // widths this thread has already reported (units ascend per thread)
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n_units;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pw = presence[u];
    for (uint32_t m = pw & ~seen & ((1u << WBINS) - 1u); m; m &= m - 1) atomicMin(&s_min[__ffs(m) - 1], u);
    seen |= pw;
  }
  __syncthreads();
  if (threadIdx.x < WBINS && s_min[threadIdx.x] != ~0ull) atomicMin(&unit_first[threadIdx.x], s_min[threadIdx.x]);
}

__global__ void __launch_bounds__(256) width_pos_kernel(const uint8_t* __restrict__ kind,
                                                        const uint64_t* __restrict__ payload, uint64_t n,
                                                        const unsigned long long* __restrict__ unit_first,
                                                        uint32_t pres_blocks, uint32_t tiles_per_range, uint32_t wt,
                                                        unsigned long long* width_first) {
  const uint32_t w = blockIdx.x / PRES_TILES + 1, t = blockIdx.x % PRES_TILES;
  const unsigned long long u = unit_first[w - 1];
  if (u == ~0ull) return;
  const uint64_t r = u / pres_blocks, b = u % pres_blocks;
  const uint64_t r_end = min(n, (r + 1) * tiles_per_range * (uint64_t)wt);
  const uint64_t lo = r * tiles_per_range * (uint64_t)wt + (b * PRES_TILES + t) * (uint64_t)wt;
  const uint64_t hi = min(r_end, lo + wt);
  unsigned long long best = ~0ull;
  for (uint64_t base = lo; base < hi; base += 16 * 256) {
    uint8_t k[16];
    uint32_t p[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // all 32 loads in flight
      const uint64_t e = base + (uint64_t)j * 256 + threadIdx.x;
      k[j] = e < hi ? kind[e] : 0;
      p[j] = e < hi ? (uint32_t)payload[e] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (k[j] == AIWC_K_INSTR && p[j] == w) best = min(best, (unsigned long long)(base + (uint64_t)j * 256 + threadIdx.x));
    if (__syncthreads_or(best != ~0ull)) break;
  }
  if (best != ~0ull) atomicMin(&width_first[w], best);
}

void launch_width_first(const uint8_t* kind, const uint64_t* payload, uint64_t n, const uint32_t* presence,
                        uint32_t n_ranges, uint32_t pres_blocks, uint32_t tiles_per_range, uint32_t wt,
                        unsigned long long* width_first, DevState* st, cudaStream_t s) {
  const uint64_t n_units = (uint64_t)n_ranges * pres_blocks;
  cudaMemsetAsync(st->width_unit, 0xFF, sizeof(st->width_unit), s);
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n_units + 1023) / 1024, 148 * 4));
  width_unit_kernel<<<g, 256, 0, s>>>(presence, n_units, st->width_unit);
  width_pos_kernel<<<WBINS * PRES_TILES, 256, 0, s>>>(kind, payload, n, st->width_unit, pres_blocks, tiles_per_range,
                                                      wt, width_first);
}

__global__ void width_list_kernel(const unsigned long long* __restrict__ count,
                                  const unsigned long long* __restrict__ first, DevState* st) {
  __shared__ unsigned long long lv[MAX_SMALL_LIST], lc[MAX_SMALL_LIST], lf[MAX_SMALL_LIST];
  __shared__ unsigned int n;
  if (threadIdx.x == 0) n = 0;
  __syncthreads();
  // widths 1..16 plus whatever the slow path saw (width 0 or > 16)
  const uint32_t lim = (uint32_t)min((unsigned long long)WIDTH_TABLE, max(17ull, st->max_width + 1));
  for (uint32_t w = threadIdx.x; w < lim; w += blockDim.x) {
    const unsigned long long c = count[w];
    if (c) {
      const unsigned int i = atomicAdd(&n, 1u);
      if (i < MAX_SMALL_LIST) { lv[i] = w; lc[i] = c; lf[i] = first[w]; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int m = min(n, (unsigned int)MAX_SMALL_LIST);
    for (unsigned int i = 1; i < m; ++i) {  // insertion sort by first index
      const unsigned long long v = lv[i], c = lc[i], f = lf[i];
      int j = (int)i - 1;
      while (j >= 0 && lf[j] > f) { lv[j + 1] = lv[j]; lc[j + 1] = lc[j]; lf[j + 1] = lf[j]; --j; }
      lv[j + 1] = v; lc[j + 1] = c; lf[j + 1] = f;
    }
    for (unsigned int i = 0; i < m; ++i) {
      st->width_list[3 * i] = lv[i]; st->width_list[3 * i + 1] = lc[i]; st->width_list[3 * i + 2] = lf[i];
    }
    st->n_widths_listed = n;
  }
}

void launch_width_list(const unsigned long long* count, const unsigned long long* first, DevState* st,
                       cudaStream_t s) {
  width_list_kernel<<<1, 1024, 0, s>>>(count, first, st);
}

}  // namespace aiwc
