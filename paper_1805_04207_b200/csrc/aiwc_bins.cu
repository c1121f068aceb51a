// aiwc_bins.cu -- random accesses into a table far larger than L2, counted by key block.
//
// A RED into a random key of a multi-GB dense table costs a DRAM sector read and
// a later write-back (C3's 2^28-key gather region: 36.6 GB of ingest traffic for
// 19.3 GB of trace).  Such accesses are counted the other way round:
//
//   zone_sample   before the ingest: sampled accesses whose trace neighbourhood
//                 (the next ZS_WIN events) holds no access within 32 keys are
//                 "random"; 64 key zones, a zone mostly random goes to the bins
//                 (device-side verdict, no host round trip);
//   ingest        accesses into random zones are appended (key | write << 31) to
//                 the warp's own segment of the bin buffer (segment = the warp
//                 range's access count, known from pass 1: no atomics);
//   compact       the warp segments into one array (scan of the fills);
//   partition     LSD radix passes on the key-block bits (8-bit digits);
//   count         one CTA per key block: shared-memory counters, then one
//                 read-modify-write of the block's table entries.
//
// Traffic per binned access: 4 B write + 4 B read (compaction) + 2 x 8 B
// (partition) + 4 B read, plus one pass over the binned zones' table; the
// statistics sweep (aiwc_dense.cu) is unchanged.  Exact: counts add, flags OR
// (the reference's merged Counter, pkg/src/aiwc/metrics.py:308-321).
#include <algorithm>

#include "aiwc_internal.cuh"
#include "aiwc_util.cuh"

namespace aiwc {

namespace {

constexpr int ZS_T = 256, ZS_CTAS = 64, ZS_WIN = 192;

// one sample per thread: the first memory access at or after a hashed position,
// and whether another access within 32 keys follows within ZS_WIN events
__global__ void __launch_bounds__(ZS_T) zone_sample_kernel(const uint8_t* __restrict__ kind,
                                                           const uint64_t* __restrict__ payload, uint64_t n,
                                                           AddrMap am, uint32_t zone_shift,
                                                           unsigned int* __restrict__ zone_counts) {
  __shared__ unsigned int zc[2 * ZONES];
  for (int i = threadIdx.x; i < 2 * ZONES; i += ZS_T) zc[i] = 0;
  __syncthreads();
  const uint64_t id = (uint64_t)blockIdx.x * ZS_T + threadIdx.x;
  uint64_t x = id * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  x = (x ^ (x >> 31)) * 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  uint64_t p = x % n;
  const uint64_t end = min(n, p + 64);
  while (p < end && !is_mem(kind[p])) ++p;
  if (p < end) {
    const uint64_t off = payload[p] - am.base;
    if (off <= am.off_max) {
      const uint64_t key = off >> am.k;
      bool near = false;
      const uint64_t wend = min(n, p + 1 + ZS_WIN);
      for (uint64_t q = p + 1; q < wend && !near; ++q) {
        if (!is_mem(kind[q])) continue;
        const uint64_t o2 = payload[q] - am.base;
        if (o2 > am.off_max) continue;
        const uint64_t k2 = o2 >> am.k;
        near = (k2 > key ? k2 - key : key - k2) <= 32;
      }
      const uint32_t z = (uint32_t)min(key >> zone_shift, (uint64_t)(ZONES - 1));
      atomicAdd(&zc[2 * z + (near ? 0 : 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * ZONES; i += ZS_T)
    if (zc[i]) atomicAdd(&zone_counts[i], zc[i]);
}

// zone mask: a zone with >= 16 sampled accesses, at least 3 of 4 of them random
__global__ void zone_verdict_kernel(const unsigned int* __restrict__ zone_counts, unsigned long long* zones_out) {
  if (threadIdx.x) return;
  unsigned long long m = 0;
  for (int z = 0; z < ZONES; ++z) {
    const unsigned int nearc = zone_counts[2 * z], far = zone_counts[2 * z + 1];
    if (far >= 16 && far >= 3 * nearc) m |= 1ull << z;
  }
  *zones_out = m;
}

// warp segments -> one dense array (dst offsets = exclusive scan of the fills)
__global__ void bin_compact_kernel(const uint32_t* __restrict__ seg, const unsigned long long* __restrict__ seg_base,
                                   const uint32_t* __restrict__ fill, const uint32_t* __restrict__ dst_off,
                                   uint32_t* __restrict__ out) {
  const uint32_t w = blockIdx.x;
  const uint32_t f = fill[w];
  const uint32_t* src = seg + seg_base[w];
  uint32_t* dst = out + dst_off[w];
  for (uint32_t i = threadIdx.x; i < f; i += blockDim.x) dst[i] = src[i];
}

// ---- LSD radix partition of u32 bin entries on the key-block digits ----
constexpr int RP_T = 256, RP_I = 16, RP_TILE = RP_T * RP_I, RP_W = RP_T / 32;

__global__ void __launch_bounds__(RP_T) bin_hist_kernel(const uint32_t* __restrict__ v, uint64_t n, int shift,
                                                        uint32_t* __restrict__ hist, uint32_t nb) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += RP_T) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * RP_TILE + (uint64_t)warp * 32 * RP_I;
  uint32_t d[RP_I];
#pragma unroll
  for (int j = 0; j < RP_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    d[j] = i < n ? ((__ldcs(v + i) & 0x7FFFFFFFu) >> shift) & 255u : 256u;
  }
#pragma unroll
  for (int j = 0; j < RP_I; ++j)
    if (d[j] < 256u) atomicAdd(&h[d[j]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += RP_T) hist[(uint64_t)i * nb + blockIdx.x] = h[i];
}

__global__ void __launch_bounds__(RP_T) bin_scatter_kernel(const uint32_t* __restrict__ v, uint32_t* __restrict__ out,
                                                           uint64_t n, int shift, const uint32_t* __restrict__ offs,
                                                           uint32_t nb) {
  __shared__ uint32_t cnt[RP_W][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RP_W * 256; i += RP_T) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * RP_TILE + (uint64_t)warp * 32 * RP_I;
  uint32_t k[RP_I], d[RP_I];
#pragma unroll
  for (int j = 0; j < RP_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    k[j] = i < n ? __ldcs(v + i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < RP_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    d[j] = i < n ? ((k[j] & 0x7FFFFFFFu) >> shift) & 255u : 256u;
    if (i < n) atomicAdd(&cnt[warp][d[j]], 1u);
  }
  __syncthreads();
  for (int dg = threadIdx.x; dg < 256; dg += RP_T) {
    uint32_t run = offs[(uint64_t)dg * nb + blockIdx.x];
    for (int w = 0; w < RP_W; ++w) {
      const uint32_t c = cnt[w][dg];
      cnt[w][dg] = run;
      run += c;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RP_I; ++j) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[j]);
    if (d[j] < 256u) out[cnt[warp][d[j]] + __popc(peers & lt)] = k[j];
    __syncwarp();
    if (d[j] < 256u && (peers & lt) == 0) cnt[warp][d[j]] += __popc(peers);
    __syncwarp();
  }
}

// segment bounds of each key block in the partitioned array
__global__ void bin_bounds_kernel(const uint32_t* __restrict__ v, uint64_t n, int bs, uint32_t blk_lo,
                                  uint32_t* __restrict__ starts, uint32_t* __restrict__ ends) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (v[i] & 0x7FFFFFFFu) >> bs;
    if (i == 0 || ((v[i - 1] & 0x7FFFFFFFu) >> bs) != b) starts[b - blk_lo] = (uint32_t)i;
    if (i == n - 1 || ((v[i + 1] & 0x7FFFFFFFu) >> bs) != b) ends[b - blk_lo] = (uint32_t)(i + 1);
  }
}

// one CTA per key block: count in shared memory, then add into the table block
template <bool E32>
__global__ void __launch_bounds__(1024) bin_count_kernel(const uint32_t* __restrict__ v,
                                                         const uint32_t* __restrict__ starts,
                                                         const uint32_t* __restrict__ ends, uint32_t n_blocks, int bs,
                                                         uint32_t blk_lo, void* table, uint64_t n_keys) {
  extern __shared__ uint32_t sc[];  // E32: count | read << 30 | write << 31; else reads [0, B), writes [B, 2B)
  const uint32_t B = 1u << bs;
  for (uint32_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const uint32_t lo = starts[blk], hi = ends[blk];
    if (hi <= lo) continue;
    for (uint32_t i = threadIdx.x; i < (E32 ? B : 2 * B); i += blockDim.x) sc[i] = 0;
    __syncthreads();
    for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const uint32_t e = v[i], k = (e & 0x7FFFFFFFu) & (B - 1), w = e >> 31;
      if (E32) {
        atomicAdd(&sc[k], 1u);
        atomicOr(&sc[k], E32_READ << w);
      } else {
        atomicAdd(&sc[w * B + k], 1u);
      }
    }
    __syncthreads();
    const uint64_t k0 = (uint64_t)(blk + blk_lo) << bs;
    for (uint32_t i = threadIdx.x; i < B && k0 + i < n_keys; i += blockDim.x) {
      if (E32) {
        const uint32_t c = sc[i];
        if (!c) continue;
        uint32_t* q = static_cast<uint32_t*>(table) + k0 + i;
        const uint32_t t = *q;
        *q = ((t & E32_COUNT) + (c & E32_COUNT)) | (t & ~E32_COUNT) | (c & ~E32_COUNT);
      } else {
        const uint32_t r = sc[i], w = sc[B + i];
        if (!(r | w)) continue;
        unsigned long long* q = static_cast<unsigned long long*>(table) + k0 + i;
        *q += (unsigned long long)r | ((unsigned long long)w << 32);
      }
    }
    __syncthreads();
  }
}

}  // namespace

void launch_zone_sample(const uint8_t* kind, const uint64_t* payload, uint64_t n, const AddrMap& am,
                        uint32_t zone_shift, unsigned int* zone_counts, unsigned long long* zones_out,
                        cudaStream_t s) {
  cudaMemsetAsync(zone_counts, 0, 2 * ZONES * sizeof(unsigned int), s);
  zone_sample_kernel<<<ZS_CTAS, ZS_T, 0, s>>>(kind, payload, n, am, zone_shift, zone_counts);
  zone_verdict_kernel<<<1, 32, 0, s>>>(zone_counts, zones_out);
}

size_t bin_scratch_bytes(uint64_t n_bins, uint32_t n_warps, uint64_t n_blocks) {
  const uint64_t nb = (n_bins + RP_TILE - 1) / RP_TILE;
  return 2 * ((n_bins * 4 + 255) & ~255ull) + ((256 * nb + scan_scratch_elems(256 * nb) + 64) * 4 + 255) +
         ((n_warps + scan_scratch_elems(n_warps) + 64) * 4 + 255) + 2 * (n_blocks + 64) * 4 + 1024;
}

// segments -> partitioned bins -> counted into the table; returns kernels launched
int bin_finish(const uint32_t* seg, const unsigned long long* seg_base, const uint32_t* fill, uint32_t n_warps,
               uint64_t n_bins, void* table, bool e32, uint64_t n_keys, void* scratch, cudaStream_t s) {
  if (!n_bins) return 0;
  int kernels = 0;
  const int bs = e32 ? 15 : 14;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t bytes) { uint8_t* q = p; p += (bytes + 255) & ~size_t(255); return q; };
  uint32_t* a = reinterpret_cast<uint32_t*>(take(n_bins * 4));
  uint32_t* b = reinterpret_cast<uint32_t*>(take(n_bins * 4));
  const uint64_t nb = (n_bins + RP_TILE - 1) / RP_TILE;
  uint32_t* hist = reinterpret_cast<uint32_t*>(take((256 * nb + scan_scratch_elems(256 * nb) + 64) * 4));
  uint32_t* offs = reinterpret_cast<uint32_t*>(take((n_warps + scan_scratch_elems(n_warps) + 64) * 4));
  // compaction: fills -> offsets
  cudaMemcpyAsync(offs, fill, (size_t)n_warps * 4, cudaMemcpyDeviceToDevice, s);
  scan_exclusive_u32(offs, n_warps, offs + n_warps + 8, nullptr, s, &kernels);
  bin_compact_kernel<<<n_warps, 256, 0, s>>>(seg, seg_base, fill, offs, a);
  ++kernels;
  // partition on the key-block bits [bs, 31)
  const uint32_t key_hi = (uint32_t)std::max<uint64_t>(n_keys, 1);
  int top = 32 - __builtin_clz(key_hi);
  uint32_t* src = a;
  uint32_t* dst = b;
  for (int sh = bs; sh < top; sh += 8) {
    bin_hist_kernel<<<(unsigned)nb, RP_T, 0, s>>>(src, n_bins, sh, hist, (uint32_t)nb);
    scan_exclusive_u32(hist, 256ull * nb, hist + 256 * nb + 8, nullptr, s, &kernels);
    bin_scatter_kernel<<<(unsigned)nb, RP_T, 0, s>>>(src, dst, n_bins, sh, hist, (uint32_t)nb);
    kernels += 2;
    std::swap(src, dst);
  }
  // block bounds, then count
  const uint32_t n_blocks = (uint32_t)((n_keys + (1ull << bs) - 1) >> bs);
  uint32_t* starts = reinterpret_cast<uint32_t*>(take((n_blocks + 64) * 4));
  uint32_t* ends = reinterpret_cast<uint32_t*>(take((n_blocks + 64) * 4));
  cudaMemsetAsync(starts, 0, (size_t)n_blocks * 4, s);
  cudaMemsetAsync(ends, 0, (size_t)n_blocks * 4, s);
  bin_bounds_kernel<<<(unsigned)std::min<uint64_t>((n_bins + 255) / 256, 148 * 8), 256, 0, s>>>(src, n_bins, bs, 0,
                                                                                               starts, ends);
  const size_t smem = (size_t)(e32 ? 1 : 2) << bs << 2;
  const unsigned grid = std::min<uint32_t>(n_blocks, 148 * 2);
  if (e32) {
    set_smem_once(bin_count_kernel<true>, (int)smem);
    bin_count_kernel<true><<<grid, 1024, smem, s>>>(src, starts, ends, n_blocks, bs, 0, table, n_keys);
  } else {
    set_smem_once(bin_count_kernel<false>, (int)smem);
    bin_count_kernel<false><<<grid, 1024, smem, s>>>(src, starts, ends, n_blocks, bs, 0, table, n_keys);
  }
  return kernels + 2;
}

}  // namespace aiwc
