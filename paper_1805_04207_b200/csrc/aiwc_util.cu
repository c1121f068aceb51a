// aiwc_util.cu -- device-wide building blocks: exclusive scan, stable LSD radix
// sort of u64 keys over a bit range, and run-length reduction of sorted keys.
// Used by the sparse address path (onesweep-style sort + RLE replacing the
// reference's Counter/dict re-keying, metrics.py:308-321 / entropy.py:32-46)
// and by the branch path (stable grouping of per-site outcome streams,
// metrics.py:145-155).
#include <mutex>

#include "aiwc_util.cuh"

namespace aiwc {

// ---------------------------------------------------------------------------
// exclusive scan of u32 (in place), three kernels
// ---------------------------------------------------------------------------
constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_TILE = SCAN_T * SCAN_I;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T ws[SCAN_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_incl_sum(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T x = lane < (int)(blockDim.x >> 5) ? ws[lane] : (T)0;
    const T xi = warp_incl_sum(x);
    ws[lane] = xi - x;
    if (lane == (int)(blockDim.x >> 5) - 1) *total = xi;
  }
  __syncthreads();
  const T r = ws[warp] + inc - v;
  __syncthreads();
  return r;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* d, uint64_t n, T* bsum) {
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_TILE;
  T s = 0;
  for (int i = 0; i < SCAN_I; ++i) {
    const uint64_t idx = b0 + (uint64_t)i * SCAN_T + threadIdx.x;
    if (idx < n) s += d[idx];
  }
  __shared__ T tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_top_kernel(T* bsum, uint32_t nb, T* total_out) {
  __shared__ T carry_s;
  __shared__ T tot;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += SCAN_T) {
    const uint32_t i = base + threadIdx.x;
    const T v = i < nb ? bsum[i] : (T)0;
    const T ex = block_excl_scan(v, &tot);
    const T c = carry_s;
    if (i < nb) bsum[i] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry_s;
}

template <typename T>
__global__ void scan_down_kernel(T* d, uint64_t n, const T* bsum) {
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_I;
  T v[SCAN_I], s = 0;
  for (int i = 0; i < SCAN_I; ++i) {
    v[i] = (b0 + i < n) ? d[b0 + i] : (T)0;
    s += v[i];
  }
  __shared__ T tot;
  T ex = block_excl_scan(s, &tot) + bsum[blockIdx.x];
  for (int i = 0; i < SCAN_I; ++i) {
    if (b0 + i < n) d[b0 + i] = ex;
    ex += v[i];
  }
}

size_t scan_scratch_elems(uint64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 1; }

template <typename T>
static void scan_exclusive(T* d, uint64_t n, T* scratch, T* total_out, cudaStream_t s, int* kernels) {
  const uint32_t nb = (uint32_t)((n + SCAN_TILE - 1) / SCAN_TILE);
  if (nb == 0) return;
  scan_reduce_kernel<T><<<nb, SCAN_T, 0, s>>>(d, n, scratch);
  scan_top_kernel<T><<<1, SCAN_T, 0, s>>>(scratch, nb, total_out);
  scan_down_kernel<T><<<nb, SCAN_T, 0, s>>>(d, n, scratch);
  if (kernels) *kernels += 3;
}

void scan_exclusive_u32(uint32_t* d, uint64_t n, uint32_t* scratch, uint32_t* total_out, cudaStream_t s,
                        int* kernels) {
  scan_exclusive<uint32_t>(d, n, scratch, total_out, s, kernels);
}

void scan_exclusive_u64(unsigned long long* d, uint64_t n, unsigned long long* scratch, unsigned long long* total_out,
                        cudaStream_t s, int* kernels) {
  scan_exclusive<unsigned long long>(d, n, scratch, total_out, s, kernels);
}

// ---------------------------------------------------------------------------
// stable LSD radix sort, 8-bit digits
// ---------------------------------------------------------------------------
constexpr int RS_T = 256, RS_I = 16, RS_TILE = RS_T * RS_I;  // 4096 keys per block
constexpr int RS_W = RS_T / 32;

size_t radix_hist_bytes(uint64_t n) {
  const uint64_t nb = (n + RS_TILE - 1) / RS_TILE;
  return (256 * nb + scan_scratch_elems(256 * nb) + 16) * sizeof(uint32_t);
}

// Each warp owns 256 consecutive keys, item j of lane l is key warp_base + 32 j + l
// (coalesced, and j-major/lane-minor order is the key order -> stable ranks).
__global__ void __launch_bounds__(RS_T) radix_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                          uint32_t mask, uint32_t* __restrict__ hist, uint32_t nb) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += RS_T) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * RS_TILE + (uint64_t)warp * 32 * RS_I;
  // all loads in flight before the first shared-memory atomic
  uint32_t d[RS_I];
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    d[j] = i < n ? (uint32_t)(__ldcs(keys + i) >> shift) & mask : 256u;
  }
#pragma unroll
  for (int j = 0; j < RS_I; ++j)
    if (d[j] < 256u) atomicAdd(&h[d[j]], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RS_T) hist[(uint64_t)d * nb + blockIdx.x] = h[d];
}

static bool scatter_direct() {
  static const bool v = [] { const char* e = getenv("AIWC_SCATTER"); return e && atoi(e) == 0; }();
  return v;
}
// Direct scatter (passes of <= 6 bits; AIWC_SCATTER=0 forces it for A/B)
__global__ void __launch_bounds__(RS_T) radix_scatter_direct_kernel(const uint64_t* __restrict__ keys,
                                                             uint64_t* __restrict__ out, uint64_t n, int shift,
                                                             uint32_t mask, const uint32_t* __restrict__ offs,
                                                             uint32_t nb) {
  __shared__ uint32_t cnt[RS_W][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_W * 256; i += RS_T) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * RS_TILE + (uint64_t)warp * 32 * RS_I;
  uint64_t k[RS_I];
  uint32_t d[RS_I];
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {  // all loads in flight before the first atomic
    const uint64_t i = base + 32 * j + lane;
    k[j] = i < n ? __ldcs(keys + i) : 0ull;
  }
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    d[j] = i < n ? ((uint32_t)(k[j] >> shift) & mask) : 256u;
    if (i < n) atomicAdd(&cnt[warp][d[j]], 1u);
  }
  __syncthreads();
  // per digit: exclusive prefix over warps + the block's global offset
  for (int dg = threadIdx.x; dg < 256; dg += RS_T) {
    uint32_t run = offs[(uint64_t)dg * nb + blockIdx.x];
    for (int w = 0; w < RS_W; ++w) {
      const uint32_t c = cnt[w][dg];
      cnt[w][dg] = run;
      run += c;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[j]);
    if (d[j] < 256u) {
      const uint32_t pos = cnt[warp][d[j]] + __popc(peers & lt);
      out[pos] = k[j];
    }
    __syncwarp();
    if (d[j] < 256u && (peers & lt) == 0) cnt[warp][d[j]] += __popc(peers);
    __syncwarp();
  }
}

// Stable scatter of one 4096-key tile: ranks by match.any (keys in j-major / lane-minor
// order, the tile's key order), then the tile is first sorted by digit in shared memory
// and written out digit run by digit run, so the global stores are contiguous per digit
// (a direct scatter writes each warp's 32 keys to up to 32 buckets).
__global__ void __launch_bounds__(RS_T) radix_scatter_kernel(const uint64_t* __restrict__ keys,
                                                             uint64_t* __restrict__ out, uint64_t n, int shift,
                                                             uint32_t mask, const uint32_t* __restrict__ offs,
                                                             uint32_t nb) {
  __shared__ uint32_t cnt[RS_W][256];
  __shared__ uint32_t dstart[256];   // tile-local start of each digit (digit-major order)
  __shared__ uint32_t gbase[256];    // the digit's global position for this tile
  __shared__ uint64_t stage[RS_TILE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_W * 256; i += RS_T) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile0 = (uint64_t)blockIdx.x * RS_TILE;
  const uint64_t base = tile0 + (uint64_t)warp * 32 * RS_I;
  uint64_t k[RS_I];
  uint32_t d[RS_I];
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {  // all loads in flight before the first atomic
    const uint64_t i = base + 32 * j + lane;
    k[j] = i < n ? __ldcs(keys + i) : 0ull;
  }
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    const uint64_t i = base + 32 * j + lane;
    d[j] = i < n ? ((uint32_t)(k[j] >> shift) & mask) : 256u;
    if (i < n) atomicAdd(&cnt[warp][d[j]], 1u);
  }
  __syncthreads();
  // per digit (thread = digit; RS_T == 256): tile-local start = exclusive scan of the
  // tile totals over digits; each warp's running offset; the tile's global base
  static_assert(RS_T == 256, "one thread per digit");
  __shared__ uint32_t wsum[RS_W];
  {
    const int dg = threadIdx.x;
    uint32_t tot = 0;
    for (int w = 0; w < RS_W; ++w) tot += cnt[w][dg];
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) wsum[warp] = inc;
    gbase[dg] = offs[(uint64_t)dg * nb + blockIdx.x];
    __syncthreads();
    uint32_t start = inc - tot;
    for (int w = 0; w < warp; ++w) start += wsum[w];
    dstart[dg] = start;
    for (int w = 0; w < RS_W; ++w) {  // running offsets per warp, over the counts
      const uint32_t c = cnt[w][dg];
      cnt[w][dg] = start;
      start += c;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[j]);
    if (d[j] < 256u) stage[cnt[warp][d[j]] + __popc(peers & lt)] = k[j];
    __syncwarp();
    if (d[j] < 256u && (peers & lt) == 0) cnt[warp][d[j]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const uint32_t m = n > tile0 ? (uint32_t)(n - tile0 < RS_TILE ? n - tile0 : RS_TILE) : 0u;
  for (uint32_t p = threadIdx.x; p < m; p += RS_T) {
    const uint64_t key = stage[p];
    const uint32_t dg = (uint32_t)(key >> shift) & mask;
    out[gbase[dg] + (p - dstart[dg])] = key;
  }
}

// stable sort of keys by bits [bit_lo, bit_hi); returns the buffer holding the
// result (keys or tmp: odd digit counts end in tmp, no copy back)
uint64_t* radix_sort_u64_any(uint64_t* keys, uint64_t* tmp, uint64_t n, int bit_lo, int bit_hi, uint32_t* hist_scratch,
                             cudaStream_t s, int* kernels) {
  if (n <= 1 || bit_hi <= bit_lo) return keys;
  const uint32_t nb = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  uint32_t* hist = hist_scratch;
  uint32_t* scan_tmp = hist_scratch + 256ull * nb;
  uint64_t* src = keys;
  uint64_t* dst = tmp;
  for (int b = bit_lo; b < bit_hi; b += 8) {
    const int bits = min(8, bit_hi - b);
    const uint32_t mask = (1u << bits) - 1u;
    radix_hist_kernel<<<nb, RS_T, 0, s>>>(src, n, b, mask, hist, nb);
    scan_exclusive_u32(hist, 256ull * nb, scan_tmp, nullptr, s, kernels);
    // few digits: a warp's 32 keys land in few buckets and the direct scatter is
    // already near-contiguous; many digits: stage the tile sorted in shared memory
    if (bits <= 6 || scatter_direct())
      radix_scatter_direct_kernel<<<nb, RS_T, 0, s>>>(src, dst, n, b, mask, hist, nb);
    else
      radix_scatter_kernel<<<nb, RS_T, 0, s>>>(src, dst, n, b, mask, hist, nb);
    if (kernels) *kernels += 2;
    uint64_t* x = src; src = dst; dst = x;
  }
  return src;
}

void radix_sort_u64(uint64_t* keys, uint64_t* tmp, uint64_t n, int bit_lo, int bit_hi, uint32_t* hist_scratch,
                    cudaStream_t s, int* kernels) {
  if (n <= 1 || bit_hi <= bit_lo) return;
  const uint32_t nb = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  uint32_t* hist = hist_scratch;
  uint32_t* scan_tmp = hist_scratch + 256ull * nb;
  uint64_t* src = keys;
  uint64_t* dst = tmp;
  for (int b = bit_lo; b < bit_hi; b += 8) {
    const int bits = min(8, bit_hi - b);
    const uint32_t mask = (1u << bits) - 1u;
    radix_hist_kernel<<<nb, RS_T, 0, s>>>(src, n, b, mask, hist, nb);
    scan_exclusive_u32(hist, 256ull * nb, scan_tmp, nullptr, s, kernels);
    // few digits: a warp's 32 keys land in few buckets and the direct scatter is
    // already near-contiguous; many digits: stage the tile sorted in shared memory
    if (bits <= 6 || scatter_direct())
      radix_scatter_direct_kernel<<<nb, RS_T, 0, s>>>(src, dst, n, b, mask, hist, nb);
    else
      radix_scatter_kernel<<<nb, RS_T, 0, s>>>(src, dst, n, b, mask, hist, nb);
    if (kernels) *kernels += 2;
    uint64_t* x = src; src = dst; dst = x;
  }
  if (src != keys) cudaMemcpyAsync(keys, src, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
}

// ---------------------------------------------------------------------------
// run-length reduction over keys sorted by (key >> shift)
// mode RLE_ONES: weight 1; RLE_RW: low key bit selects read(0)/write(1) count;
// RLE_SUM: weights from `w`.
// ---------------------------------------------------------------------------
constexpr int RL_T = 256, RL_I = 8, RL_TILE = RL_T * RL_I;

__device__ __forceinline__ bool rl_head(const uint64_t* keys, uint64_t i, int shift) {
  return i == 0 || (keys[i] >> shift) != (keys[i - 1] >> shift);
}

__global__ void rle_count_kernel(const uint64_t* __restrict__ keys, uint64_t n, int shift, uint32_t* bc) {
  const uint64_t b0 = (uint64_t)blockIdx.x * RL_TILE + (uint64_t)threadIdx.x * RL_I;
  uint32_t c = 0;
  for (int i = 0; i < RL_I; ++i)
    if (b0 + i < n && rl_head(keys, b0 + i, shift)) ++c;
  __shared__ uint32_t tot;
  block_excl_scan(c, &tot);
  if (threadIdx.x == 0) bc[blockIdx.x] = tot;
}

__global__ void rle_write_kernel(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ wts,
                                 uint64_t n, int shift, int mode, const uint32_t* bc, uint64_t* out_key,
                                 unsigned long long* out_a, unsigned long long* out_b) {
  const uint64_t b0 = (uint64_t)blockIdx.x * RL_TILE + (uint64_t)threadIdx.x * RL_I;
  uint32_t c = 0;
  for (int i = 0; i < RL_I; ++i)
    if (b0 + i < n && rl_head(keys, b0 + i, shift)) ++c;
  __shared__ uint32_t tot;
  int64_t seg = (int64_t)bc[blockIdx.x] + block_excl_scan(c, &tot) - 1;
  unsigned long long ra = 0, rb = 0;
  for (int i = 0; i < RL_I; ++i) {
    const uint64_t idx = b0 + i;
    if (idx >= n) break;
    const uint64_t key = keys[idx];
    if (rl_head(keys, idx, shift)) {
      if (seg >= 0 && (ra | rb)) {
        if (ra) atomicAdd(&out_a[seg], ra);
        if (rb) atomicAdd(&out_b[seg], rb);
      }
      ra = rb = 0;
      ++seg;
      out_key[seg] = key >> shift;
    }
    if (mode == RLE_RW) {
      if (key & 1) ++rb; else ++ra;
    } else if (mode == RLE_SUM) {
      ra += wts[idx];
    } else {
      ++ra;
    }
  }
  if (seg >= 0 && (ra | rb)) {
    if (ra) atomicAdd(&out_a[seg], ra);
    if (rb && out_b) atomicAdd(&out_b[seg], rb);
  }
}

size_t rle_scratch_elems(uint64_t n) {
  const uint64_t nb = (n + RL_TILE - 1) / RL_TILE;
  return nb + scan_scratch_elems(nb) + 4;
}

// Returns the number of runs (synchronizes the stream once).
uint64_t rle_reduce(const uint64_t* keys, const unsigned long long* wts, uint64_t n, int shift, int mode,
                    uint64_t* out_key, unsigned long long* out_a, unsigned long long* out_b, uint32_t* scratch,
                    cudaStream_t s, int* kernels) {
  if (n == 0) return 0;
  const uint32_t nb = (uint32_t)((n + RL_TILE - 1) / RL_TILE);
  uint32_t* bc = scratch;
  uint32_t* total = scratch + nb;
  uint32_t* sscr = scratch + nb + 1;
  rle_count_kernel<<<nb, RL_T, 0, s>>>(keys, n, shift, bc);
  scan_exclusive_u32(bc, nb, sscr, total, s, kernels);
  uint32_t h_total = 0;
  cudaMemcpyAsync(&h_total, total, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaMemsetAsync(out_a, 0, h_total * sizeof(unsigned long long), s);
  if (out_b) cudaMemsetAsync(out_b, 0, h_total * sizeof(unsigned long long), s);
  rle_write_kernel<<<nb, RL_T, 0, s>>>(keys, wts, n, shift, mode, bc, out_key, out_a, out_b);
  if (kernels) *kernels += 2;
  return h_total;
}

// per (kernel, device) high-water mark of the dynamic shared memory attribute
cudaError_t set_smem_attr(const void* kernel, int bytes) {
  struct Entry { const void* k; int dev, bytes; };
  static Entry seen[64];
  static int n_seen = 0;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n_seen; ++i)
    if (seen[i].k == kernel && seen[i].dev == dev && seen[i].bytes >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && n_seen < 64) seen[n_seen++] = Entry{kernel, dev, bytes};
  return e;
}

}  // namespace aiwc
