// aiwc_branch.cu -- Yokota and average-linear branch entropy.
//
// Replaces consume()'s per-(site, group) outcome streams
// (pkg/src/aiwc/metrics.py:145-155) and entropy.branch_entropy
// (pkg/src/aiwc/entropy.py:76-133) plus the site statistics of finalize
// (metrics.py:323-341).
//
// The ingest pass wrote one record per branch execution in stream order:
//     site << 32 | group_key << 1 | taken
// A stable radix sort on the site bits groups each site's executions while
// keeping stream order, so a reference stream -- a maximal run of one site's
// executions with the same group id -- is a maximal run of equal
// (record >> 1).  Execution i is an observation iff its run started at least
// H executions earlier; its pattern is the previous H outcomes, oldest as MSB
// (entropy.py:112-114).  Observations land in one pooled 2^H table of
// (total << 32 | taken) counters.
#include <math.h>

#include <algorithm>

#include "aiwc_util.cuh"

namespace aiwc {

constexpr int PT_T = 256;
constexpr int PT_CHUNK = 64;  // records per thread

__global__ void __launch_bounds__(PT_T) pattern_kernel(const uint64_t* __restrict__ rec, uint64_t n, uint32_t H,
                                                       unsigned long long* __restrict__ tab) {
  const uint32_t mask = (H >= 32) ? 0xFFFFFFFFu : ((1u << H) - 1u);
  for (uint64_t c0 = ((uint64_t)blockIdx.x * PT_T + threadIdx.x) * PT_CHUNK; c0 < n;
       c0 += (uint64_t)gridDim.x * PT_T * PT_CHUNK) {
    const uint64_t c1 = min(n, c0 + PT_CHUNK);
    const uint64_t s0 = c0 >= H ? c0 - H : 0;
    uint64_t prev = s0 > 0 ? (rec[s0 - 1] >> 1) : ~0ull;
    uint32_t since = s0 > 0 ? H : 0, hist = 0;
    uint32_t run_pat = 0xFFFFFFFFu;
    unsigned long long run_val = 0;
    for (uint64_t i = s0; i < c1; ++i) {
      const uint64_t r = rec[i];
      const uint64_t key = r >> 1;
      const uint32_t bit = (uint32_t)(r & 1);
      if (i == 0 || key != prev) { since = 0; hist = 0; }
      if (i >= c0 && since >= H) {
        if (hist != run_pat) {
          if (run_val) atomicAdd(&tab[run_pat], run_val);
          run_pat = hist; run_val = 0;
        }
        run_val += (1ull << 32) | bit;
      }
      hist = ((hist << 1) | bit) & mask;
      since = min(since + 1, H);
      prev = key;
    }
    if (run_val) atomicAdd(&tab[run_pat], run_val);
  }
}

// site boundaries of the site-sorted records: (site, first position)
__global__ void site_heads_kernel(const uint64_t* __restrict__ rec, uint64_t n, DevState* st,
                                  unsigned long long* big_list) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t site = rec[i] >> 32;
    if (i == 0 || (rec[i - 1] >> 32) != site) {
      const unsigned long long j = atomicAdd(&st->n_sites, 1ull);
      if (j < (unsigned long long)MAX_SMALL_LIST) {
        st->site_list[2 * j] = site; st->site_list[2 * j + 1] = i;
      }
      big_list[2 * j] = site; big_list[2 * j + 1] = i;
    }
  }
}

constexpr int BF_T = 1024;

// yokota = sum_t w_t h(p_t), linear = sum_t w_t min(p_t, 1 - p_t), w_t = total_t / observations
__global__ void __launch_bounds__(BF_T) branch_finish_kernel(const unsigned long long* __restrict__ tab,
                                                             uint32_t size, DevState* st) {
  __shared__ unsigned long long ro[BF_T / 32];
  __shared__ double ry[BF_T / 32], rl[BF_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long obs = 0;
  for (uint32_t i = threadIdx.x; i < size; i += BF_T) obs += tab[i] >> 32;
  obs = warp_sum(obs);
  if (lane == 0) ro[warp] = obs;
  __syncthreads();
  obs = 0;
  for (int w = 0; w < BF_T / 32; ++w) obs += ro[w];
  double y = 0.0, l = 0.0;
  if (obs) {
    const double dobs = (double)obs;
    for (uint32_t i = threadIdx.x; i < size; i += BF_T) {
      const unsigned long long e = tab[i];
      const unsigned long long tot = e >> 32;
      if (!tot) continue;
      const double dt = (double)tot;
      const double p = (double)(e & 0xFFFFFFFFull) / dt;
      const double q = 1.0 - p;
      const double h = -((p > 0 ? p * log2(p) : 0.0) + (q > 0 ? q * log2(q) : 0.0));
      const double wgt = dt / dobs;
      y += wgt * h;
      l += wgt * (p < q ? p : q);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    y += __shfl_xor_sync(0xffffffffu, y, o);
    l += __shfl_xor_sync(0xffffffffu, l, o);
  }
  if (lane == 0) { ry[warp] = y; rl[warp] = l; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ty = 0.0, tl = 0.0;
    for (int w = 0; w < BF_T / 32; ++w) { ty += ry[w]; tl += rl[w]; }
    st->yokota = ty; st->linear = tl; st->n_obs = obs;
  }
}

size_t branch_scratch_bytes(uint64_t n) {
  return n * 8 /* sort tmp */ + radix_hist_bytes(n) + 2 * 8 * (n + 1) /* site list */ + 4096;
}

int branch_stats(uint64_t* recs, uint64_t n, uint32_t site_bits, uint32_t history_len, DevState* st,
                 unsigned long long* tables, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  (void)scratch_bytes;
  int kernels = 0;
  if (n == 0) return 0;
  uint64_t* tmp = reinterpret_cast<uint64_t*>(scratch);
  uint32_t* hist = reinterpret_cast<uint32_t*>(tmp + n);
  unsigned long long* big = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<uint8_t*>(hist) + ((radix_hist_bytes(n) + 15) & ~size_t(15)));
  if (site_bits) radix_sort_u64(recs, tmp, n, 32, 32 + (int)site_bits, hist, s, &kernels);
  const uint64_t per = (uint64_t)PT_T * PT_CHUNK;
  const uint32_t blocks = (uint32_t)std::min<uint64_t>((n + per - 1) / per, 148 * 8);
  const uint32_t size = 1u << history_len;
  cudaMemsetAsync(tables, 0, size * sizeof(unsigned long long), s);
  pattern_kernel<<<blocks, PT_T, 0, s>>>(recs, n, history_len, tables);
  const uint32_t hb = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  site_heads_kernel<<<hb, 256, 0, s>>>(recs, n, st, big);
  branch_finish_kernel<<<1, BF_T, 0, s>>>(tables, size, st);
  return kernels + 3;
}

}  // namespace aiwc
