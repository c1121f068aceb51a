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
// (entropy.py:112-114).  Observations are counted into one pooled 2^H table.
//
//   branch_stage_kernel    one coalesced pass (two records per 16-byte load):
//                          record -> byte (taken | head << 1), plus the
//                          (site, first position) list
//   pattern_walk_kernel    one walk over the bytes (16-record warm-up per 32
//                          records): code = pattern << 1 | taken per observation
//   pattern_count_kernel   blocks = code chunks x 2^14-pattern partitions; each
//                          block counts its partition's observations in shared
//                          memory (taken / not-taken counters: one atomic per
//                          observation, no global atomics), then writes its
//                          partition to a per-chunk partial table
//   pattern_reduce_kernel  sums the per-chunk partials into the table
//   branch_finish_kernel   yokota / linear in fixed reduction order
#include <math.h>

#include <algorithm>

#include "aiwc_util.cuh"

namespace aiwc {

constexpr int PC_T = 1024;                // threads per counting block (one block per SM: loads in flight)
constexpr int PC_PER = 32;                // records per thread per step
constexpr int PC_HALO = 16;               // warm-up window (>= history_len)
constexpr int PC_PART_BITS = 14;          // patterns per partition: 2^14 (128 KB of counters)
constexpr int PC_CHUNK_ALIGN = 16;

__device__ __forceinline__ void stage_one(uint64_t i, uint64_t r, uint64_t prev, uint8_t* __restrict__ bits,
                                          DevState* st, unsigned long long* big_list) {
  const bool head = (i == 0) || ((prev >> 1) != (r >> 1));
  bits[i] = (uint8_t)((r & 1) | (head ? 2 : 0));
  const uint64_t site = r >> 32;
  if (i == 0 || (prev >> 32) != site) {
    const unsigned long long j = atomicAdd(&st->n_sites, 1ull);
    if (j < (unsigned long long)MAX_SMALL_LIST) {
      st->site_list[2 * j] = site; st->site_list[2 * j + 1] = i;
    }
    big_list[2 * j] = site; big_list[2 * j + 1] = i;
  }
}

// two consecutive records per thread from one 16-byte load (the first one's
// predecessor is re-read, usually an L1 hit); records are 16-byte aligned
__global__ void branch_stage_kernel(const uint64_t* __restrict__ rec, uint64_t n, uint8_t* __restrict__ bits,
                                    DevState* st, unsigned long long* big_list) {
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * p < n; p += T) {
    const uint64_t i = 2 * p;
    if (i + 1 < n) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(rec + i);
      const uint64_t prev = i ? rec[i - 1] : ~v.x;
      stage_one(i, v.x, prev, bits, st, big_list);
      stage_one(i + 1, v.y, v.x, bits, st, big_list);
    } else {
      stage_one(i, rec[i], i ? rec[i - 1] : ~rec[i], bits, st, big_list);
    }
  }
}

__device__ __forceinline__ uint32_t byte_at(const uint8_t* bits, int64_t g, uint64_t n) {
  return (g < 0 || (uint64_t)g >= n) ? 2u : bits[g];  // outside the array: a stream head
}

constexpr uint32_t NO_OBS = 0xFFFFFFFFu;

// One walk over the staged bytes: code[i] = pattern << 1 | taken when record i
// is an observation, NO_OBS otherwise.  Thread = 32 consecutive records after a
// 16-record warm-up; starting "saturated" is exact because any head inside the
// window resets it.
__global__ void __launch_bounds__(256) pattern_walk_kernel(const uint8_t* __restrict__ bits, uint64_t n, uint32_t H,
                                                           uint32_t* __restrict__ code) {
  const uint32_t mask = (1u << H) - 1u;
  for (uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * PC_PER; s < n;
       s += (uint64_t)gridDim.x * blockDim.x * PC_PER) {
    uint32_t since = H, hist = 0;
    uint32_t out[PC_PER];
    const int64_t base = (int64_t)s - PC_HALO;
    const bool aligned = base >= 0 && (uint64_t)(base + PC_HALO + PC_PER) <= n;
    uint4 q[3];
    if (aligned) {
#pragma unroll
      for (int k = 0; k < 3; ++k) q[k] = *reinterpret_cast<const uint4*>(bits + base + 16 * k);
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      uint32_t word;
      if (aligned) word = k % 4 == 0 ? q[k / 4].x : k % 4 == 1 ? q[k / 4].y : k % 4 == 2 ? q[k / 4].z : q[k / 4].w;
      else
        word = byte_at(bits, base + 4 * k, n) | (byte_at(bits, base + 4 * k + 1, n) << 8) |
               (byte_at(bits, base + 4 * k + 2, n) << 16) | (byte_at(bits, base + 4 * k + 3, n) << 24);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = 4 * k + b;
        const uint32_t v = (word >> (8 * b)) & 0xFFu;
        if (v & 2) { since = 0; hist = 0; }
        if (i >= PC_HALO) out[i - PC_HALO] = since >= H ? (hist << 1) | (v & 1) : NO_OBS;
        hist = ((hist << 1) | (v & 1)) & mask;
        since = min(since + 1, H);
      }
    }
    if (s + PC_PER <= n) {
      uint4* dst = reinterpret_cast<uint4*>(code + s);
#pragma unroll
      for (int k = 0; k < PC_PER / 4; ++k) dst[k] = make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < PC_PER; ++k)
        if (s + k < n) code[s + k] = out[k];
    }
  }
}

// Counts the observations of one 2^14-pattern partition in one chunk of codes,
// entirely in shared memory, and writes the partition to the chunk's partial table.
__global__ void __launch_bounds__(PC_T) pattern_count_kernel(const uint32_t* __restrict__ code, uint64_t n,
                                                             uint32_t H, uint32_t n_parts, uint64_t chunk_len,
                                                             unsigned long long* __restrict__ partials) {
  extern __shared__ uint32_t cnt[];  // [2][part_size]: not taken, taken (one atomic per observation)
  const uint32_t part = blockIdx.x % n_parts, chunk = blockIdx.x / n_parts;
  const uint32_t part_size = (1u << H) / n_parts;
  const uint32_t shift = 31 - __clz(part_size) + 1;  // code >> shift = partition
  uint32_t* nt = cnt;
  uint32_t* tk = cnt + part_size;
  for (uint32_t i = threadIdx.x; i < 2 * part_size; i += PC_T) cnt[i] = 0;
  __syncthreads();
  const uint64_t c0 = (uint64_t)chunk * chunk_len, c1 = min(n, c0 + chunk_len);
  // coalesced 16-byte loads, eight in flight per thread; equal neighbours inside a
  // load are merged before touching shared memory (loop back-edges repeat one
  // pattern for long stretches and would serialise on one bin)
  auto add = [&](uint32_t c, uint32_t k) {
    if (c != NO_OBS && (c >> shift) == part) {
      const uint32_t slot = (c >> 1) & (part_size - 1);
      atomicAdd(((c & 1) ? tk : nt) + slot, k);
    }
  };
  auto count4 = [&](const uint4 q) {
    if (q.x == q.y && q.y == q.z && q.z == q.w) { add(q.x, 4); return; }
    add(q.x, 1); add(q.y, 1); add(q.z, 1); add(q.w, 1);
  };
  const uint64_t v0 = (c0 + 3) & ~3ull, v1 = c1 & ~3ull;  // uint4-aligned body
  for (uint64_t i = c0 + threadIdx.x; i < min(v0, c1); i += PC_T) add(code[i], 1);
  const uint4* q4 = reinterpret_cast<const uint4*>(code);
  const uint64_t nq = v1 > v0 ? (v1 - v0) / 4 : 0, q0 = v0 / 4;
  uint64_t j = threadIdx.x;
  for (; j + 7 * PC_T < nq; j += 8 * PC_T) {  // eight 16-byte loads in flight per thread
    uint4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldcs(q4 + q0 + j + u * PC_T);
#pragma unroll
    for (int u = 0; u < 8; ++u) count4(a[u]);
  }
  for (; j < nq; j += PC_T) count4(__ldcs(q4 + q0 + j));
  for (uint64_t i = max(v1, v0) + threadIdx.x; i < c1; i += PC_T) add(code[i], 1);
  __syncthreads();
  unsigned long long* out = partials + (uint64_t)chunk * (1u << H) + (uint64_t)part * part_size;
  for (uint32_t i = threadIdx.x; i < part_size; i += PC_T)
    out[i] = ((unsigned long long)(nt[i] + tk[i]) << 32) | tk[i];
}

// tab[p] = sum over chunks of the partial tables
__global__ void pattern_reduce_kernel(const unsigned long long* __restrict__ partials, uint32_t chunks, uint32_t size,
                                      unsigned long long* __restrict__ tab) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= size) return;
  unsigned long long v = 0;
  for (uint32_t c = 0; c < chunks; ++c) v += partials[(uint64_t)c * size + p];
  tab[p] = v;
}

constexpr int BF_T = 256, BF_BLOCKS = 64;

// per-block partial sums of observations, total * h(p) and total * min(p, 1 - p)
// over the pooled pattern table (entropy.py:123-132); fixed-order final reduction
__global__ void __launch_bounds__(BF_T) branch_partial_kernel(const unsigned long long* __restrict__ tab,
                                                              uint32_t size, double* __restrict__ part) {
  __shared__ double ry[BF_T / 32], rl[BF_T / 32];
  __shared__ unsigned long long ro[BF_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long obs = 0;
  double y = 0.0, l = 0.0;
  for (uint32_t i = blockIdx.x * BF_T + threadIdx.x; i < size; i += BF_T * gridDim.x) {
    const unsigned long long e = tab[i];
    const unsigned long long tot = e >> 32;
    if (!tot) continue;
    obs += tot;
    const double dt = (double)tot;
    const double p = (double)(e & 0xFFFFFFFFull) / dt;
    const double q = 1.0 - p;
    const double h = -((p > 0 ? p * log2(p) : 0.0) + (q > 0 ? q * log2(q) : 0.0));
    y += dt * h;
    l += dt * (p < q ? p : q);
  }
  obs = warp_sum(obs);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    y += __shfl_xor_sync(0xffffffffu, y, o);
    l += __shfl_xor_sync(0xffffffffu, l, o);
  }
  if (lane == 0) { ro[warp] = obs; ry[warp] = y; rl[warp] = l; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long to = 0;
    double ty = 0.0, tl = 0.0;
    for (int w = 0; w < BF_T / 32; ++w) { to += ro[w]; ty += ry[w]; tl += rl[w]; }
    part[3 * blockIdx.x] = (double)to; part[3 * blockIdx.x + 1] = ty; part[3 * blockIdx.x + 2] = tl;
  }
}

// yokota = sum w h(p), linear = sum w min(p, 1 - p), w = total / observations
__global__ void branch_finish_kernel(const double* __restrict__ part, uint32_t blocks, DevState* st) {
  if (threadIdx.x) return;
  double obs = 0.0, y = 0.0, l = 0.0;
  for (uint32_t b = 0; b < blocks; ++b) { obs += part[3 * b]; y += part[3 * b + 1]; l += part[3 * b + 2]; }
  st->n_obs = (unsigned long long)obs;
  st->yokota = obs > 0 ? y / obs : 0.0;
  st->linear = obs > 0 ? l / obs : 0.0;
}

// ---- launch geometry and scratch layout --------------------------------------
static uint32_t n_parts_for(uint32_t H) { return H > PC_PART_BITS ? 1u << (H - PC_PART_BITS) : 1u; }
static uint32_t n_chunks_for(uint64_t n, uint32_t parts) {
  const uint32_t blocks_target = 148 * 2;  // 128 KB smem: at most one block per SM at a time
  const uint32_t chunks = std::max<uint32_t>(1, blocks_target / parts);
  const uint64_t min_len = (uint64_t)PC_T * PC_PER;
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(chunks, (n + min_len - 1) / min_len));
}

// [sort tmp (8n) = observation codes (4n) + stage bytes (n)][partial tables][radix histograms][site list]
static uint64_t partial_bytes(uint64_t n) { return (uint64_t)n_chunks_for(n, 4) * (1ull << 16) * 8; }
static uint64_t branch_tmp_bytes(uint64_t n) { return ((8 * n + 15) & ~15ull) + partial_bytes(n); }

size_t branch_site_list_offset(uint64_t n) {
  return ((branch_tmp_bytes(n) + 15) & ~15ull) + ((radix_hist_bytes(n) + 15) & ~size_t(15));
}

size_t branch_scratch_bytes(uint64_t n) { return branch_site_list_offset(n) + 2 * 8 * (n + 1) + 4096; }

int branch_stats(uint64_t* recs, uint64_t n, uint32_t site_bits, uint32_t history_len, DevState* st,
                 unsigned long long* tables, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  (void)scratch_bytes;
  int kernels = 0;
  if (n == 0) return 0;
  uint8_t* base = reinterpret_cast<uint8_t*>(scratch);
  uint64_t* tmp = reinterpret_cast<uint64_t*>(base);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + ((branch_tmp_bytes(n) + 15) & ~15ull));
  unsigned long long* big = reinterpret_cast<unsigned long long*>(base + branch_site_list_offset(n));
  // stable grouping by site; the result stays in whichever buffer the last digit wrote
  const uint64_t* sorted = site_bits ? radix_sort_u64_any(recs, tmp, n, 32, 32 + (int)site_bits, hist, s, &kernels)
                                     : recs;
  // the other 8n-byte buffer is free: observation codes + stage bytes
  uint8_t* free8n = sorted == tmp ? reinterpret_cast<uint8_t*>(recs) : base;
  const uint32_t H = history_len, size = 1u << H;
  const uint32_t parts = n_parts_for(H), chunks = n_chunks_for(n, parts);
  uint32_t* code = reinterpret_cast<uint32_t*>(free8n);
  uint8_t* bits = free8n + 4 * ((n + 3) & ~3ull);
  unsigned long long* partials = reinterpret_cast<unsigned long long*>(base + ((8 * n + 15) & ~15ull));
  const uint32_t sb = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  branch_stage_kernel<<<sb, 256, 0, s>>>(sorted, n, bits, st, big);
  const uint32_t wb = (uint32_t)std::min<uint64_t>((n + 256 * PC_PER - 1) / (256 * PC_PER), 148 * 8);
  pattern_walk_kernel<<<wb, 256, 0, s>>>(bits, n, H, code);
  const uint64_t chunk_len = ((n + chunks - 1) / chunks + PC_CHUNK_ALIGN - 1) / PC_CHUNK_ALIGN * PC_CHUNK_ALIGN;
  const size_t smem = 2 * (size_t)(size / parts) * sizeof(uint32_t);
  set_smem_once(pattern_count_kernel, (int)smem);
  pattern_count_kernel<<<chunks * parts, PC_T, smem, s>>>(code, n, H, parts, chunk_len, partials);
  pattern_reduce_kernel<<<(size + 255) / 256, 256, 0, s>>>(partials, chunks, size, tables);
  // the per-chunk partial tables are consumed: their space holds the finish partials
  double* fin = reinterpret_cast<double*>(partials);
  const uint32_t fb = std::min<uint32_t>(BF_BLOCKS, (size + BF_T - 1) / BF_T);
  branch_partial_kernel<<<fb, BF_T, 0, s>>>(tables, size, fin);
  branch_finish_kernel<<<1, 32, 0, s>>>(fin, fb, st);
  return kernels + 6;
}

}  // namespace aiwc
