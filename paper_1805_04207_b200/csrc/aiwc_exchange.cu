// aiwc_exchange.cu -- the multi-GPU dense exchange.
//
// Every rank ingests its work-group shard into a dense table over the WHOLE
// job's key map (key = (addr - base) >> k from the all-gathered address
// statistics), exactly as the single-GPU ingest does, and marks the 1024-key
// chunks it touches in a bitmap.  Chunks are the exchange unit: an LSB-skip
// level <= 10 groups keys of one chunk only, so a chunk's statistics need its
// complete counts at one rank -- its owner:
//
//   owner(c) = the only rank that touched c, when exactly one did (streaming
//              shards: nearly every chunk, nothing moves), else hash(c) % nranks
//              (chunks many ranks touch -- gathers, shared scratch -- spread evenly).
//
// A rank packs its touched chunks owned elsewhere as runs of equal non-zero
// table entries (two words: key | length << 32, entry), grouped by owner, for
// one all-to-all; the owner adds the received runs into its own table and sweeps
// its owned chunks with the single-GPU dense statistics kernel (the reference's
// merge_accumulators additivity, pkg/src/aiwc/metrics.py:235-270, is what makes
// the per-key sums exact).  Finally every chunk a rank wrote is cleared again, so
// the next trace starts from a clean table without a full-table memset.
#include "aiwc_internal.cuh"

namespace aiwc {

namespace {

constexpr int XT = 256;            // threads per CTA
constexpr int XW = XT / 32;

template <typename E>
__device__ __forceinline__ E shfl_e(E v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <typename E>
__device__ __forceinline__ E shfl_up_e(E v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }

// Runs of one chunk owned by another rank.  Row q of the chunk = keys 32 q + lane
// (coalesced loads); position i = 32 q + lane.  A position is a boundary when its
// entry differs from the previous one (position 0 always), a head when it is a
// non-zero boundary; a run ends at the next boundary.
template <typename E>
__global__ void __launch_bounds__(XT) pack_kernel(const E* __restrict__ tab, const uint32_t* __restrict__ all_bits,
                                                  uint64_t words, uint32_t rank, uint32_t nranks, int pass,
                                                  unsigned long long* __restrict__ cursor, uint64_t* __restrict__ out) {
  __shared__ uint32_t s_bm[XW][33];
  __shared__ uint32_t s_pre[XW][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* mine = all_bits + (uint64_t)rank * words;
  const uint64_t n_warps = (uint64_t)gridDim.x * XW;
  for (uint64_t w = (uint64_t)blockIdx.x * XW + warp; w < words; w += n_warps) {
    uint32_t bits = mine[w];
    while (bits) {
      const uint32_t b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint64_t c = w * 32 + b;
      if (chunk_owner(all_bits, words, c, nranks) == rank) continue;
      const E* src = tab + c * 1024;
      E e[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) e[q] = src[32 * q + lane];
      uint32_t hm_lane = 0;  // lane q: heads of row q
      uint32_t bm_lane = 0;  // lane q: boundaries of row q
      E last = 0;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        E prev = shfl_up_e(e[q], 1);
        const E wrap = shfl_e(last, 31);
        if (lane == 0) prev = wrap;
        const bool bnd = (q == 0 && lane == 0) || e[q] != prev;
        const uint32_t bm = __ballot_sync(0xffffffffu, bnd);
        const uint32_t hm = __ballot_sync(0xffffffffu, bnd && e[q] != 0);
        if (lane == q) { bm_lane = bm; hm_lane = hm; }
        last = e[q];
      }
      // heads before each row (exclusive scan over rows = lanes)
      uint32_t cnt = __popc(hm_lane), inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
      s_bm[warp][lane] = bm_lane;
      s_pre[warp][lane] = inc - cnt;
      s_bm[warp][32] = 1u;  // position 1024 ends every run
      __syncwarp();
      unsigned long long base = 0;
      if (lane == 0 && total) base = atomicAdd(&cursor[chunk_owner(all_bits, words, c, nranks)], (unsigned long long)total);
      if (pass == 1 && total) {
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t hm = __shfl_sync(0xffffffffu, hm_lane, q);
          if (!((hm >> lane) & 1u)) continue;
          // run end: the next boundary after position 32 q + lane
          uint32_t qq = q, m = s_bm[warp][q] & ~((2u << lane) - 1u);
          while (!m) { ++qq; m = qq < 32 ? s_bm[warp][qq] : 1u; }
          const uint32_t end = qq < 32 ? 32 * qq + (__ffs(m) - 1) : 1024u;
          const uint32_t pos = 32 * q + lane;
          const uint64_t slot = base + s_pre[warp][q] + __popc(hm & ((1u << lane) - 1u));
          out[2 * slot] = (c * 1024 + pos) | ((uint64_t)(end - pos) << 32);
          out[2 * slot + 1] = (uint64_t)e[q];
        }
      }
      __syncwarp();
    }
  }
}

// owner side: add the received runs into the own table (entries add; u32 entries
// OR their read / write flags); a key outside the owned chunks is an error
template <typename E>
__global__ void apply_kernel(E* __restrict__ tab, const uint64_t* __restrict__ runs, uint64_t n_runs, uint64_t n_keys,
                             const uint32_t* __restrict__ all_bits, uint64_t words, uint32_t rank, uint32_t nranks,
                             unsigned long long* flags) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_runs; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w0 = runs[2 * r], v = runs[2 * r + 1];
    const uint64_t key = w0 & 0xFFFFFFFFull, len = w0 >> 32;
    if (len == 0 || len > 1024 || key + len > n_keys || ((key & 1023) + len) > 1024 ||
        chunk_owner(all_bits, words, key >> 10, nranks) != rank) {
      atomicOr(flags, (unsigned long long)F_SLOT_RANGE);
      continue;
    }
    for (uint64_t i = 0; i < len; ++i) {
      if (sizeof(E) == 4) {
        uint32_t* q = reinterpret_cast<uint32_t*>(tab) + key + i;
        atomicAdd(q, (uint32_t)v & E32_COUNT);
        if ((uint32_t)v >> 30) atomicOr(q, (uint32_t)v & ~E32_COUNT);
      } else {
        atomicAdd(reinterpret_cast<unsigned long long*>(tab) + key + i, (unsigned long long)v);
      }
    }
  }
}

// every chunk this rank wrote (touched, or owned and touched by any rank) back to
// zero, then the rank's bitmap: one warp per bitmap word, coalesced stores
template <typename E>
__global__ void __launch_bounds__(XT) clear_kernel(E* __restrict__ tab, uint64_t n_keys,
                                                   const uint32_t* __restrict__ all_bits, uint64_t words,
                                                   uint32_t rank, uint32_t nranks, uint32_t* __restrict__ my_bits) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n_warps = (uint64_t)gridDim.x * XW;
  for (uint64_t w = (uint64_t)blockIdx.x * XW + warp; w < words; w += n_warps) {
    uint32_t any = 0;
    for (uint32_t r = 0; r < nranks; ++r) any |= all_bits[(uint64_t)r * words + w];
    const uint32_t mine = all_bits[(uint64_t)rank * words + w];
    while (any) {
      const uint32_t b = __ffs(any) - 1;
      any &= any - 1;
      const uint64_t c = w * 32 + b;
      if (!((mine >> b) & 1u) && chunk_owner(all_bits, words, c, nranks) != rank) continue;
      const uint64_t k0 = c * 1024, k1 = min(n_keys, k0 + 1024);
      for (uint64_t k = k0 + lane; k < k1; k += 32) tab[k] = 0;
    }
    if (lane == 0) my_bits[w] = 0;
  }
}

// ---- accumulator state export / merge (merge_accumulators, metrics.py:235-270) ----
// entry64 = count | read seen << 62 | write seen << 63 (both table forms)
template <typename E>
__device__ __forceinline__ uint64_t entry64(E e);
template <>
__device__ __forceinline__ uint64_t entry64<uint32_t>(uint32_t e) {
  return (uint64_t)(e & E32_COUNT) | ((uint64_t)((e >> 30) & 1u) << 62) | ((uint64_t)(e >> 31) << 63);
}
template <>
__device__ __forceinline__ uint64_t entry64<unsigned long long>(unsigned long long e) {
  const uint64_t r = e & 0xFFFFFFFFull, w = e >> 32;
  return (r + w) | ((uint64_t)(r != 0) << 62) | ((uint64_t)(w != 0) << 63);
}

// runs of equal non-zero entries of every chunk of the table (pass 0 counts into
// *cursor, pass 1 emits at the reserved slots); one warp per 1024-key chunk
template <typename E>
__global__ void __launch_bounds__(XT) pack_all_kernel(const E* __restrict__ tab, uint64_t n_keys, int pass,
                                                      unsigned long long* __restrict__ cursor,
                                                      uint64_t* __restrict__ out, uint64_t cap) {
  __shared__ uint32_t s_bm[XW][33];
  __shared__ uint32_t s_pre[XW][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n_chunks = (n_keys + 1023) / 1024;
  const uint64_t n_warps = (uint64_t)gridDim.x * XW;
  for (uint64_t c = (uint64_t)blockIdx.x * XW + warp; c < n_chunks; c += n_warps) {
    const E* src = tab + c * 1024;
    E e[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const uint64_t key = c * 1024 + 32 * q + lane;
      e[q] = key < n_keys ? src[32 * q + lane] : (E)0;
    }
    uint32_t hm_lane = 0, bm_lane = 0;
    E last = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      E prev = shfl_up_e(e[q], 1);
      const E wrap = shfl_e(last, 31);
      if (lane == 0) prev = wrap;
      const bool bnd = (q == 0 && lane == 0) || e[q] != prev;
      const uint32_t bm = __ballot_sync(0xffffffffu, bnd);
      const uint32_t hm = __ballot_sync(0xffffffffu, bnd && e[q] != 0);
      if (lane == q) { bm_lane = bm; hm_lane = hm; }
      last = e[q];
    }
    uint32_t cnt = __popc(hm_lane), inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    if (!total) continue;
    s_bm[warp][lane] = bm_lane;
    s_pre[warp][lane] = inc - cnt;
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cursor, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (pass == 1 && base + total <= cap) {  // (runs in chunk-claim order: a merge does not care)
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t hm = __shfl_sync(0xffffffffu, hm_lane, q);
        if (!((hm >> lane) & 1u)) continue;
        uint32_t qq = q, m = s_bm[warp][q] & ~((2u << lane) - 1u);
        while (!m) { ++qq; m = qq < 32 ? s_bm[warp][qq] : 1u; }
        const uint32_t end = qq < 32 ? 32 * qq + (__ffs(m) - 1) : 1024u;
        const uint32_t pos = 32 * q + lane;
        const uint64_t slot = base + s_pre[warp][q] + __popc(hm & ((1u << lane) - 1u));
        out[2 * slot] = (c * 1024 + pos) | ((uint64_t)(end - pos) << 32);
        out[2 * slot + 1] = entry64<E>(e[q]);
      }
    }
    __syncwarp();
  }
}

// one part's runs into the merged u64 table (reads | writes << 32 form, the
// (count, read seen, write seen) of each key kept exactly: count - 1 | 1 << 32
// when both were seen), keys translated through the addresses
__global__ void merge_apply_kernel(const uint64_t* __restrict__ runs, uint64_t n_runs, uint64_t base_p,
                                   uint64_t low_p, uint32_t k_p, uint64_t base_m, uint32_t k_m, uint64_t n_keys_m,
                                   unsigned long long* __restrict__ tab, unsigned long long* flags) {
  // one warp per run (the exported runs are long: streaming / strided traces)
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_runs; r += nw) {
    const uint64_t w0 = runs[2 * r], v = runs[2 * r + 1];
    const uint64_t key = w0 & 0xFFFFFFFFull, len = w0 >> 32;
    const uint64_t c = v & ((1ull << 62) - 1), rd = (v >> 62) & 1, wr = v >> 63;
    const unsigned long long add = (rd && wr) ? (c - 1) | (1ull << 32) : (rd ? c : (c << 32));
    for (uint64_t i = lane; i < len; i += 32) {
      const uint64_t addr = base_p + ((key + i) << k_p) + low_p;
      const uint64_t km = (addr - base_m) >> k_m;
      if (km >= n_keys_m) { atomicOr(flags, (unsigned long long)F_SLOT_RANGE); continue; }
      atomicAdd(&tab[km], add);
    }
  }
}

}  // namespace

uint64_t launch_pack_all(const void* tab, bool e32, uint64_t n_keys, unsigned long long* cursor, uint64_t* out,
                         int pass, uint32_t n_sms, cudaStream_t s, uint64_t cap) {
  const uint64_t n_chunks = (n_keys + 1023) / 1024;
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n_chunks + XW - 1) / XW, (uint64_t)n_sms * 8));
  if (e32) pack_all_kernel<uint32_t><<<grid, XT, 0, s>>>(static_cast<const uint32_t*>(tab), n_keys, pass, cursor, out,
                                                         cap);
  else pack_all_kernel<unsigned long long><<<grid, XT, 0, s>>>(static_cast<const unsigned long long*>(tab), n_keys,
                                                               pass, cursor, out, cap);
  return 1;
}

void launch_merge_apply(const uint64_t* runs, uint64_t n_runs, uint64_t base_p, uint64_t low_p, uint32_t k_p,
                        uint64_t base_m, uint32_t k_m, uint64_t n_keys_m, unsigned long long* tab,
                        unsigned long long* flags, uint32_t n_sms, cudaStream_t s) {
  if (!n_runs) return;
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n_runs + 7) / 8, (uint64_t)n_sms * 8));
  merge_apply_kernel<<<grid, 256, 0, s>>>(runs, n_runs, base_p, low_p, k_p, base_m, k_m, n_keys_m, tab, flags);
}

int launch_pack(const void* tab, bool e32, const uint32_t* all_bits, uint64_t words, uint32_t rank, uint32_t nranks,
                int pass, unsigned long long* cursor, uint64_t* out, uint32_t n_sms, cudaStream_t s) {
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((words + XW - 1) / XW, (uint64_t)n_sms * 8));
  if (e32) pack_kernel<uint32_t><<<grid, XT, 0, s>>>(static_cast<const uint32_t*>(tab), all_bits, words, rank, nranks,
                                                     pass, cursor, out);
  else pack_kernel<unsigned long long><<<grid, XT, 0, s>>>(static_cast<const unsigned long long*>(tab), all_bits,
                                                           words, rank, nranks, pass, cursor, out);
  return 1;
}

int launch_apply_runs(void* tab, bool e32, const uint64_t* runs, uint64_t n_runs, uint64_t n_keys,
                      const uint32_t* all_bits, uint64_t words, uint32_t rank, uint32_t nranks,
                      unsigned long long* flags, uint32_t n_sms, cudaStream_t s) {
  if (!n_runs) return 0;
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n_runs + 255) / 256, (uint64_t)n_sms * 8));
  if (e32) apply_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<uint32_t*>(tab), runs, n_runs, n_keys, all_bits,
                                                       words, rank, nranks, flags);
  else apply_kernel<unsigned long long><<<grid, 256, 0, s>>>(static_cast<unsigned long long*>(tab), runs, n_runs,
                                                             n_keys, all_bits, words, rank, nranks, flags);
  return 1;
}

int launch_clear_chunks(void* tab, bool e32, uint64_t n_keys, const uint32_t* all_bits, uint64_t words, uint32_t rank,
                        uint32_t nranks, uint32_t* my_bits, uint32_t n_sms, cudaStream_t s) {
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((words + XW - 1) / XW, (uint64_t)n_sms * 8));
  if (e32) clear_kernel<uint32_t><<<grid, XT, 0, s>>>(static_cast<uint32_t*>(tab), n_keys, all_bits, words, rank,
                                                      nranks, my_bits);
  else clear_kernel<unsigned long long><<<grid, XT, 0, s>>>(static_cast<unsigned long long*>(tab), n_keys, all_bits,
                                                            words, rank, nranks, my_bits);
  return 1;
}

}  // namespace aiwc
