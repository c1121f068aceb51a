// aiwc_dense.cu -- one sweep over the dense address table (the dense memory path).
//
// Replaces finalize's merged Counter, shannon_entropy, local_entropy x10 and
// coverage_count over memory (pkg/src/aiwc/metrics.py:308-321,
// pkg/src/aiwc/entropy.py:20-66) for traces whose address span fits a table
// indexed by key = (addr - base) >> k.  Entries are u32 (count | read seen <<
// 30 | write seen << 31) below 2^30 accesses, else u64 (reads | writes << 32).
//
// Each 128-thread CTA sweeps 1024-key chunks (8 consecutive keys per thread,
// next chunk prefetched while the current one is folded).  Level n groups
// addresses by addr >> n, i.e. keys by key >> max(0, n - k): groups of up to 8
// keys are summed inside a thread, up to 256 across the warp (xor shuffles),
// 512 and 1024 across the CTA.  Every non-empty group adds one to the level's
// count-of-counts histogram (warp-aggregated with match.any: in streaming
// traces every lane carries the same count), counts >= CBINS add their fp64
// p*log2(p) term to a thread-owned partial and, at level 0, their exact value
// to the overflow list the coverage walk needs.
//
// Fast path: a warp whose 256 table entries are all equal (streaming and
// strided traces: every key touched the same number of times, or not at all)
// only extends a run-length counter held by the warp; every level <= 8 of a
// run of R such chunks with key count c is R * (256 >> j) groups of count
// c << j, recorded once when the run ends.
#include <math.h>

#include <algorithm>

#include "aiwc_internal.cuh"

namespace aiwc {

namespace {

constexpr int T = 128;      // threads per CTA
constexpr int K = 8;        // keys per thread
constexpr int CHUNK = T * K;

__device__ __forceinline__ double plogp(unsigned long long c, double m) {
  const double p = (double)c / m;
  return p * log2(p);
}

struct DenseShared {
  double part[NLEVELS][T];  // thread-owned big-count partials (deterministic reduction)
  unsigned long long wsum[T / 32];
};

struct Ctx {
  uint32_t* h;               // smem [nlev][CBINS] count-of-counts
  double* part;              // &part[0][t]
  unsigned long long* ovf;   // level-0 counts >= CBINS
  unsigned long long* ovf_n;
  double m;
  int lane;
  // one lane's group(s): c == 0 means "no group here"; safe in divergent code
  __device__ __forceinline__ void rec(int j, unsigned long long c, uint32_t mult) {
    if (c == 0) return;
    if (c < (unsigned long long)CBINS) {
      atomicAdd(&h[j * CBINS + (uint32_t)c], mult);
    } else {
      part[j * T] += plogp(c, m) * mult;
      if (j == 0)
        for (uint32_t i = 0; i < mult; ++i) ovf[atomicAdd(ovf_n, 1ull)] = c;
    }
  }
  // called by all 32 lanes together.  Streaming traces give every lane the same
  // count: then lane 0 adds the whole warp's groups at once (no 32-way conflict).
  __device__ __forceinline__ void rec_warp(int j, unsigned long long c, uint32_t mult, bool participant,
                                           uint32_t groups) {
    if (!participant) c = 0;
    const unsigned long long c0 = __shfl_sync(0xffffffffu, c, 0);  // lane 0 always participates
    const bool same = __all_sync(0xffffffffu, !participant || c == c0);
    if (same && c0 != 0 && c0 < (unsigned long long)CBINS) {
      if (lane == 0) atomicAdd(&h[j * CBINS + (uint32_t)c0], mult * groups);
    } else {
      rec(j, c, mult);
    }
  }
};

// entry -> (access count, read seen, write seen)
template <typename E>
__device__ __forceinline__ void decode(E e, unsigned long long& c, uint32_t& r, uint32_t& w);
template <>
__device__ __forceinline__ void decode<uint32_t>(uint32_t e, unsigned long long& c, uint32_t& r, uint32_t& w) {
  c = e & E32_COUNT; r = (e >> 30) & 1u; w = e >> 31;
}
template <>
__device__ __forceinline__ void decode<unsigned long long>(unsigned long long e, unsigned long long& c, uint32_t& r,
                                                           uint32_t& w) {
  const unsigned long long lo = e & 0xFFFFFFFFull, hi = e >> 32;
  c = lo + hi; r = lo != 0; w = hi != 0;
}

// CLEAR: the table is zeroed as it is read (each thread stores zeros over the words
// it just loaded), so the next trace finds it clean without a separate memset pass
template <typename E, bool CLEAR>
__global__ void __launch_bounds__(T, 4) dense_stats_kernel(E* tab,
                                                           uint64_t n_keys, int nlev, double m, DevState* st,
                                                           double* partials, uint32_t n_parts,
                                                           unsigned long long* lvl0_ovf, const uint32_t* own_bits,
                                                           uint64_t own_words, uint32_t rank, uint32_t nranks) {
  extern __shared__ uint32_t hsm[];
  __shared__ DenseShared D;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < nlev * CBINS; i += T) hsm[i] = 0;
#pragma unroll
  for (int j = 0; j < NLEVELS; ++j) D.part[j][t] = 0.0;
  __syncthreads();
  Ctx X{hsm, &D.part[0][t], lvl0_ovf, &st->lvl0_ovf_n, m, lane};
  unsigned long long ur = 0, uw = 0, fp = 0;
  const uint64_t n_chunks = (n_keys + CHUNK - 1) / CHUNK;

  auto load = [&](uint64_t ch, E (&c)[K]) {
    const uint64_t k0 = ch * CHUNK + (uint64_t)t * K;
    if (own_bits && !chunk_is_owned(own_bits, own_words, ch, rank, nranks)) {  // another rank's chunk: empty here
#pragma unroll
      for (int i = 0; i < K; ++i) c[i] = (E)0;
    } else if (k0 + K <= n_keys) {
      const uint4* p = reinterpret_cast<const uint4*>(tab + k0);
      constexpr int V = K * (int)sizeof(E) / 16;
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const uint4 v = __ldcs(p + q);  // streamed once: do not keep in L2
        *reinterpret_cast<uint4*>(&c[q * (16 / sizeof(E))]) = v;
      }
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) c[i] = (k0 + i < n_keys) ? tab[k0 + i] : (E)0;
    }
  };

  // CLEAR: zeros over a chunk's words once the fold consumed them (stores issued right
  // after the loads would wait for them and serialise the loads in flight)
  auto clear_chunk = [&](uint64_t ch) {
    if (!CLEAR) return;
    const uint64_t k0 = ch * CHUNK + (uint64_t)t * K;
    if (k0 + K <= n_keys) {
      uint4* p = reinterpret_cast<uint4*>(tab + k0);
      constexpr int V = K * (int)sizeof(E) / 16;
#pragma unroll
      for (int q = 0; q < V; ++q) __stcs(p + q, make_uint4(0u, 0u, 0u, 0u));
    } else {
      for (int i = 0; i < K; ++i)
        if (k0 + i < n_keys) tab[k0 + i] = (E)0;
    }
  };

  // warp-uniform run: run_n chunks of 256 keys, every entry == run_e (warp-uniform registers)
  E run_e = 0;
  unsigned long long run_n = 0;
  const int fast_lev = nlev < 9 ? nlev : 9;
  auto flush_run = [&]() {
    if (run_n == 0) return;
    unsigned long long c;
    uint32_t r, w;
    decode<E>(run_e, c, r, w);
    const unsigned long long keys = run_n * 256ull;
    if (lane == 0) {
      ur += r ? keys : 0ull; uw += w ? keys : 0ull; fp += keys;
      for (int j = 0; j < fast_lev; ++j) {
        const unsigned long long v = c << j, groups = keys >> j;
        if (v < (unsigned long long)CBINS) atomicAdd(&hsm[j * CBINS + (uint32_t)v], (uint32_t)groups);
        else X.part[j * T] += plogp(v, m) * (double)groups;
      }
    }
    if (c >= (unsigned long long)CBINS) {  // level-0 overflow list: one entry per key
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(X.ovf_n, keys);
      b = __shfl_sync(0xffffffffu, b, 0);
      for (unsigned long long i = lane; i < keys; i += 32) X.ovf[b + i] = c;
    }
    run_n = 0;
  };

  // fold one chunk (all lanes, CTA-uniform)
  auto fold = [&](const E (&cur)[K]) {
      bool same = true;
#pragma unroll
      for (int i = 1; i < K; ++i) same &= cur[i] == cur[0];
      const E e0 = __shfl_sync(0xffffffffu, cur[0], 0);
      unsigned long long s;  // sum of the warp's 256 counts (levels 9, 10)
      if (__all_sync(0xffffffffu, same && cur[0] == e0)) {
        // ---- warp-uniform chunk: extend the run ----
        if (e0 != run_e) { flush_run(); run_e = e0; }
        if (e0) ++run_n;
        unsigned long long c0;
        uint32_t r0, w0;
        decode<E>(e0, c0, r0, w0);
        s = c0 * 256ull;
      } else {
        unsigned long long c[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          uint32_t r, w;
          decode<E>(cur[i], c[i], r, w);
          ur += r; uw += w; fp += c[i] != 0;
        }
        // level 0: one warp-wide add when every lane's 8 counts agree, else per-thread runs
        bool uni = true;
#pragma unroll
        for (int i = 1; i < K; ++i) uni &= c[i] == c[0];
        if (__all_sync(0xffffffffu, uni)) {
          X.rec_warp(0, c[0], K, true, 32);
        } else {
          unsigned long long v = c[0];
          uint32_t run = 1;
#pragma unroll
          for (int i = 1; i < K; ++i) {
            if (c[i] == v) { ++run; }
            else { X.rec(0, v, run); v = c[i]; run = 1; }
          }
          X.rec(0, v, run);
        }
        unsigned long long s1[4], s2[2], s3;
#pragma unroll
        for (int i = 0; i < 4; ++i) s1[i] = c[2 * i] + c[2 * i + 1];
        s2[0] = s1[0] + s1[1]; s2[1] = s1[2] + s1[3];
        s3 = s2[0] + s2[1];
        if (nlev > 1) {
          const bool u1 = s1[0] == s1[1] && s1[1] == s1[2] && s1[2] == s1[3];
          if (__all_sync(0xffffffffu, u1)) X.rec_warp(1, s1[0], 4, true, 32);
          else { X.rec(1, s1[0], 1); X.rec(1, s1[1], 1); X.rec(1, s1[2], 1); X.rec(1, s1[3], 1); }
        }
        if (nlev > 2) {
          if (__all_sync(0xffffffffu, s2[0] == s2[1])) X.rec_warp(2, s2[0], 2, true, 32);
          else { X.rec(2, s2[0], 1); X.rec(2, s2[1], 1); }
        }
        if (nlev > 3) X.rec_warp(3, s3, 1, true, 32);
        s = s3;
#pragma unroll
        for (int j = 4; j <= 8; ++j) {
          s += __shfl_xor_sync(0xffffffffu, s, 1 << (j - 4));
          if (j < nlev) X.rec_warp(j, s, 1, (lane & ((1 << (j - 3)) - 1)) == 0, 32u >> (j - 3));
        }
      }
      if (nlev > 9) {  // levels 9, 10 need the whole CTA (k < 2 only)
        if (lane == 0) D.wsum[warp] = s;
        __syncthreads();
        if (t == 0) {
          const unsigned long long g[3] = {D.wsum[0] + D.wsum[1], D.wsum[2] + D.wsum[3],
                                           D.wsum[0] + D.wsum[1] + D.wsum[2] + D.wsum[3]};
          for (int q = 0; q < 3; ++q) {
            const int j = q < 2 ? 9 : 10;
            if (j >= nlev || g[q] == 0) continue;
            if (g[q] < (unsigned long long)CBINS) atomicAdd(&hsm[j * CBINS + (uint32_t)g[q]], 1u);
            else D.part[j][0] += plogp(g[q], m);
          }
        }
        __syncthreads();
      }
  };

  // four chunks in flight: fold two per iteration while the next two load
  E c0[K], c1[K], n0[K], n1[K];
  const uint64_t g = gridDim.x;
  uint64_t ch = blockIdx.x;
  if (ch < n_chunks) load(ch, c0);
  if (ch + g < n_chunks) load(ch + g, c1);
  for (; ch < n_chunks; ch += 2 * g) {
    if (ch + 2 * g < n_chunks) load(ch + 2 * g, n0);
    if (ch + 3 * g < n_chunks) load(ch + 3 * g, n1);
    fold(c0);
    clear_chunk(ch);
    if (ch + g < n_chunks) { fold(c1); clear_chunk(ch + g); }
#pragma unroll
    for (int i = 0; i < K; ++i) { c0[i] = n0[i]; c1[i] = n1[i]; }
  }
  flush_run();
  __syncthreads();
  // ---- flush: counters, histograms, fixed-order fp64 partials ----
  ur = warp_sum(ur); uw = warp_sum(uw); fp = warp_sum(fp);
  if (lane == 0) {
    if (ur) atomicAdd(&st->unique_r, ur);
    if (uw) atomicAdd(&st->unique_w, uw);
    if (fp) atomicAdd(&st->footprint, fp);
  }
  if (t < nlev) {
    double v = 0.0;
    for (int i = 0; i < T; ++i) v += D.part[t][i];
    partials[t * n_parts + blockIdx.x] = v;
  }
  for (int i = t; i < nlev * CBINS; i += T) {
    const uint32_t v = hsm[i];
    if (v) {
      if (i < CBINS) atomicAdd(&st->cnt_hist0[i], (unsigned long long)v);
      else atomicAdd(&st->cnt_hist[i / CBINS][i % CBINS], (unsigned long long)v);
    }
  }
}

}  // namespace

template <typename E>
static void dense_stats_launch(void* tab, bool clear, uint32_t n_ctas, size_t smem, cudaStream_t s, uint64_t n_keys,
                               int nlev, double m, DevState* st, double* partials, unsigned long long* ovf,
                               const uint32_t* own_bits, uint64_t own_words, uint32_t rank, uint32_t nranks) {
  E* t = static_cast<E*>(tab);
  if (clear) {
    set_smem_once(dense_stats_kernel<E, true>, (int)smem);
    dense_stats_kernel<E, true><<<n_ctas, T, smem, s>>>(t, n_keys, nlev, m, st, partials, n_ctas, ovf, own_bits,
                                                        own_words, rank, nranks);
  } else {
    set_smem_once(dense_stats_kernel<E, false>, (int)smem);
    dense_stats_kernel<E, false><<<n_ctas, T, smem, s>>>(t, n_keys, nlev, m, st, partials, n_ctas, ovf, own_bits,
                                                         own_words, rank, nranks);
  }
}

void launch_dense_stats(const void* tab, bool e32, uint64_t n_keys, uint32_t k, uint64_t total_m, DevState* st,
                        double* partials, uint32_t n_ctas, uint64_t* lvl0_ovf, cudaStream_t s,
                        const uint32_t* own_bits, uint64_t own_words, uint32_t rank, uint32_t nranks, bool clear) {
  const int nlev = k >= 10 ? 1 : 11 - (int)k;
  const size_t smem = (size_t)nlev * CBINS * sizeof(uint32_t);
  unsigned long long* ovf = reinterpret_cast<unsigned long long*>(lvl0_ovf);
  void* t = const_cast<void*>(tab);
  if (e32)
    dense_stats_launch<uint32_t>(t, clear && !own_bits, n_ctas, smem, s, n_keys, nlev, (double)total_m, st, partials,
                                 ovf, own_bits, own_words, rank, nranks);
  else
    dense_stats_launch<unsigned long long>(t, clear && !own_bits, n_ctas, smem, s, n_keys, nlev, (double)total_m, st,
                                           partials, ovf, own_bits, own_words, rank, nranks);
}

}  // namespace aiwc
