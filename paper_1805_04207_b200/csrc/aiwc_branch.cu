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
#include <stdlib.h>

#include <algorithm>

#include "aiwc_util.cuh"

namespace aiwc {

constexpr int PC_T = 1024;                // threads per counting block (one block per SM: loads in flight)
constexpr int PC_PER = 32;                // records per thread per step
constexpr int PC_HALO = 16;               // warm-up window (>= history_len)
constexpr int PC_PART_BITS = 15;          // patterns per partition: 2^15 (128 KB of 16-bit counter pairs)
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

// Counts the observations of one 2^15-pattern partition in one chunk of codes,
// entirely in shared memory, and writes the partition to the chunk's partial
// table.  One 32-bit word per pattern holds two 16-bit counters (not taken,
// taken); the add that carries a counter across 0x8000 takes 0x8000 back out
// and moves it to the global overflow table (1024 threads cannot push a
// counter from 0x8000 past 0xFFFF before that subtraction lands).
__global__ void __launch_bounds__(PC_T) pattern_count_kernel(const uint32_t* __restrict__ code, uint64_t n,
                                                             uint32_t H, uint32_t n_parts, uint64_t chunk_len,
                                                             unsigned long long* __restrict__ partials,
                                                             unsigned long long* __restrict__ ovf) {
  extern __shared__ uint32_t cnt[];  // [part_size]: taken << 16 | not taken
  const uint32_t part = blockIdx.x % n_parts, chunk = blockIdx.x / n_parts;
  const uint32_t part_size = (1u << H) / n_parts;
  const uint32_t shift = 31 - __clz(part_size) + 1;  // code >> shift = partition
  for (uint32_t i = threadIdx.x; i < part_size; i += PC_T) cnt[i] = 0;
  __syncthreads();
  const uint64_t c0 = (uint64_t)chunk * chunk_len, c1 = min(n, c0 + chunk_len);
  // coalesced 16-byte loads, eight in flight per thread; equal neighbours inside a
  // load are merged before touching shared memory (loop back-edges repeat one
  // pattern for long stretches and would serialise on one bin)
  auto add = [&](uint32_t c, uint32_t k) {
    if (c != NO_OBS && (c >> shift) == part) {
      const uint32_t slot = (c >> 1) & (part_size - 1), sh = (c & 1) ? 16 : 0;
      const uint32_t old = (atomicAdd(cnt + slot, k << sh) >> sh) & 0xFFFFu;
      if (old < 0x8000u && old + k >= 0x8000u) {
        atomicSub(cnt + slot, 0x8000u << sh);
        atomicAdd(ovf + (c >> 1), (0x8000ull << 32) | ((c & 1) ? 0x8000ull : 0ull));
      }
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
  for (uint32_t i = threadIdx.x; i < part_size; i += PC_T) {
    const uint32_t w = cnt[i], nt = w & 0xFFFFu, tk = w >> 16;
    out[i] = ((unsigned long long)(nt + tk) << 32) | tk;
  }
}

// tab[p] = sum over chunks of the partial tables
__global__ void pattern_reduce_kernel(const unsigned long long* __restrict__ partials, uint32_t chunks, uint32_t size,
                                      const unsigned long long* __restrict__ ovf, unsigned long long* __restrict__ tab) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= size) return;
  unsigned long long v = ovf[p];
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


// ---- sort-free walk (traces with <= BW_MAX_SITES sites) ----------------------
//
// The records are already in trace order, and a stream's history only depends
// on the earlier records of its own site, so no global sort is needed.  The
// record array is cut into R ranges (one CTA each).  bw_pass_kernel walks every
// range once, writes every observation code that does not depend on the state
// its sites arrive with, defers the few that do, and records per range and site
// a summary of what the range does to the site's stream state:
//     present, first group, last group, reset (a stream head after the range's
//     first record of the site), n = min(tail length, H), hist = last n outcomes
// Summaries compose associatively (bw_compose): bw_scan_kernel (one block per
// site) turns them into each range's carry-in, bw_fix_kernel writes the
// deferred codes, and pattern_count_kernel counts them all.  Sites map to slots
// of a 128-entry table (more than BW_MAX_SITES sites: the sort path).
constexpr int BW_SLOTS = 128, BW_MAX_SITES = 64;
constexpr int BW_CTAS = 148 * 3;  // ranges (one CTA each; three resident per SM)
constexpr unsigned long long BW_EMPTY = ~0ull;
constexpr uint32_t BW_PRESENT = 0x80000000u, BW_RESET = 0x80000000u, BW_LOW31 = 0x7FFFFFFFu;

struct BwGlobal {
  unsigned long long* keys;    // [BW_SLOTS] site of each slot, BW_EMPTY when free
  unsigned long long* counts;  // [BW_SLOTS] executions per slot
  unsigned int* n_sites;       // sites inserted
};

__device__ __forceinline__ uint32_t bw_hash(unsigned long long site) {
  return (uint32_t)((site * 0x9E3779B97F4A7C15ull) >> 57);  // 7 bits: BW_SLOTS
}

// slot of `site` in the global table, through the block's mirror of it (slots
// never move once claimed); -1 when the table is full or (lookup only) absent
__device__ int bw_slot(unsigned long long site, volatile unsigned long long* mirror, const BwGlobal& g, bool insert) {
  uint32_t i = bw_hash(site);
  for (int probe = 0; probe < BW_SLOTS; ++probe, i = (i + 1) & (BW_SLOTS - 1)) {
    unsigned long long k = mirror[i];
    if (k == BW_EMPTY && insert) {
      k = atomicCAS(g.keys + i, BW_EMPTY, site);
      if (k == BW_EMPTY) {
        if (atomicAdd(g.n_sites, 1u) >= (unsigned)BW_MAX_SITES) return -1;
        k = site;
      }
      mirror[i] = k;
    }
    if (k == site) return i;
    if (k == BW_EMPTY) return -1;
  }
  return -1;
}

struct BwSum {
  uint32_t first, last, hist, n;  // first: BW_PRESENT | group; n: BW_RESET | min(len, H)
};

// the summary of range a followed by range b
__device__ __forceinline__ BwSum bw_compose(const BwSum a, const BwSum b, uint32_t H, uint32_t hmask) {
  if (!(b.first & BW_PRESENT)) return a;
  if (!(a.first & BW_PRESENT)) return b;
  const uint32_t an = a.n & BW_LOW31, bn = b.n & BW_LOW31;
  const bool b_reset = b.n & BW_RESET;
  const bool joins = !b_reset && a.last == (b.first & BW_LOW31);
  BwSum r;
  r.first = a.first;
  r.last = b.last;
  if (joins) {
    r.n = min(H, an + bn);
    r.hist = bn >= H ? b.hist : (uint32_t)((((uint64_t)a.hist << bn) | b.hist) & hmask);
  } else {
    r.n = bn;
    r.hist = b.hist;
  }
  if ((a.n & BW_RESET) || !joins) r.n |= BW_RESET;
  return r;
}

// One pass.  A CTA owns one contiguous range of records and takes it in tiles
// of up to BT_TILE records.  Each tile is counting-sorted by site slot into
// shared memory (stable: a warp ranks 32 records with one match.any), so each
// site's records of the tile form one contiguous block in trace order; a thread
// then walks 16 sorted positions, starting from a 16-record warm-up inside the
// block or from the site's state at the block start (carried tile to tile).
// A range does not know the state its sites arrive with, but only a site's
// first < H records of the range before its first stream head depend on it
// ("prefix" records): their codes are deferred -- (code index, k, the k in-range
// outcomes, taken) -- and bw_fix_kernel writes them once bw_scan_kernel has
// composed the ranges' end states (the summaries) into each range's carry-in.
constexpr int BT_T = 256, BT_W = BT_T / 32, BT_I = 16, BT_TILE = BT_T * BT_I, BT_PER = 16;
constexpr int BW_DEF_CAP = BW_MAX_SITES * 16;  // prefix records per range: < H <= 16 per site
constexpr uint32_t F_SEEN = 1u, F_PREFIX = 2u;

struct BwPassSmem {
  uint32_t val[BT_TILE];           // sorted records, low word: group << 1 | taken
  uint8_t slot[BT_TILE];           // slot of each sorted position
  uint32_t cnt[BT_W][BW_SLOTS];    // per-warp counts, then each warp's first position per slot
  uint32_t start[BW_SLOTS], len[BW_SLOTS];
  uint32_t wsum[BT_W];
  // per-slot stream state at the start of the tile's block, and at its end
  uint32_t fl[BW_SLOTS], last[BW_SLOTS], hist[BW_SLOTS], k[BW_SLOTS], first[BW_SLOTS];
  uint32_t nfl[BW_SLOTS], nlast[BW_SLOTS], nhist[BW_SLOTS], nk[BW_SLOTS];
  unsigned long long count[BW_SLOTS];
  unsigned long long mirror[BW_SLOTS];
  uint32_t ndef;
  int stop;
};

struct BwGeom {
  uint64_t len;       // records per CTA range (a multiple of tile)
  uint32_t tile;      // records per tile (<= BT_TILE)
  uint32_t R;         // ranges = CTAs
};

__device__ __forceinline__ unsigned long long bw_def(uint64_t idx, uint32_t slot, uint32_t k, uint32_t hist,
                                                     uint32_t t) {
  return idx | ((unsigned long long)slot << 32) | ((unsigned long long)k << 39) |
         ((unsigned long long)hist << 44) | ((unsigned long long)t << 60);
}

__global__ void __launch_bounds__(BT_T, 3) bw_pass_kernel(const uint64_t* __restrict__ rec, uint64_t n, BwGeom geo,
                                                       uint32_t H, BwGlobal g, BwSum* __restrict__ sums,
                                                       unsigned long long* __restrict__ def,
                                                       uint32_t* __restrict__ ndef, uint32_t* __restrict__ code,
                                                       DevState* st) {
  extern __shared__ __align__(16) unsigned char bw_smem_raw[];
  BwPassSmem& sm = *reinterpret_cast<BwPassSmem*>(bw_smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  const uint32_t hmask = (1u << H) - 1u;
  const uint64_t lo = min(n, (uint64_t)blockIdx.x * geo.len), hi = min(n, lo + geo.len);
  unsigned long long* mydef = def + (uint64_t)blockIdx.x * BW_DEF_CAP;
  for (int i = tid; i < BW_SLOTS; i += BT_T) {
    sm.mirror[i] = BW_EMPTY;
    sm.fl[i] = 0; sm.last[i] = 0; sm.hist[i] = 0; sm.k[i] = 0; sm.first[i] = 0;
    sm.count[i] = 0;
  }
  if (tid == 0) sm.ndef = 0;
  bool overflow = false;
  const uint32_t wbase = warp * 32 * BT_I;
  uint64_t r[BT_I];  // the tile's records; the next tile's are loaded while this one is walked
#pragma unroll
  for (int j = 0; j < BT_I; ++j) {
    const uint64_t i = lo + wbase + 32 * j + lane;
    r[j] = i < min(hi, lo + geo.tile) ? __ldcs(rec + i) : 0ull;
  }
  for (uint64_t t0 = lo; t0 < hi; t0 += geo.tile) {
    const uint32_t m = (uint32_t)(hi - t0 < geo.tile ? hi - t0 : geo.tile);
    for (int i = tid; i < BT_W * BW_SLOTS; i += BT_T) (&sm.cnt[0][0])[i] = 0;
    if (tid == 0) sm.stop = *reinterpret_cast<volatile unsigned long long*>(&st->bw_overflow) != 0;
    __syncthreads();
    if (sm.stop) break;
    // ---- slot and rank within (warp, slot) of the tile loaded into r (warp = 512 records) ----
    uint32_t sr[BT_I];  // slot << 16 | rank within (warp, slot)
#pragma unroll
    for (int j = 0; j < BT_I; ++j) {
      const bool valid = wbase + 32 * j + lane < m;
      const unsigned long long site = r[j] >> 32;
      int slot = 0;
      if (valid) {
        const uint32_t h = bw_hash(site);
        slot = sm.mirror[h] == site ? (int)h : bw_slot(site, sm.mirror, g, true);
        if (slot < 0) { overflow = true; slot = 0; }
      }
      const unsigned peers = __match_any_sync(FULL, valid ? (uint32_t)slot : 0x100u + lane);
      const int lead = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == lead && valid) {
        base = sm.cnt[warp][slot];
        sm.cnt[warp][slot] = base + __popc(peers);
      }
      base = __shfl_sync(FULL, base, lead);
      sr[j] = ((uint32_t)slot << 16) | (base + __popc(peers & lt));
    }
    __syncthreads();
    // ---- block offsets: slot blocks in slot order, warps in order inside a block ----
    if (tid < BW_SLOTS) {
      uint32_t tot = 0;
      for (int w = 0; w < BT_W; ++w) tot += sm.cnt[w][tid];
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += u;
      }
      if (lane == 31) sm.wsum[warp] = inc;
      sm.len[tid] = tot;
      sm.start[tid] = inc - tot;  // warp-local for now
    }
    __syncthreads();
    if (tid < BW_SLOTS) {
      uint32_t s0 = sm.start[tid];
      for (int w = 0; w < warp; ++w) s0 += sm.wsum[w];
      sm.start[tid] = s0;
      for (int w = 0; w < BT_W; ++w) {
        const uint32_t c = sm.cnt[w][tid];
        sm.cnt[w][tid] = s0;
        s0 += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < BT_I; ++j) {
      if (wbase + 32 * j + lane < m) {
        const uint32_t sj = sr[j] >> 16;
        const uint32_t pos = sm.cnt[warp][sj] + (sr[j] & 0xFFFFu);
        sm.val[pos] = (uint32_t)r[j];
        sm.slot[pos] = (uint8_t)sj;
      }
    }
    {
      const uint64_t t1 = t0 + geo.tile, e1 = min(hi, t1 + geo.tile);
#pragma unroll
      for (int j = 0; j < BT_I; ++j) {
        const uint64_t i = t1 + wbase + 32 * j + lane;
        r[j] = i < e1 ? __ldcs(rec + i) : 0ull;
      }
    }
    __syncthreads();
    // ---- the thread's 16 sorted positions as 16-byte shared loads ----
    const uint32_t p0 = tid * BT_PER;
    if (p0 < m) {
      uint32_t v[BT_PER];
      uint8_t so[BT_PER];
      {
        const uint4* vq = reinterpret_cast<const uint4*>(sm.val + p0);
#pragma unroll
        for (int q = 0; q < BT_PER / 4; ++q) {
          const uint4 x = vq[q];
          v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
        }
        const uint4 sq = *reinterpret_cast<const uint4*>(sm.slot + p0);
        const uint32_t sw[4] = {sq.x, sq.y, sq.z, sq.w};
#pragma unroll
        for (int q = 0; q < BT_PER; ++q) so[q] = (uint8_t)(sw[q / 4] >> (8 * (q % 4)));
      }
      uint32_t out[BT_PER];
      const uint32_t pe = min(p0 + BT_PER, m);
      const uint32_t s0 = so[0], b0 = sm.start[s0], e0 = b0 + sm.len[s0] - 1;
      // fast path (almost every thread): the 17 positions before ours and our 16 lie
      // inside one site block, in one work-group, and the block does not end here --
      // no stream head, no prefix, no state to write: every code is the previous H
      // outcomes of a 32-bit window and the taken bit
      bool fast = p0 + BT_PER <= m && p0 - b0 > BT_PER && e0 > p0 + BT_PER - 1;
      if (fast) {
        const uint32_t s4 = s0 * 0x01010101u;
        const uint4 sq = *reinterpret_cast<const uint4*>(sm.slot + p0);
        fast = sq.x == s4 && sq.y == s4 && sq.z == s4 && sq.w == s4;
      }
      if (fast) {
        const uint32_t g0 = sm.val[p0 - BT_PER - 1];
        const uint4* wq = reinterpret_cast<const uint4*>(sm.val + p0 - BT_PER);
        uint32_t x = 0, W = 0;
#pragma unroll
        for (int q = 0; q < BT_PER / 4; ++q) {
          const uint4 y = wq[q];
          const uint32_t w4[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            x |= w4[e] ^ g0;
            W |= (w4[e] & 1u) << (31 - (4 * q + e));
          }
        }
#pragma unroll
        for (int q = 0; q < BT_PER; ++q) {
          x |= v[q] ^ g0;
          W |= (v[q] & 1u) << (15 - q);
        }
        fast = (x >> 1) == 0;
#pragma unroll
        for (int q = 0; q < BT_PER; ++q) out[q] = (((W >> (16 - q)) & hmask) << 1) | (v[q] & 1u);
      }
      if (!fast) {
        uint32_t s = so[0];
        const uint32_t b = sm.start[s];
        uint32_t fl, last, hist, kk;
        if (p0 - b > BT_PER) {  // warm-up inside the block: saturated start, a head resets it
          const uint4* wq = reinterpret_cast<const uint4*>(sm.val + p0 - BT_PER);
          fl = F_SEEN; last = sm.val[p0 - BT_PER - 1] >> 1; hist = 0; kk = H;
#pragma unroll
          for (int q = 0; q < BT_PER / 4; ++q) {
            const uint4 x = wq[q];
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t gq = w4[e] >> 1;
              if (gq != last) { kk = 0; hist = 0; }
              hist = ((hist << 1) | (w4[e] & 1u)) & hmask;
              kk = min(kk + 1, H);
              last = gq;
            }
          }
        } else {  // from the block start: the state the site's previous blocks left
          fl = sm.fl[s]; last = sm.last[s]; hist = sm.hist[s]; kk = sm.k[s];
          for (uint32_t q = b; q < p0; ++q) {
            const uint32_t x = sm.val[q], gq = x >> 1;
            if (!(fl & F_SEEN)) { fl = F_SEEN | F_PREFIX; kk = 0; hist = 0; }
            else if (gq != last) { fl = F_SEEN; kk = 0; hist = 0; }
            hist = ((hist << 1) | (x & 1u)) & hmask;
            kk = min(kk + 1, H);
            last = gq;
          }
        }
        uint32_t end = b + sm.len[s] - 1;
#pragma unroll
        for (int q = 0; q < BT_PER; ++q) {
          const uint32_t p = p0 + q;
          out[q] = NO_OBS;
          if (p < pe) {
            if (so[q] != s) {  // the next site's block starts here
              s = so[q];
              end = p + sm.len[s] - 1;
              fl = sm.fl[s]; last = sm.last[s]; hist = sm.hist[s]; kk = sm.k[s];
            }
            const uint32_t gq = v[q] >> 1, t = v[q] & 1u;
            if (!(fl & F_SEEN)) {  // the site's first record in the range
              fl = F_SEEN | F_PREFIX; kk = 0; hist = 0;
              sm.first[s] = gq;
            } else if (gq != last) {  // a stream head: the state no longer depends on the carry-in
              fl = F_SEEN; kk = 0; hist = 0;
            }
            if ((fl & F_PREFIX) && kk < H) {
              const uint32_t d = atomicAdd(&sm.ndef, 1u);
              if (d < (uint32_t)BW_DEF_CAP) mydef[d] = bw_def(t0 + p, s, kk, hist, t);
              else overflow = true;  // (cannot happen: < H prefix records per site) -> the sort path
            } else if (kk >= H) {
              out[q] = (hist << 1) | t;
            }
            hist = ((hist << 1) | t) & hmask;
            kk = min(kk + 1, H);
            last = gq;
            if (p == end) { sm.nfl[s] = fl; sm.nlast[s] = last; sm.nhist[s] = hist; sm.nk[s] = kk; }
          }
        }
      }
      uint32_t* dst = code + t0 + p0;
      if (pe == p0 + BT_PER && (((uintptr_t)dst) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < BT_PER; q += 4)
          *reinterpret_cast<uint4*>(dst + q) = make_uint4(out[q], out[q + 1], out[q + 2], out[q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < BT_PER; ++q)
          if (p0 + q < pe) dst[q] = out[q];
      }
    }
    __syncthreads();
    for (int i = tid; i < BW_SLOTS; i += BT_T) {
      const uint32_t l = sm.len[i];
      if (l) {
        sm.fl[i] = sm.nfl[i]; sm.last[i] = sm.nlast[i]; sm.hist[i] = sm.nhist[i]; sm.k[i] = sm.nk[i];
        sm.count[i] += l;
      }
    }
  }
  if (__syncthreads_or(overflow)) {
    if (tid == 0) atomicOr(&st->bw_overflow, 1ull);
    return;
  }
  // the range's summary per slot (bw_compose): a prefix that never ended means no reset
  for (int i = tid; i < BW_SLOTS; i += BT_T) {
    const uint32_t f = sm.fl[i];
    sums[(uint64_t)blockIdx.x * BW_SLOTS + i] =
        BwSum{(f & F_SEEN) ? BW_PRESENT | sm.first[i] : 0u, sm.last[i], sm.hist[i],
              sm.k[i] | ((f & F_PREFIX) ? 0u : BW_RESET)};
    if (sm.count[i]) atomicAdd(g.counts + i, sm.count[i]);
  }
  if (tid == 0) ndef[blockIdx.x] = min(sm.ndef, (uint32_t)BW_DEF_CAP);
}

// The deferred prefix records: with the carry-in the range's sites arrive with.
__global__ void __launch_bounds__(256) bw_fix_kernel(const unsigned long long* __restrict__ def,
                                                     const uint32_t* __restrict__ ndef, const BwSum* __restrict__ sums,
                                                     const BwSum* __restrict__ carry, uint32_t H,
                                                     uint32_t* __restrict__ code, const DevState* st) {
  if (st->bw_overflow) return;
  const uint32_t r = blockIdx.x, nd = ndef[r];
  const uint32_t hmask = (1u << H) - 1u;
  for (uint32_t i = threadIdx.x; i < nd; i += blockDim.x) {
    const unsigned long long e = def[(uint64_t)r * BW_DEF_CAP + i];
    const uint32_t idx = (uint32_t)e, s = (uint32_t)(e >> 32) & 0x7Fu, k = (uint32_t)(e >> 39) & 0x1Fu;
    const uint32_t part = (uint32_t)(e >> 44) & 0xFFFFu, t = (uint32_t)(e >> 60) & 1u;
    const BwSum c = carry[(uint64_t)r * BW_SLOTS + s];
    const uint32_t first = sums[(uint64_t)r * BW_SLOTS + s].first & BW_LOW31;
    uint32_t out = NO_OBS;
    if ((c.first & BW_PRESENT) && c.last == first && min(H, (c.n & BW_LOW31) + k) >= H)
      out = ((uint32_t)((((uint64_t)c.hist << k) | part) & hmask) << 1) | t;
    code[idx] = out;
  }
}

// Phase 2, one block per slot: carry[r] = the composition of the summaries of
// ranges 0 .. r-1 (exclusive scan under bw_compose).
constexpr int BW_SCAN_T = 256;
__global__ void __launch_bounds__(BW_SCAN_T) bw_scan_kernel(const BwSum* __restrict__ sums, uint32_t R, uint32_t H,
                                                            BwGlobal g, BwSum* __restrict__ carry,
                                                            const DevState* st) {
  const uint32_t slot = blockIdx.x;
  if (st->bw_overflow || g.keys[slot] == BW_EMPTY) return;
  const uint32_t hmask = (1u << H) - 1u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t per = (R + BW_SCAN_T - 1) / BW_SCAN_T;
  const uint32_t r0 = min(R, threadIdx.x * per), r1 = min(R, r0 + per);
  BwSum agg{0, 0, 0, 0};
  for (uint32_t r = r0; r < r1; ++r) agg = bw_compose(agg, sums[(uint64_t)r * BW_SLOTS + slot], H, hmask);
  auto shfl = [&](const BwSum x, int src) {
    return BwSum{__shfl_sync(0xffffffffu, x.first, src), __shfl_sync(0xffffffffu, x.last, src),
                 __shfl_sync(0xffffffffu, x.hist, src), __shfl_sync(0xffffffffu, x.n, src)};
  };
  BwSum inc = agg;  // inclusive warp scan (earlier lanes on the left of the composition)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const BwSum u = shfl(inc, max(lane - o, 0));
    if (lane >= o) inc = bw_compose(u, inc, H, hmask);
  }
  __shared__ BwSum wtot[BW_SCAN_T / 32];
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  BwSum run{0, 0, 0, 0};
  for (int k = 0; k < warp; ++k) run = bw_compose(run, wtot[k], H, hmask);
  const BwSum ex = shfl(inc, max(lane - 1, 0));
  if (lane > 0) run = bw_compose(run, ex, H, hmask);
  for (uint32_t r = r0; r < r1; ++r) {
    const BwSum x = sums[(uint64_t)r * BW_SLOTS + slot];
    carry[(uint64_t)r * BW_SLOTS + slot] = run;
    run = bw_compose(run, x, H, hmask);
  }
}

// the (site, first position) list in ascending site order, as the sort path leaves it
__global__ void __launch_bounds__(BW_SLOTS) bw_sites_kernel(BwGlobal g, DevState* st) {
  __shared__ unsigned long long k[BW_SLOTS], c[BW_SLOTS];
  const int i = threadIdx.x;
  k[i] = g.keys[i];
  c[i] = g.counts[i];
  const int used = __syncthreads_count(k[i] != BW_EMPTY);
  if (k[i] == BW_EMPTY) return;
  uint32_t rank = 0;
  unsigned long long pos = 0;
  for (int j = 0; j < BW_SLOTS; ++j)
    if (k[j] != BW_EMPTY && k[j] < k[i]) { ++rank; pos += c[j]; }
  st->site_list[2 * rank] = k[i];
  st->site_list[2 * rank + 1] = pos;
  if (rank == 0) st->n_sites = (unsigned long long)used;
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
// per-chunk partial tables (H <= 16: at most 2 partitions) + the overflow table
static uint64_t partial_bytes(uint64_t n) { return ((uint64_t)n_chunks_for(n, 2) + 1) * (1ull << 16) * 8; }
static uint64_t branch_tmp_bytes(uint64_t n) { return ((8 * n + 15) & ~15ull) + partial_bytes(n); }

size_t branch_site_list_offset(uint64_t n) {
  return ((branch_tmp_bytes(n) + 15) & ~15ull) + ((radix_hist_bytes(n) + 15) & ~size_t(15));
}

static BwGeom bw_geometry(uint64_t n) {
  // tests force short tiles / ranges so carries cross every boundary
  static const uint32_t forced_tile = [] {
    const char* e = getenv("AIWC_BRANCH_TILE");
    return e ? (uint32_t)std::min<uint64_t>(BT_TILE, std::max<uint64_t>(1, strtoull(e, nullptr, 10))) : 0u;
  }();
  static const uint64_t forced_tiles = [] {
    const char* e = getenv("AIWC_BRANCH_RANGE");
    return e ? std::max<uint64_t>(1, strtoull(e, nullptr, 10)) : 0ull;
  }();
  BwGeom G;
  G.tile = forced_tile ? forced_tile : BT_TILE;
  const uint64_t tiles = std::max<uint64_t>(1, (n + G.tile - 1) / G.tile);
  const uint64_t per = forced_tiles ? forced_tiles : (tiles + BW_CTAS - 1) / BW_CTAS;
  G.len = per * G.tile;
  G.R = (uint32_t)std::max<uint64_t>(1, (n + G.len - 1) / G.len);
  return G;
}

static size_t bw_offset(uint64_t n) { return (branch_site_list_offset(n) + 2 * 8 * (n + 1) + 4095) & ~size_t(4095); }

struct BwLayout {
  BwGlobal g;
  BwSum *sums, *carry;
  unsigned long long* def;
  uint32_t* ndef;
  BwGeom geo;
};

static BwLayout bw_layout(void* scratch, uint64_t n) {
  BwLayout L;
  L.geo = bw_geometry(n);
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch) + bw_offset(n);
  L.g.keys = reinterpret_cast<unsigned long long*>(p);
  L.g.counts = L.g.keys + BW_SLOTS;
  L.g.n_sites = reinterpret_cast<unsigned int*>(L.g.counts + BW_SLOTS);
  L.sums = reinterpret_cast<BwSum*>(p + 4096);
  L.carry = L.sums + (size_t)L.geo.R * BW_SLOTS;
  L.def = reinterpret_cast<unsigned long long*>(L.carry + (size_t)L.geo.R * BW_SLOTS);
  L.ndef = reinterpret_cast<uint32_t*>(L.def + (size_t)L.geo.R * BW_DEF_CAP);
  return L;
}

size_t branch_scratch_bytes(uint64_t n) {
  const size_t R = bw_geometry(n).R;
  return bw_offset(n) + 4096 + R * (2 * BW_SLOTS * sizeof(BwSum) + BW_DEF_CAP * 8 + 4);
}

int branch_walk_prepare(const uint64_t* recs, uint64_t n, uint32_t history_len, DevState* st, void* scratch,
                        cudaStream_t s) {
  static const bool sort_only = [] { const char* e = getenv("AIWC_BRANCH_SORT"); return e && atoi(e) != 0; }();
  if (n == 0) return 0;
  if (sort_only || n >= (1ull << 32)) {  // codes are indexed by 32 bits
    cudaMemsetAsync(&st->bw_overflow, 1, 1, s);
    return 0;
  }
  const BwLayout L = bw_layout(scratch, n);
  cudaMemsetAsync(&st->bw_overflow, 0, sizeof(st->bw_overflow), s);
  cudaMemsetAsync(L.g.keys, 0xFF, BW_SLOTS * 8, s);
  cudaMemsetAsync(L.g.counts, 0, BW_SLOTS * 8 + 16, s);
  // codes in the first 4n bytes of the sort tmp region (free: the sort path runs only without a walk)
  bw_pass_kernel<<<L.geo.R, BT_T, sizeof(BwPassSmem), s>>>(recs, n, L.geo, history_len, L.g, L.sums, L.def, L.ndef,
                                                         reinterpret_cast<uint32_t*>(scratch), st);
  return 1;
}

int branch_stats(uint64_t* recs, uint64_t n, uint32_t site_bits, uint32_t history_len, bool walk, DevState* st,
                 unsigned long long* tables, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  (void)scratch_bytes;
  int kernels = 0;
  if (n == 0) return 0;
  uint8_t* base = reinterpret_cast<uint8_t*>(scratch);
  uint64_t* tmp = reinterpret_cast<uint64_t*>(base);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + ((branch_tmp_bytes(n) + 15) & ~15ull));
  unsigned long long* big = reinterpret_cast<unsigned long long*>(base + branch_site_list_offset(n));
  const uint32_t H = history_len, size = 1u << H;
  const uint32_t parts = n_parts_for(H), chunks = n_chunks_for(n, parts);
  unsigned long long* partials = reinterpret_cast<unsigned long long*>(base + ((8 * n + 15) & ~15ull));
  uint32_t* code;
  if (walk) {  // <= BW_MAX_SITES sites: no sort; bw_pass_kernel left the codes in the first 4n bytes of tmp
    const BwLayout L = bw_layout(scratch, n);
    code = reinterpret_cast<uint32_t*>(base);
    bw_scan_kernel<<<BW_SLOTS, BW_SCAN_T, 0, s>>>(L.sums, L.geo.R, H, L.g, L.carry, st);
    bw_fix_kernel<<<L.geo.R, 256, 0, s>>>(L.def, L.ndef, L.sums, L.carry, H, code, st);
    bw_sites_kernel<<<1, BW_SLOTS, 0, s>>>(L.g, st);
    kernels += 3;
  } else {
    // stable grouping by site; the result stays in whichever buffer the last digit wrote
    const uint64_t* sorted = site_bits ? radix_sort_u64_any(recs, tmp, n, 32, 32 + (int)site_bits, hist, s, &kernels)
                                       : recs;
    // the other 8n-byte buffer is free: observation codes + stage bytes
    uint8_t* free8n = sorted == tmp ? reinterpret_cast<uint8_t*>(recs) : base;
    code = reinterpret_cast<uint32_t*>(free8n);
    uint8_t* bits = free8n + 4 * ((n + 3) & ~3ull);
    const uint32_t sb = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 8);
    branch_stage_kernel<<<sb, 256, 0, s>>>(sorted, n, bits, st, big);
    const uint32_t wb = (uint32_t)std::min<uint64_t>((n + 256 * PC_PER - 1) / (256 * PC_PER), 148 * 8);
    pattern_walk_kernel<<<wb, 256, 0, s>>>(bits, n, H, code);
    kernels += 2;
  }
  const uint64_t chunk_len = ((n + chunks - 1) / chunks + PC_CHUNK_ALIGN - 1) / PC_CHUNK_ALIGN * PC_CHUNK_ALIGN;
  const size_t smem = (size_t)(size / parts) * sizeof(uint32_t);
  unsigned long long* ovf = partials + (uint64_t)chunks * size;
  cudaMemsetAsync(ovf, 0, (size_t)size * 8, s);
  set_smem_once(pattern_count_kernel, (int)smem);
  pattern_count_kernel<<<chunks * parts, PC_T, smem, s>>>(code, n, H, parts, chunk_len, partials, ovf);
  pattern_reduce_kernel<<<(size + 255) / 256, 256, 0, s>>>(partials, chunks, size, ovf, tables);
  // the per-chunk partial tables are consumed: their space holds the finish partials
  double* fin = reinterpret_cast<double*>(partials);
  const uint32_t fb = std::min<uint32_t>(BF_BLOCKS, (size + BF_T - 1) / BF_T);
  branch_partial_kernel<<<fb, BF_T, 0, s>>>(tables, size, fin);
  branch_finish_kernel<<<1, 32, 0, s>>>(fin, fb, st);
  return kernels + 4;
}

}  // namespace aiwc
