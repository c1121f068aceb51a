// aiwc_synth.cu -- deterministic synthetic traces for the BASELINE configs
// (SURVEY.md §8d), generated directly into HBM.  Every event is a pure function
// of (config, work-items, seed, event index), so any chunk can be produced
// independently and the numpy twin (paper_1805_04207_b200/synth.py) matches
// bit for bit.  Geometry follows the reference simulator: work-groups in
// order, work-items sequential inside a group until a barrier, 4-byte
// elements at 4096-aligned buffer bases (pkg/src/aiwc/sim.py:38-39,131-139,
// 242-350); a conditional branch emits `instr br` then `branch`, a barrier
// `instr barrier` then `barrier`.
//
//   1  sweep4   (C1) wi_begin, load, mem A+4gid, wi_end                       local 64
//   2  kmeans   (C2) 8x(load, mem A+4(8gid+k), fmul) 4x fadd.w4, store, mem B+4gid  local 256
//   3  mixed    (C3) 4 global-stream + 4 scratch + 2 gather loads, store, 8 compute local 256
//   4  branchy  (C4) 32 x (xor, load T[h&255], br crc-bit@10, br coin@12, add, br loop@14) local 256
//   5  barrier  (C5) 4 stages x (2 loads, 21 compute, store, barrier), resume, end   local 256
#include <algorithm>

#include "aiwc_internal.cuh"

namespace aiwc {

struct SynthGeo {
  uint64_t W, LV, per_group, groups;
  uint64_t A, B, C, D;  // buffer bases
  uint32_t n_opc;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(seed ^ mix64(a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull)));
}
__host__ __device__ inline uint64_t align4k(uint64_t x) { return (x + 4095) & ~4095ull; }

__host__ __device__ inline bool synth_geo(int cfg, uint64_t W, SynthGeo* g) {
  g->W = W;
  g->A = 4096;
  switch (cfg) {
    case 1: g->LV = 64; g->per_group = 2 + 64 * 4; g->n_opc = 1; break;
    case 2:
      g->LV = 256; g->per_group = 2 + 256 * 32; g->n_opc = 4;
      g->B = g->A + align4k(4 * 8 * W);
      break;
    case 3:
      g->LV = 256; g->per_group = 2 + 256 * 32; g->n_opc = 4;
      g->B = g->A + align4k(4 * 4 * W);      // scratch (1024 elements)
      g->C = g->B + 4096;                    // gather table: 4W elements (2^28 at 2^26 work-items)
      g->D = g->C + 16 * W;                  // store target
      break;
    case 4: g->LV = 256; g->per_group = 2 + 256 * 322; g->n_opc = 5; break;
    case 5:
      g->LV = 256; g->per_group = 2 + 256 * 122; g->n_opc = 6;
      g->B = g->A + align4k(4 * 2 * W);
      break;
    default: return false;
  }
  if (W == 0 || W % g->LV) return false;
  g->groups = W / g->LV;
  return true;
}

enum : uint32_t { OP_LOAD = 0, OP_STORE = 1, OP_FMUL = 2, OP_FADD = 3, OP_XOR = 2, OP_BR = 3, OP_ADD = 4,
                  OP_BARRIER = 2 };

__host__ __device__ inline uint64_t ins(uint32_t op, uint32_t w) { return ((uint64_t)op << 32) | w; }

// event of one work-item segment body; `pos` within the body
__host__ __device__ inline void wi_event(int cfg, const SynthGeo& g, uint64_t seed, uint64_t gid, uint64_t lid,
                                         uint64_t pos, uint32_t stage, uint8_t* k, uint64_t* p) {
  switch (cfg) {
    case 1:  // load, mem
      if (pos == 0) { *k = AIWC_K_INSTR; *p = ins(0, 1); }
      else { *k = AIWC_K_LOAD; *p = g.A + 4 * gid; }
      return;
    case 2: {
      if (pos < 24) {
        const uint64_t it = pos / 3, r = pos % 3;
        if (r == 0) { *k = AIWC_K_INSTR; *p = ins(OP_LOAD, 1); }
        else if (r == 1) { *k = AIWC_K_LOAD; *p = g.A + 4 * (8 * gid + it); }
        else { *k = AIWC_K_INSTR; *p = ins(OP_FMUL, 1); }
      } else if (pos < 28) { *k = AIWC_K_INSTR; *p = ins(OP_FADD, 4); }
      else if (pos == 28) { *k = AIWC_K_INSTR; *p = ins(OP_STORE, 1); }
      else { *k = AIWC_K_STORE; *p = g.B + 4 * gid; }
      return;
    }
    case 3: {
      if (pos < 20) {
        const uint64_t it = pos / 2;
        if ((pos & 1) == 0) { *k = AIWC_K_INSTR; *p = ins(OP_LOAD, 1); return; }
        *k = AIWC_K_LOAD;
        if (it < 4) *p = g.A + 4 * (4 * gid + it);
        else if (it < 8) *p = g.B + 4 * ((4 * lid + (it - 4)) & 1023);
        else *p = g.C + 4 * (hash3(seed, gid, it) % (4 * g.W));
      } else if (pos == 20) { *k = AIWC_K_INSTR; *p = ins(OP_STORE, 1); }
      else if (pos == 21) { *k = AIWC_K_STORE; *p = g.D + 4 * gid; }
      else { const uint64_t j = pos - 22; *k = AIWC_K_INSTR; *p = ins((j & 1) ? OP_FADD : OP_FMUL, (j & 2) ? 1 : 4); }
      return;
    }
    case 4: {
      const uint64_t it = pos / 10, r = pos % 10;
      const uint64_t h = hash3(seed, gid, it);
      switch (r) {
        case 0: *k = AIWC_K_INSTR; *p = ins(OP_XOR, 1); return;
        case 1: *k = AIWC_K_INSTR; *p = ins(OP_LOAD, 1); return;
        case 2: *k = AIWC_K_LOAD; *p = g.A + 4 * (h & 255); return;
        case 3: case 5: case 8: *k = AIWC_K_INSTR; *p = ins(OP_BR, 1); return;
        case 4: {  // CRC-16/0xA001 LFSR bit of the work-item's running state
          uint32_t crc = (uint32_t)((gid * 0x9E37u) ^ 0xFFFFu) & 0xFFFFu;
          uint32_t bit = 0;
          for (uint64_t s = 0; s <= it; ++s) {
            bit = crc & 1u;
            crc = (crc >> 1) ^ (bit ? 0xA001u : 0u);
          }
          *k = AIWC_K_BRANCH; *p = (10ull << 1) | bit; return;
        }
        case 6: *k = AIWC_K_BRANCH; *p = (12ull << 1) | ((h >> 40) & 1); return;
        case 7: *k = AIWC_K_INSTR; *p = ins(OP_ADD, 1); return;
        default: *k = AIWC_K_BRANCH; *p = (14ull << 1) | (it < 31 ? 1 : 0); return;
      }
    }
    case 5: {  // one stage (29 events): 2 x (load, mem), 21 compute, store, mem, barrier instr, barrier
      if (pos < 4) {
        if ((pos & 1) == 0) { *k = AIWC_K_INSTR; *p = ins(OP_LOAD, 1); }
        else { *k = AIWC_K_LOAD; *p = g.A + 4 * ((2 * gid + pos / 2 + 2 * stage) % (2 * g.W)); }
      } else if (pos < 25) {
        const uint64_t j = pos - 4;
        *k = AIWC_K_INSTR; *p = ins(3 + (uint32_t)(j % 3), 1u << (j % 3));
      } else if (pos == 25) { *k = AIWC_K_INSTR; *p = ins(OP_STORE, 1); }
      else if (pos == 26) { *k = AIWC_K_STORE; *p = g.B + 4 * (stage * g.W + gid); }
      else if (pos == 27) { *k = AIWC_K_INSTR; *p = ins(OP_BARRIER, 1); }
      else { *k = AIWC_K_BARRIER; *p = 0; }
      return;
    }
  }
}

__host__ __device__ inline void synth_event(int cfg, const SynthGeo& g, uint64_t seed, uint64_t i, uint8_t* k,
                                            uint64_t* p) {
  const uint64_t n = 2 + g.groups * g.per_group;
  if (i == 0) { *k = AIWC_K_KERNEL_BEGIN; *p = 0; return; }
  if (i == n - 1) { *k = AIWC_K_KERNEL_END; *p = 0; return; }
  const uint64_t grp = (i - 1) / g.per_group, r = (i - 1) % g.per_group;
  if (r == 0) { *k = AIWC_K_WG_BEGIN; *p = grp; return; }
  if (r == g.per_group - 1) { *k = AIWC_K_WG_END; *p = grp; return; }
  uint64_t q = r - 1;
  if (cfg != 5) {
    const uint64_t per_wi = (g.per_group - 2) / g.LV;
    const uint64_t lid = q / per_wi, pos = q % per_wi;
    const uint64_t gid = grp * g.LV + lid;
    if (pos == 0) { *k = AIWC_K_WI_BEGIN; *p = lid; return; }
    if (pos == per_wi - 1) { *k = AIWC_K_WI_END; *p = lid; return; }
    wi_event(cfg, g, seed, gid, lid, pos - 1, 0, k, p);
    return;
  }
  // C5: phases 0..3 = (open + 29-event stage) per work-item, phase 4 = (resume, end)
  const uint64_t ph_len = g.LV * 30;
  const uint64_t phase = q / ph_len;
  if (phase < 4) {
    const uint64_t rr = q % ph_len, lid = rr / 30, pos = rr % 30;
    const uint64_t gid = grp * g.LV + lid;
    if (pos == 0) { *k = phase == 0 ? AIWC_K_WI_BEGIN : AIWC_K_WI_RESUME; *p = lid; return; }
    wi_event(cfg, g, seed, gid, lid, pos - 1, (uint32_t)phase, k, p);
    return;
  }
  const uint64_t rr = q - 4 * ph_len, lid = rr / 2;
  *k = (rr & 1) ? AIWC_K_WI_END : AIWC_K_WI_RESUME;
  *p = lid;
}

__global__ void synth_kernel(int cfg, SynthGeo g, uint64_t seed, uint8_t* __restrict__ kind,
                             uint64_t* __restrict__ payload, uint64_t first, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t k;
    uint64_t p;
    synth_event(cfg, g, seed, first + i, &k, &p);
    kind[i] = k;
    payload[i] = p;
  }
}

}  // namespace aiwc

using namespace aiwc;

extern "C" uint64_t aiwc_synth_size(int cfg, uint64_t W, aiwc_trace_info* info) {
  SynthGeo g{};
  if (!synth_geo(cfg, W, &g)) return 0;
  const uint64_t n = 2 + g.groups * g.per_group;
  if (info) {
    *info = aiwc_trace_info{};
    info->n_events = n;
    info->local_volume = (uint32_t)g.LV;
    info->n_opcodes = g.n_opc;
    info->has_addr_stats = 1;
    info->addr_min = g.A;
    info->addr_and = 0;            // every address is 4-byte aligned: bits 0..1 constant 0
    info->addr_or = ~3ull;
    switch (cfg) {
      case 1: info->addr_max = g.A + 4 * (W - 1); break;
      case 2: info->addr_max = g.B + 4 * (W - 1); break;
      case 3: info->addr_max = g.D + 4 * (W - 1); break;
      case 4: info->addr_max = g.A + 4 * 255; break;
      case 5: info->addr_max = g.B + 4 * (4 * W - 1); break;
    }
    // class totals per work-item of each recipe (wi_event above)
    static const uint64_t per_wi[6][4] = {{0, 0, 0, 0}, {1, 1, 0, 0}, {21, 8, 1, 0}, {19, 10, 1, 0},
                                          {192, 32, 0, 96}, {100, 8, 4, 0}};
    info->has_counts = 1;
    info->n_instr = per_wi[cfg][0] * W; info->n_reads = per_wi[cfg][1] * W;
    info->n_writes = per_wi[cfg][2] * W; info->n_branches = per_wi[cfg][3] * W;
    info->n_groups = g.groups;
    info->any_barrier_or_resume = cfg == 5;
  }
  return n;
}

extern "C" int aiwc_synth_fill(int cfg, uint64_t W, uint64_t seed, uint8_t* kind, uint64_t* payload, uint64_t first,
                               uint64_t n, void* stream) {
  SynthGeo g{};
  if (!synth_geo(cfg, W, &g)) return AIWC_ERR_ARGUMENT;
  if (n == 0) return AIWC_OK;
  const uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  synth_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cfg, g, seed, kind, payload, first, n);
  return cudaGetLastError() == cudaSuccess ? AIWC_OK : AIWC_ERR_CUDA;
}
