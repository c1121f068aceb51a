// aiwc_sim.cu -- the .aiwck NDRange producer on the device (sim.py:171-372).
//
// The reference runs work-groups one after another and, inside a group, one
// work-item at a time until its next barrier or return, every store visible to
// every later load (sim.py:242-280).  The event stream is therefore a pure
// function of the program and the launch, and so is each (group, barrier
// round, local id) *segment* of it.  Here:
//
//  * speculative mode: each work-item is interpreted by its own thread against
//    the launch's initial buffers plus a private log of its own stores.  That
//    is exact unless a work-item loads an element a *different* work-item
//    stored earlier in the reference's order.  Pass COUNT records per buffer
//    element the earliest (group, round, local id) store key and whether one
//    or several work-items stored it; pass VERIFY re-runs every load against
//    those tables.  A dependence (or a full store log) switches the launch to
//  * group mode: one thread per work-group executing the reference's schedule
//    for that group literally (real stores, barrier rounds in local order),
//    groups in parallel.  Exact unless two groups touch an element one of them
//    stores -- recorded per element during the pass -- which switches to
//  * sequential mode: one thread executing the whole launch literally.
//
// Either way COUNT leaves per-segment event / instruction counts; a scan lays
// the segments out in the reference's order and pass EMIT writes each event
// straight into its final column slot.  Faults are resolved exactly as the
// reference raises them: the earliest faulting segment, the first divergent
// group's barrier round, or the (limit+1)-th instruction charge, whichever the
// reference's schedule reaches first.
#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "aiwc_util.cuh"

namespace {

using u64 = unsigned long long;

constexpr int SIMW = AIWC_SIM_WORDS;
enum : int32_t { K_COMPUTE = 0, K_LOAD, K_STORE, K_BR, K_JMP, K_BARRIER, K_RET };
enum : int { MODE_COUNT = 0, MODE_VERIFY = 1, MODE_EMIT = 2, MODE_DETAIL = 3 };
enum : int { END_BARRIER = 0, END_RET = 1, END_ERROR = 2, END_CAP = 3 };
enum : uint32_t { SF_LOG = 1, SF_KEY = 2, SF_PHASES = 4, SF_CONFLICT = 8 };
enum : int { MEM_SPEC = 0, MEM_SEQ = 1, MEM_GROUP = 2 };
enum : int { STOP_NONE = 0, STOP_FAULT = 1, STOP_CAP = 2, STOP_DIV = 3 };
constexpr uint32_t FIN_NEVER = 0xFFFFFFFFu;
constexpr uint32_t OWN_EMPTY = 0xFFFFFFFFu, OWN_MULTI = 0xFFFFFFFEu;
constexpr uint32_t LOGCAP = 32;
constexpr int SPEC_TPB = 128;

struct Fault {
  int32_t code, line;
  uint32_t reg, lanes, width, buf;
  long long index;
};

struct SimGlobals {
  u64 err_key;         // earliest faulting segment key (speculative COUNT)
  u64 charges;         // sequential mode: instruction charges so far
  u64 tot[5];          // instructions, reads, writes, branches, barriers
  u64 ord;             // ordinal-sum result
  uint32_t flags, max_nph;
  uint32_t div_group;  // first divergent group (stream order) or ~0
  uint32_t culprit, waiting, pad0;
  Fault f;             // detail run / sequential mode
  int32_t last_br;     // detail work-item's last branch line at its end
  uint32_t s_stop;     // sequential: 0 ran to the end, 1 fault, 2 step limit, 3 divergence
  uint32_t s_group, s_round, s_wi, s_phase;
};

struct SimArgs {
  const int32_t* code;
  const u64* imm;
  uint32_t n_regs, wmax;
  const u64* bbase;  // per buffer: byte address
  const u64* blen;   // elements
  const u64* boff;   // element offset into mem
  u64* mem;          // speculative: the initial values (read only); sequential: working copy
  u64 gsz[3], lsz[3], ngrp[3];
  u64 V, G, n_wi;
  u64 cap;           // speculative: charges one work-item may make (limit + 1); sequential: limit
  // register file: value (r, lane) of slot s at regs[(r * wmax + lane) * stride + s]
  u64* regs;
  uint32_t* rlen;
  u64 stride;
  u64 *log_e, *log_v;  // own-store log, entry i of slot s at [i * stride + s]
  u64* smin;
  uint32_t* sown;      // speculative: storing work-item / group mode: storing group (or MULTI)
  uint32_t* sacc;      // group mode: accessing group (or MULTI)
  int kb_l, kb_p;      // key = g << (kb_p + kb_l) | p << kb_l | l
  uint32_t pmax;       // largest phase the key holds
  uint32_t* nph;       // per work-item: segments opened
  uint8_t* wend;       // per work-item: END_* of the last segment
  uint32_t *segcnt, *seginstr;
  uint32_t pcap;       // [w * pcap + p]
  uint32_t *gnph, *gfin_min, *gfin_max;
  SimGlobals* gl;
  uint8_t* okind;
  u64* opay;
  const u64* segpos;   // exclusive scan of segment lengths (S + 1 entries)
  const u64* gseg;     // per group: first segment index (G + 1 entries)
  // group / sequential mode: per-work-item state of the groups in flight, [slot * V + l]
  uint32_t* s_pc;
  int32_t* s_br;
  uint8_t* s_status;
};

struct Totals {
  u64 instr = 0, rd = 0, wr = 0, br = 0, bar = 0;
};

__device__ __forceinline__ u64 mk_key(const SimArgs& a, u64 g, u64 p, u64 l) {
  return (g << (a.kb_p + a.kb_l)) | (p << a.kb_l) | l;
}

__device__ __forceinline__ void builtins_of(const SimArgs& a, u64 g, u64 l, u64 (&bi)[15], uint32_t& lin_l,
                                            u64& gkey) {
  // stream order is lexicographic (dimension 0 slowest); keys / linear local ids
  // are dimension-0-fastest (trace.py group_of_key / local_of_id)
  const u64 g2 = g % a.ngrp[2], g1 = (g / a.ngrp[2]) % a.ngrp[1], g0 = g / (a.ngrp[2] * a.ngrp[1]);
  const u64 l2 = l % a.lsz[2], l1 = (l / a.lsz[2]) % a.lsz[1], l0 = l / (a.lsz[2] * a.lsz[1]);
  const u64 grp[3] = {g0, g1, g2}, lid[3] = {l0, l1, l2};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    bi[d] = grp[d] * a.lsz[d] + lid[d];
    bi[3 + d] = lid[d];
    bi[6 + d] = grp[d];
    bi[9 + d] = a.gsz[d];
    bi[12 + d] = a.lsz[d];
  }
  lin_l = (uint32_t)(l0 + a.lsz[0] * (l1 + a.lsz[1] * l2));
  gkey = g0 + a.ngrp[0] * (g1 + a.ngrp[1] * g2);
}

__device__ __forceinline__ u64 py_div(long long x, long long y) {
  if (y == 0) return 0;
  if (x == LLONG_MIN && y == -1) return (u64)LLONG_MIN;
  long long q = x / y;
  if ((x % y != 0) && ((x < 0) != (y < 0))) --q;
  return (u64)q;
}

__device__ __forceinline__ u64 py_mod(long long x, long long y) {
  if (y == 0 || y == -1) return 0;
  long long r = x % y;
  if (r != 0 && ((r < 0) != (y < 0))) r += y;
  return (u64)r;
}

// SEMANTICS (sim.py:56-83), values mod 2^64, signed where the reference uses _s
__device__ __forceinline__ u64 sem_eval(int sem, u64 x, u64 y, u64 z) {
  const long long sx = (long long)x, sy = (long long)y;
  switch (sem) {
    case 0: return x;
    case 1: return ~x;
    case 2: return 0ull - x;
    case 3: return sx < 0 ? 0ull - x : x;
    case 4: return x + y;
    case 5: return x - y;
    case 6: return x * y;
    case 7: return py_div(sx, sy);
    case 8:
    case 9: return py_mod(sx, sy);
    case 10: return x & y;
    case 11: return x | y;
    case 12: return x ^ y;
    case 13: return x << (y & 63);
    case 14: return x >> (y & 63);
    case 15: return sx < sy ? x : y;
    case 16: return sx > sy ? x : y;
    case 17: return x == y;
    case 18: return x != y;
    case 19: return sx < sy;
    case 20: return sx <= sy;
    case 21: return sx > sy;
    case 22: return sx >= sy;
    case 23: return x * y + z;
    default: return x != 0 ? y : z;  // select
  }
}

__device__ __forceinline__ int arity(int sem) { return sem <= 3 ? 1 : (sem >= 23 ? 3 : 2); }

template <int MODE, int MEM>
struct Machine {
  const SimArgs& a;
  u64 slot, w, grp;
  const u64 (&bi)[15];
  uint32_t nlog = 0;

  __device__ Machine(const SimArgs& a_, u64 slot_, u64 w_, u64 g_, const u64 (&bi_)[15])
      : a(a_), slot(slot_), w(w_), grp(g_), bi(bi_) {}

  __device__ __forceinline__ u64& reg(uint32_t r, uint32_t lane) const {
    return a.regs[((u64)r * a.wmax + lane) * a.stride + slot];
  }
  __device__ __forceinline__ uint32_t& rl(uint32_t r) const { return a.rlen[(u64)r * a.stride + slot]; }

  // group mode, pass COUNT: which groups touch / store an element
  __device__ __forceinline__ void mark(uint32_t* tab, u64 e) const {
    const uint32_t g = (uint32_t)grp, old = atomicCAS(&tab[e], OWN_EMPTY, g);
    if (old != OWN_EMPTY && old != g && old != OWN_MULTI) atomicExch(&tab[e], OWN_MULTI);
  }

  __device__ __forceinline__ u64 load_elem(u64 e) const {
    if (MEM == MEM_SPEC) {
      for (uint32_t i = 0; i < nlog; ++i)
        if (a.log_e[(u64)i * a.stride + slot] == e) return a.log_v[(u64)i * a.stride + slot];
    }
    if (MEM == MEM_GROUP && MODE == MODE_COUNT) mark(a.sacc, e);
    return a.mem[e];
  }
  __device__ __forceinline__ void store_elem(u64 e, u64 v, u64 key) {
    if (MEM != MEM_SPEC) {
      if (MEM == MEM_GROUP && MODE == MODE_COUNT) {
        mark(a.sown, e);
        mark(a.sacc, e);
      }
      a.mem[e] = v;
      return;
    }
    if (MODE == MODE_COUNT) {
      atomicMin(&a.smin[e], key);
      const uint32_t old = atomicCAS(&a.sown[e], OWN_EMPTY, (uint32_t)w);
      if (old != OWN_EMPTY && old != (uint32_t)w && old != OWN_MULTI) atomicExch(&a.sown[e], OWN_MULTI);
    }
    for (uint32_t i = 0; i < nlog; ++i)
      if (a.log_e[(u64)i * a.stride + slot] == e) {
        a.log_v[(u64)i * a.stride + slot] = v;
        return;
      }
    if (nlog < LOGCAP) {
      a.log_e[(u64)nlog * a.stride + slot] = e;
      a.log_v[(u64)nlog * a.stride + slot] = v;
      ++nlog;
    } else {
      atomicOr(&a.gl->flags, SF_LOG);
    }
  }

  __device__ __forceinline__ void emit(u64& pos, uint8_t k, u64 p) const {
    if (MODE == MODE_EMIT) {
      a.okind[pos] = k;
      a.opay[pos] = p;
    }
    ++pos;
  }

  // one segment: until barrier / ret / fault / charge cap (sim.py:282-344)
  __device__ int segment(u64 key, uint32_t& pc, u64& charges, int32_t& last_br, u64& pos, uint32_t& ninstr,
                         Totals& t, Fault* fault) {
    for (;;) {
      const int4* rec = reinterpret_cast<const int4*>(a.code + (size_t)pc * SIMW);
      const int4 q0 = __ldg(rec), q1 = __ldg(rec + 1), q2 = __ldg(rec + 2);
      const int kind = q0.x;
      if (kind == K_RET) return END_RET;
      if (charges >= a.cap) return END_CAP;
      ++charges;
      ++ninstr;
      ++t.instr;
      const uint32_t width = (uint32_t)q0.z;
      const int32_t line = q2.w;
      emit(pos, AIWC_K_INSTR, ((u64)(uint32_t)q2.z << 32) | width);
      auto fail = [&](int code, uint32_t reg, uint32_t lanes, long long index) {
        if (fault) *fault = Fault{code, line, reg, lanes, width, (uint32_t)q1.w, index};
        return END_ERROR;
      };
      // scalar operand (sim.py:225-231): a never-written register is a TypeError
      auto scalar = [&](uint32_t spec, bool& ok) -> u64 {
        const uint32_t mode = spec >> 30, idx = spec & 0x3FFFFFFFu;
        ok = true;
        if (mode == 1) return __ldg(a.imm + idx);
        if (mode == 2) return bi[idx];
        if (rl(idx) == 0) {
          ok = false;
          return 0;
        }
        return reg(idx, 0);
      };
      switch (kind) {
        case K_COMPUTE: {
          const int sem = q0.y, n = arity(sem);
          const uint32_t src[3] = {(uint32_t)q1.x, (uint32_t)q1.y, (uint32_t)q1.z};
          bool vec[3] = {false, false, false};
          u64 sv[3] = {0, 0, 0};
          for (int i = 0; i < n; ++i) {  // _lanes checks, in operand order (sim.py:205-223)
            const uint32_t mode = src[i] >> 30, idx = src[i] & 0x3FFFFFFFu;
            if (mode == 0) {
              const uint32_t len = rl(idx);
              if (len == 0) return fail(AIWC_SIM_NONE_LEN, idx, 0, 0);
              if (len != width && len != 1) return fail(AIWC_SIM_WIDTH, idx, len, 0);
              vec[i] = len != 1;
              sv[i] = reg(idx, 0);
            } else {
              sv[i] = mode == 1 ? __ldg(a.imm + idx) : bi[idx];
            }
          }
          if (width > AIWC_SIM_MAX_WIDTH) return fail(AIWC_SIM_UNSUPPORTED, 0, 0, 0);
          const uint32_t d = (uint32_t)q0.w;
          for (uint32_t lane = 0; lane < width; ++lane) {
            const u64 x = vec[0] ? reg(src[0] & 0x3FFFFFFFu, lane) : sv[0];
            const u64 y = vec[1] ? reg(src[1] & 0x3FFFFFFFu, lane) : sv[1];
            const u64 z = vec[2] ? reg(src[2] & 0x3FFFFFFFu, lane) : sv[2];
            reg(d, lane) = sem_eval(sem, x, y, z);
          }
          rl(d) = width;
          ++pc;
          break;
        }
        case K_LOAD:
        case K_STORE: {
          const uint32_t b = (uint32_t)q1.w;
          bool ok;
          const long long idx = (long long)scalar((uint32_t)q1.x, ok);
          if (!ok) return fail(AIWC_SIM_NONE_INDEX, q1.x & 0x3FFFFFFF, 0, 0);
          const u64 len = __ldg(a.blen + b);
          if (idx < 0 || (u64)idx + width > len) return fail(AIWC_SIM_OUT_OF_BOUNDS, 0, 0, idx);
          const u64 e0 = __ldg(a.boff + b) + (u64)idx, addr0 = __ldg(a.bbase + b) + 4ull * (u64)idx;
          const bool atomic = q0.y != 0;
          if (kind == K_LOAD) {
            if (width > AIWC_SIM_MAX_WIDTH) return fail(AIWC_SIM_UNSUPPORTED, 0, 0, 0);
            const uint32_t d = (uint32_t)q0.w;
            for (uint32_t lane = 0; lane < width; ++lane) {
              const u64 e = e0 + lane;
              if (MEM == MEM_SPEC && MODE == MODE_VERIFY) {
                const uint32_t own = a.sown[e];
                if (own != OWN_EMPTY && own != (uint32_t)w && a.smin[e] < key) atomicOr(&a.gl->flags, SF_CONFLICT);
              }
              const u64 v = load_elem(e);
              emit(pos, atomic ? AIWC_K_ATOMIC_LOAD : AIWC_K_LOAD, addr0 + 4ull * lane);
              reg(d, lane) = v;
            }
            rl(d) = width;
            t.rd += width;
          } else {
            const uint32_t sspec = (uint32_t)q1.y, smode = sspec >> 30, sidx = sspec & 0x3FFFFFFFu;
            bool vec = false;
            u64 sval = 0;
            if (smode == 0) {
              const uint32_t l = rl(sidx);
              if (l == 0) return fail(AIWC_SIM_NONE_LEN, sidx, 0, 0);
              if (l != width && l != 1) return fail(AIWC_SIM_WIDTH, sidx, l, 0);
              vec = l != 1;
              sval = reg(sidx, 0);
            } else {
              sval = smode == 1 ? __ldg(a.imm + sidx) : bi[sidx];
            }
            for (uint32_t lane = 0; lane < width; ++lane) {
              emit(pos, atomic ? AIWC_K_ATOMIC_STORE : AIWC_K_STORE, addr0 + 4ull * lane);
              store_elem(e0 + lane, vec ? reg(sidx, lane) : sval, key);
            }
            t.wr += width;
          }
          ++pc;
          break;
        }
        case K_BR: {
          bool ok;
          const u64 c = scalar((uint32_t)q1.x, ok);
          if (!ok) return fail(AIWC_SIM_NONE_INDEX, q1.x & 0x3FFFFFFF, 0, 0);
          const bool taken = c != 0;
          emit(pos, AIWC_K_BRANCH, ((u64)(uint32_t)line << 1) | (taken ? 1u : 0u));
          ++t.br;
          last_br = line;
          pc = (uint32_t)(taken ? q2.x : q2.y);
          break;
        }
        case K_JMP:
          pc = (uint32_t)q2.x;
          break;
        default:  // K_BARRIER: `instr barrier` inside the segment, the barrier event closes it
          ++pc;
          ++t.bar;
          return END_BARRIER;
      }
    }
  }
};

__device__ __forceinline__ void add_totals(const SimArgs& a, const Totals& t) {  // one thread
  const u64 v[5] = {t.instr, t.rd, t.wr, t.br, t.bar};
  for (int i = 0; i < 5; ++i) a.gl->tot[i] += v[i];
}

__device__ __forceinline__ void flush_totals(const SimArgs& a, Totals& t) {  // whole warps
  u64 v[5] = {t.instr, t.rd, t.wr, t.br, t.bar};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    u64 x = v[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&a.gl->tot[i], x);
  }
}

__device__ __forceinline__ void record_segment(const SimArgs& a, u64 w, uint32_t p, uint32_t cnt, uint32_t ni) {
  if (p < a.pcap) {
    a.segcnt[w * a.pcap + p] = cnt;
    a.seginstr[w * a.pcap + p] = ni;
  }
}

// ---- speculative mode: one thread per work-item, all its barrier rounds ----
template <int MODE>
__global__ void __launch_bounds__(SPEC_TPB) sim_spec_kernel(SimArgs a) {
  const u64 slot = (u64)blockIdx.x * blockDim.x + threadIdx.x, T = (u64)gridDim.x * blockDim.x;
  Totals tot;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < a.n_wi; base += T) {
    const u64 w = base + threadIdx.x;
    if (w < a.n_wi) {
      const u64 g = w / a.V, l = w % a.V;
      u64 bi[15];
      uint32_t lin_l;
      u64 gkey;
      builtins_of(a, g, l, bi, lin_l, gkey);
      for (uint32_t r = 0; r < a.n_regs; ++r) a.rlen[(u64)r * a.stride + slot] = 0;
      Machine<MODE, MEM_SPEC> m(a, slot, w, g, bi);
      uint32_t pc = 0, p = 0;
      u64 charges = 0;
      int32_t last_br = -1;
      int end;
      for (;; ++p) {
        if (p > a.pmax) atomicOr(&a.gl->flags, SF_KEY);
        const u64 key = mk_key(a, g, p, l);
        u64 pos = 0;
        if (MODE == MODE_EMIT) {
          const u64 open = 2 + 2 * g + a.segpos[a.gseg[g] + (u64)p * a.V + l];
          a.okind[open] = p ? AIWC_K_WI_RESUME : AIWC_K_WI_BEGIN;
          a.opay[open] = lin_l;
          pos = open + 1;
        }
        const u64 pos0 = pos;
        uint32_t ni = 0;
        end = m.segment(key, pc, charges, last_br, pos, ni, tot, nullptr);
        if (MODE == MODE_COUNT) record_segment(a, w, p, (uint32_t)(pos - pos0), ni);
        if (MODE == MODE_EMIT && (end == END_BARRIER || end == END_RET)) {
          a.okind[pos] = end == END_BARRIER ? AIWC_K_BARRIER : AIWC_K_WI_END;
          a.opay[pos] = end == END_BARRIER ? 0ull : lin_l;
        }
        if (end != END_BARRIER) break;
      }
      if (MODE == MODE_COUNT) {
        a.nph[w] = p + 1;
        a.wend[w] = (uint8_t)end;
        const uint32_t fin = (end == END_RET || end == END_ERROR) ? p : FIN_NEVER;
        atomicMax(&a.gnph[g], p + 1);
        atomicMin(&a.gfin_min[g], fin);
        atomicMax(&a.gfin_max[g], fin);
        atomicMax(&a.gl->max_nph, p + 1);
        if (end == END_ERROR) atomicMin(&a.gl->err_key, mk_key(a, g, p, l));
      }
      if (MODE == MODE_EMIT && l == 0) {
        a.okind[1 + 2 * g + a.segpos[a.gseg[g]]] = AIWC_K_WG_BEGIN;
        a.opay[1 + 2 * g + a.segpos[a.gseg[g]]] = gkey;
        a.okind[2 + 2 * g + a.segpos[a.gseg[g + 1]]] = AIWC_K_WG_END;
        a.opay[2 + 2 * g + a.segpos[a.gseg[g + 1]]] = gkey;
      }
    }
  }
  if (MODE == MODE_COUNT) flush_totals(a, tot);
}

// one work-item again (speculative mode), recording its fault and its last branch line
__global__ void sim_detail_kernel(SimArgs a, u64 w) {
  if (threadIdx.x || blockIdx.x) return;
  const u64 g = w / a.V, l = w % a.V;
  u64 bi[15];
  uint32_t lin_l;
  u64 gkey;
  builtins_of(a, g, l, bi, lin_l, gkey);
  for (uint32_t r = 0; r < a.n_regs; ++r) a.rlen[(u64)r * a.stride] = 0;
  Machine<MODE_DETAIL, MEM_SPEC> m(a, 0, w, g, bi);
  uint32_t pc = 0;
  u64 charges = 0, pos = 0;
  int32_t last_br = -1;
  Totals t;
  Fault f{0, -1, 0, 0, 0, 0, 0};
  for (uint32_t p = 0;; ++p) {
    uint32_t ni = 0;
    const int end = m.segment(mk_key(a, g, p, l), pc, charges, last_br, pos, ni, t, &f);
    if (end != END_BARRIER) break;
  }
  a.gl->f = f;
  a.gl->last_br = last_br;
}

struct GroupStop {
  int stop;
  uint32_t round, l;          // fault / cap: round and local id; divergence: round
  uint32_t culprit, waiting;  // divergence: local ids
  int32_t last_br;            // divergence: culprit's last branch
  Fault f;
};

// one work-group in the reference's schedule (sim.py:242-280): barrier rounds,
// work-items in local order until their next barrier / return.  `sb` is the
// first per-work-item state slot; the memory is written through.
template <int MODE, int MEM>
__device__ void run_group(const SimArgs& a, u64 g, u64 sb, u64& charges, Totals& tot, GroupStop& gs) {
  enum : uint8_t { READY = 0, AT_BARRIER = 1, DONE = 2 };
  gs.stop = STOP_NONE;
  for (u64 l = 0; l < a.V; ++l) {
    a.s_pc[sb + l] = 0;
    a.s_br[sb + l] = -1;
    a.s_status[sb + l] = READY;
    for (uint32_t r = 0; r < a.n_regs; ++r) a.rlen[(u64)r * a.stride + sb + l] = 0;
    if (MODE == MODE_COUNT) a.nph[g * a.V + l] = 0;
  }
  u64 gkey = 0;
  {
    u64 bi0[15];
    uint32_t l0;
    builtins_of(a, g, 0, bi0, l0, gkey);
  }
  if (MODE == MODE_EMIT) {
    a.okind[1 + 2 * g + a.segpos[a.gseg[g]]] = AIWC_K_WG_BEGIN;
    a.opay[1 + 2 * g + a.segpos[a.gseg[g]]] = gkey;
  }
  for (uint32_t p = 0;; ++p) {
    bool any_done = false, all_done = true;
    for (u64 l = 0; l < a.V; ++l) {
      if (a.s_status[sb + l] != READY) {
        all_done &= a.s_status[sb + l] == DONE;
        continue;
      }
      const u64 w = g * a.V + l;
      u64 bi[15];
      uint32_t lin_l;
      builtins_of(a, g, l, bi, lin_l, gkey);
      Machine<MODE, MEM> m(a, sb + l, w, g, bi);
      u64 pos = 0;
      if (MODE == MODE_EMIT) {
        const u64 open = 2 + 2 * g + a.segpos[a.gseg[g] + (u64)p * a.V + l];
        a.okind[open] = p ? AIWC_K_WI_RESUME : AIWC_K_WI_BEGIN;
        a.opay[open] = lin_l;
        pos = open + 1;
      }
      const u64 pos0 = pos;
      uint32_t ni = 0, pc = a.s_pc[sb + l];
      int32_t last_br = a.s_br[sb + l];
      const int end = m.segment(mk_key(a, g, p, l), pc, charges, last_br, pos, ni, tot, &gs.f);
      a.s_pc[sb + l] = pc;
      a.s_br[sb + l] = last_br;
      if (MODE == MODE_COUNT) {
        record_segment(a, w, p, (uint32_t)(pos - pos0), ni);
        a.nph[w] = p + 1;
        a.wend[w] = (uint8_t)end;
        a.gnph[g] = max(a.gnph[g], p + 1);
        atomicMax(&a.gl->max_nph, p + 1);
      }
      if (MODE == MODE_EMIT && (end == END_BARRIER || end == END_RET)) {
        a.okind[pos] = end == END_BARRIER ? AIWC_K_BARRIER : AIWC_K_WI_END;
        a.opay[pos] = end == END_BARRIER ? 0ull : lin_l;
      }
      if (end == END_ERROR || end == END_CAP) {
        gs.stop = end == END_ERROR ? STOP_FAULT : STOP_CAP;
        gs.round = p;
        gs.l = (uint32_t)l;
        return;
      }
      if (end == END_RET) {
        a.s_status[sb + l] = DONE;
        any_done = true;
      } else {
        a.s_status[sb + l] = AT_BARRIER;
        all_done = false;
      }
    }
    if (all_done) break;
    if (any_done) {  // sim.py:262-275: first finished work-item, first one waiting
      u64 c = 0, wt = 0;
      while (a.s_status[sb + c] != DONE) ++c;
      while (a.s_status[sb + wt] != AT_BARRIER) ++wt;
      gs.stop = STOP_DIV;
      gs.round = p;
      gs.culprit = (uint32_t)c;
      gs.waiting = (uint32_t)wt;
      gs.last_br = a.s_br[sb + c];
      return;
    }
    for (u64 l = 0; l < a.V; ++l) a.s_status[sb + l] = READY;
  }
  if (MODE == MODE_EMIT) {
    a.okind[2 + 2 * g + a.segpos[a.gseg[g + 1]]] = AIWC_K_WG_END;
    a.opay[2 + 2 * g + a.segpos[a.gseg[g + 1]]] = gkey;
  }
}

// ---- group mode: one thread per work-group, groups in parallel ----
// g_only != ~0: run that group alone and record its stop in the globals (detail run)
template <int MODE>
__global__ void sim_group_kernel(SimArgs a, u64 g_only) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x, T = (u64)gridDim.x * blockDim.x;
  Totals tot;
  const u64 g0 = g_only != ~0ull ? (t == 0 ? g_only : a.G) : t;
  const u64 step = g_only != ~0ull ? a.G : T;
  for (u64 g = g0; g < a.G; g += step) {
    u64 charges = 0;
    GroupStop gs;
    gs.f = Fault{0, -1, 0, 0, 0, 0, 0};
    run_group<MODE, MEM_GROUP>(a, g, t * a.V, charges, tot, gs);
    if (MODE == MODE_COUNT) {
      const uint32_t r = gs.stop == STOP_DIV ? gs.round : 0;
      a.gfin_min[g] = r;
      a.gfin_max[g] = gs.stop == STOP_DIV ? r + 1 : r;
      if (gs.stop == STOP_FAULT) atomicMin(&a.gl->err_key, mk_key(a, g, gs.round, gs.l));
    }
    if (MODE == MODE_DETAIL) {
      a.gl->f = gs.f;
      a.gl->culprit = (uint32_t)(g * a.V + gs.culprit);
      a.gl->waiting = (uint32_t)(g * a.V + gs.waiting);
      a.gl->last_br = gs.last_br;
    }
  }
  if (MODE == MODE_COUNT) flush_totals(a, tot);
}

// ---- sequential mode: the whole launch in the reference's schedule, one thread ----
template <int MODE>
__global__ void sim_seq_kernel(SimArgs a) {
  if (threadIdx.x || blockIdx.x) return;
  Totals tot;
  u64 charges = 0;  // launch-wide: the (limit+1)-th charge is the step-limit fault itself
  for (u64 g = 0; g < a.G; ++g) {
    GroupStop gs;
    gs.f = Fault{0, -1, 0, 0, 0, 0, 0};
    run_group<MODE, MEM_SEQ>(a, g, 0, charges, tot, gs);
    if (gs.stop != STOP_NONE) {
      if (MODE == MODE_COUNT) {
        SimGlobals* gl = a.gl;
        gl->s_stop = gs.stop;
        gl->f = gs.f;
        gl->s_group = (uint32_t)g;
        gl->s_round = gs.round;
        gl->s_wi = (uint32_t)(g * a.V + gs.l);
        gl->culprit = (uint32_t)(g * a.V + gs.culprit);
        gl->waiting = (uint32_t)(g * a.V + gs.waiting);
        gl->last_br = gs.last_br;
        add_totals(a, tot);
      }
      return;
    }
  }
  if (MODE == MODE_COUNT) add_totals(a, tot);
}

// ---- layout and fault resolution helpers ----
__global__ void sim_init_kernel(SimArgs a, u64 n_elem, int mode) {
  const u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  if (mode != MEM_SEQ)
    for (u64 i = i0; i < n_elem; i += st) {
      if (mode == MEM_SPEC) a.smin[i] = ~0ull;
      else a.sacc[i] = OWN_EMPTY;
      a.sown[i] = OWN_EMPTY;
    }
  for (u64 g = i0; g < a.G; g += st) {
    a.gnph[g] = 0;
    a.gfin_min[g] = FIN_NEVER;
    a.gfin_max[g] = 0;
  }
  if (i0 == 0) {
    unsigned char* z = reinterpret_cast<unsigned char*>(a.gl);
    for (size_t i = 0; i < sizeof(SimGlobals); ++i) z[i] = 0;
    a.gl->err_key = ~0ull;
    a.gl->div_group = ~0u;
    a.gl->culprit = ~0u;
    a.gl->waiting = ~0u;
    a.gl->last_br = -1;
    a.gl->f.line = -1;
  }
}

// group mode: an element stored by one group and touched by another
__global__ void sim_group_check_kernel(SimArgs a, u64 n_elem) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n_elem; i += (u64)gridDim.x * blockDim.x)
    if (a.sown[i] != OWN_EMPTY && a.sacc[i] == OWN_MULTI) {
      atomicOr(&a.gl->flags, SF_CONFLICT);
      return;
    }
}

__global__ void sim_group_seg_kernel(SimArgs a, u64* gseg) {
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < a.G; g += (u64)gridDim.x * blockDim.x)
    gseg[g] = (u64)a.gnph[g] * a.V;
}

__global__ void sim_segv_kernel(SimArgs a, u64* segv) {
  for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < a.n_wi; w += (u64)gridDim.x * blockDim.x) {
    const u64 g = w / a.V, l = w % a.V;
    const uint32_t np = a.nph[w], gp = a.gnph[g];
    for (uint32_t p = 0; p < gp; ++p) {
      u64 len = 0;
      if (p < np) {
        const bool closed = p + 1 < np || a.wend[w] == END_RET || a.wend[w] == END_BARRIER;
        len = 1 + (u64)a.segcnt[w * a.pcap + p] + (closed ? 1 : 0);
      }
      segv[a.gseg[g] + (u64)p * a.V + l] = len;
    }
  }
}

// instructions charged in segments before (G, P, L) in the reference's order
__global__ void sim_ordinal_kernel(SimArgs a, u64 G0, u64 P0, u64 L0) {
  u64 s = 0;
  for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < a.n_wi; w += (u64)gridDim.x * blockDim.x) {
    const u64 g = w / a.V, l = w % a.V;
    const uint32_t np = min(a.nph[w], a.pcap);
    for (uint32_t p = 0; p < np; ++p) {
      const bool before = g < G0 || (g == G0 && (p < P0 || (p == P0 && l < L0)));
      if (before) s += a.seginstr[w * a.pcap + p];
    }
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&a.gl->ord, s);
}

__global__ void sim_divergence_kernel(SimArgs a) {
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < a.G; g += (u64)gridDim.x * blockDim.x)
    if (a.gfin_min[g] < a.gfin_max[g]) atomicMin(&a.gl->div_group, (uint32_t)g);
}

__global__ void sim_culprit_kernel(SimArgs a) {
  const u64 g = a.gl->div_group;
  const uint32_t r = a.gfin_min[g];
  for (u64 l = (u64)blockIdx.x * blockDim.x + threadIdx.x; l < a.V; l += (u64)gridDim.x * blockDim.x) {
    const u64 w = g * a.V + l;
    const uint32_t fin = (a.wend[w] == END_RET || a.wend[w] == END_ERROR) ? a.nph[w] - 1 : FIN_NEVER;
    if (fin == r) atomicMin(&a.gl->culprit, (uint32_t)w);
    if (fin > r) atomicMin(&a.gl->waiting, (uint32_t)w);
  }
}

__global__ void sim_ends_kernel(uint8_t* kind, u64* pay, u64 n) {
  kind[0] = AIWC_K_KERNEL_BEGIN;
  pay[0] = 0;
  kind[n - 1] = AIWC_K_KERNEL_END;
  pay[n - 1] = 0;
}

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t grow(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    bytes = std::max<size_t>(bytes, 256);
    const cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

int bitwidth(u64 x) { return x ? 64 - __builtin_clzll(x) : 0; }

}  // namespace

struct aiwc_sim {
  std::string err;
  DBuf code, imm, bbase, blen, boff, mem, regs, rlen, log_e, log_v, smin, sown, sacc, nph, wend, segcnt, seginstr,
      gnph, gfin_min, gfin_max, gseg, segv, scan_scratch, gl, s_pc, s_br, s_status;
  SimArgs a{};
  bool planned = false;
  int mode = MEM_SPEC;
  u64 n_events = 0, n_elem = 0, spec_grid = 0, group_grid = 0;
  const u64* mem_init = nullptr;
};

namespace {

int sim_fail(aiwc_sim* s, int code, const std::string& m) {
  s->err = m;
  return code;
}

#define SCK(x)                                                                               \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) return sim_fail(sim, AIWC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int read_globals(aiwc_sim* sim, SimGlobals& h, cudaStream_t st) {
  SCK(cudaMemcpyAsync(&h, sim->gl.p, sizeof(SimGlobals), cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  return AIWC_OK;
}

int fresh_memory(aiwc_sim* sim, cudaStream_t st) {
  if (sim->n_elem)
    SCK(cudaMemcpyAsync(sim->mem.p, sim->mem_init, sim->n_elem * 8, cudaMemcpyDeviceToDevice, st));
  return AIWC_OK;
}

// pass COUNT in `mode`, growing the per-round arrays until every round fits
int run_count(aiwc_sim* sim, int mode, SimGlobals& h, cudaStream_t st) {
  SimArgs& a = sim->a;
  for (;;) {
    SCK(sim->segcnt.grow(a.n_wi * a.pcap * 4));
    SCK(sim->seginstr.grow(a.n_wi * a.pcap * 4));
    a.segcnt = sim->segcnt.as<uint32_t>();
    a.seginstr = sim->seginstr.as<uint32_t>();
    sim_init_kernel<<<592, 256, 0, st>>>(a, sim->n_elem, mode);
    if (mode == MEM_SPEC) {
      sim_spec_kernel<MODE_COUNT><<<(unsigned)sim->spec_grid, SPEC_TPB, 0, st>>>(a);
    } else {
      if (int r = fresh_memory(sim, st)) return r;
      SCK(cudaMemsetAsync(a.nph, 0, a.n_wi * 4, st));
      if (mode == MEM_GROUP) {
        sim_group_kernel<MODE_COUNT><<<(unsigned)sim->group_grid, 32, 0, st>>>(a, ~0ull);
        sim_group_check_kernel<<<592, 256, 0, st>>>(a, sim->n_elem);
      } else {
        sim_seq_kernel<MODE_COUNT><<<1, 32, 0, st>>>(a);
      }
    }
    SCK(cudaGetLastError());
    if (int r = read_globals(sim, h, st)) return r;
    if (h.max_nph <= a.pcap) return AIWC_OK;
    a.pcap = h.max_nph;
  }
}

}  // namespace

extern "C" aiwc_sim* aiwc_sim_create(void) { return new (std::nothrow) aiwc_sim(); }

extern "C" void aiwc_sim_destroy(aiwc_sim* sim) {
  if (!sim) return;
  DBuf* bufs[] = {&sim->code, &sim->imm, &sim->bbase, &sim->blen, &sim->boff, &sim->mem, &sim->regs,
                  &sim->rlen, &sim->log_e, &sim->log_v, &sim->smin, &sim->sown, &sim->sacc, &sim->nph,
                  &sim->wend, &sim->segcnt, &sim->seginstr, &sim->gnph, &sim->gfin_min, &sim->gfin_max,
                  &sim->gseg, &sim->segv, &sim->scan_scratch, &sim->gl, &sim->s_pc, &sim->s_br, &sim->s_status};
  for (DBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  delete sim;
}

extern "C" const char* aiwc_sim_last_error(const aiwc_sim* sim) { return sim ? sim->err.c_str() : "null sim"; }

extern "C" int aiwc_sim_plan(aiwc_sim* sim, const aiwc_sim_launch* L, aiwc_sim_result* out, void* stream) {
  if (!sim || !L || !out) return AIWC_ERR_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  memset(out, 0, sizeof(*out));
  out->line = -1;
  sim->planned = false;
  SimArgs& a = sim->a;
  a = SimArgs{};
  if (!L->code || L->n_instr == 0) return sim_fail(sim, AIWC_ERR_ARGUMENT, "empty program");
  u64 V = 1, G = 1;
  for (int d = 0; d < 3; ++d) {
    if (L->local_size[d] == 0 || L->global_size[d] % L->local_size[d])
      return sim_fail(sim, AIWC_ERR_ARGUMENT, "local size must divide the global size");
    a.gsz[d] = L->global_size[d];
    a.lsz[d] = L->local_size[d];
    a.ngrp[d] = L->global_size[d] / L->local_size[d];
    V *= a.lsz[d];
    G *= a.ngrp[d];
  }
  if (V * G >= (1ull << 32) || V * G / V != G) {
    out->error = AIWC_SIM_UNSUPPORTED;
    return sim_fail(sim, AIWC_ERR_UNSUPPORTED, "more than 2^32 work-items");
  }
  a.V = V;
  a.G = G;
  a.n_wi = V * G;
  a.n_regs = std::max(L->n_regs, 1u);
  a.wmax = std::min(std::max(L->max_width, 1u), AIWC_SIM_MAX_WIDTH);
  // device copies of the program and the buffer table
  std::vector<u64> boff(L->n_buffers + 1, 0);
  for (uint32_t b = 0; b < L->n_buffers; ++b) boff[b + 1] = boff[b] + L->buf_len[b];
  sim->n_elem = boff[L->n_buffers];
  SCK(sim->code.grow((size_t)L->n_instr * SIMW * 4));
  SCK(sim->imm.grow(std::max<size_t>(L->n_imm, 1) * 8));
  SCK(sim->bbase.grow(std::max<size_t>(L->n_buffers, 1) * 8));
  SCK(sim->blen.grow(std::max<size_t>(L->n_buffers, 1) * 8));
  SCK(sim->boff.grow(std::max<size_t>(L->n_buffers, 1) * 8));
  SCK(cudaMemcpyAsync(sim->code.p, L->code, (size_t)L->n_instr * SIMW * 4, cudaMemcpyHostToDevice, st));
  if (L->n_imm) SCK(cudaMemcpyAsync(sim->imm.p, L->imm, (size_t)L->n_imm * 8, cudaMemcpyHostToDevice, st));
  if (L->n_buffers) {
    SCK(cudaMemcpyAsync(sim->bbase.p, L->buf_base, (size_t)L->n_buffers * 8, cudaMemcpyHostToDevice, st));
    SCK(cudaMemcpyAsync(sim->blen.p, L->buf_len, (size_t)L->n_buffers * 8, cudaMemcpyHostToDevice, st));
    SCK(cudaMemcpyAsync(sim->boff.p, boff.data(), (size_t)L->n_buffers * 8, cudaMemcpyHostToDevice, st));
  }
  a.code = sim->code.as<int32_t>();
  a.imm = sim->imm.as<u64>();
  a.bbase = sim->bbase.as<u64>();
  a.blen = sim->blen.as<u64>();
  a.boff = sim->boff.as<u64>();
  sim->mem_init = reinterpret_cast<const u64*>(L->mem_dev);
  SCK(sim->mem.grow(std::max<u64>(sim->n_elem, 1) * 8));
  // register-file slots: speculative mode one per thread, group mode V per thread
  // (one group each), sequential mode V; register file within ~1 GiB where possible
  const u64 per_slot = (u64)a.n_regs * a.wmax * 8 + (u64)a.n_regs * 4 + 2ull * LOGCAP * 8 + 9;
  u64 slots = std::min<u64>((a.n_wi + SPEC_TPB - 1) / SPEC_TPB, 148ull * 16) * SPEC_TPB;
  while (slots > SPEC_TPB && slots * per_slot > (1ull << 30)) slots /= 2;
  slots = std::max<u64>(slots / SPEC_TPB, 1) * SPEC_TPB;
  sim->spec_grid = slots / SPEC_TPB;
  u64 gthreads = std::min<u64>(G, 148ull * 64);
  while (gthreads > 32 && gthreads * V * per_slot > (1ull << 30)) gthreads /= 2;
  sim->group_grid = (gthreads + 31) / 32;
  const u64 stride = std::max<u64>(slots, sim->group_grid * 32 * V);
  if (stride * per_slot > (48ull << 30)) {
    out->error = AIWC_SIM_UNSUPPORTED;
    return sim_fail(sim, AIWC_ERR_UNSUPPORTED, "register file of one work-group exceeds 48 GiB");
  }
  a.stride = stride;
  SCK(sim->regs.grow(stride * a.n_regs * a.wmax * 8));
  SCK(sim->rlen.grow(stride * a.n_regs * 4));
  // log entry i of slot s lives at [i * stride + s]: the logs span the whole stride
  SCK(sim->log_e.grow(stride * LOGCAP * 8));
  SCK(sim->log_v.grow(stride * LOGCAP * 8));
  SCK(sim->smin.grow(std::max<u64>(sim->n_elem, 1) * 8));
  SCK(sim->sown.grow(std::max<u64>(sim->n_elem, 1) * 4));
  SCK(sim->sacc.grow(std::max<u64>(sim->n_elem, 1) * 4));
  SCK(sim->nph.grow(a.n_wi * 4));
  SCK(sim->wend.grow(a.n_wi));
  SCK(sim->gnph.grow(G * 4));
  SCK(sim->gfin_min.grow(G * 4));
  SCK(sim->gfin_max.grow(G * 4));
  SCK(sim->gseg.grow((G + 1) * 8));
  SCK(sim->gl.grow(sizeof(SimGlobals)));
  SCK(sim->s_pc.grow(stride * 4));
  SCK(sim->s_br.grow(stride * 4));
  SCK(sim->s_status.grow(stride));
  a.regs = sim->regs.as<u64>();
  a.rlen = sim->rlen.as<uint32_t>();
  a.log_e = sim->log_e.as<u64>();
  a.log_v = sim->log_v.as<u64>();
  a.smin = sim->smin.as<u64>();
  a.sown = sim->sown.as<uint32_t>();
  a.sacc = sim->sacc.as<uint32_t>();
  a.nph = sim->nph.as<uint32_t>();
  a.wend = sim->wend.as<uint8_t>();
  a.gnph = sim->gnph.as<uint32_t>();
  a.gfin_min = sim->gfin_min.as<uint32_t>();
  a.gfin_max = sim->gfin_max.as<uint32_t>();
  a.gl = sim->gl.as<SimGlobals>();
  a.s_pc = sim->s_pc.as<uint32_t>();
  a.s_br = sim->s_br.as<int32_t>();
  a.s_status = sim->s_status.as<uint8_t>();
  a.kb_l = std::max(bitwidth(V - 1), 1);
  const int kb_g = std::max(bitwidth(G - 1), 1);
  a.kb_p = 64 - a.kb_l - kb_g;
  a.pmax = a.kb_p >= 32 ? 0xFFFFFFFEu : (uint32_t)((1ull << a.kb_p) - 1);
  a.pcap = 2;
  const u64 limit = std::min<u64>(L->step_limit, 1ull << 62);

  // ---- speculative -> group -> sequential, each only when the previous one cannot prove exactness ----
  SimGlobals h{};
  int mode = (L->flags & AIWC_SIM_FORCE_SEQUENTIAL) || a.kb_p < 1 ? MEM_SEQ
             : (L->flags & AIWC_SIM_FORCE_GROUP)                   ? MEM_GROUP
                                                                   : MEM_SPEC;
  if (mode == MEM_SPEC) {
    a.mem = const_cast<u64*>(sim->mem_init);
    a.cap = limit + 1;
    if (int r = run_count(sim, MEM_SPEC, h, st)) return r;
    bool dep = (h.flags & (SF_LOG | SF_KEY)) != 0;
    if (!dep) {
      sim_spec_kernel<MODE_VERIFY><<<(unsigned)sim->spec_grid, SPEC_TPB, 0, st>>>(a);
      SCK(cudaGetLastError());
      SimGlobals hv;
      if (int r = read_globals(sim, hv, st)) return r;
      dep = (hv.flags & (SF_CONFLICT | SF_LOG)) != 0;
    }
    if (dep) mode = MEM_GROUP;
  }
  if (mode == MEM_GROUP) {
    a.mem = sim->mem.as<u64>();
    a.cap = limit + 1;
    if (int r = run_count(sim, MEM_GROUP, h, st)) return r;
    if (h.flags & SF_CONFLICT) mode = MEM_SEQ;
  }
  if (mode == MEM_SEQ) {
    a.mem = sim->mem.as<u64>();
    a.cap = limit;
    if (int r = run_count(sim, MEM_SEQ, h, st)) return r;
  }
  sim->mode = mode;
  out->sequential = mode == MEM_SEQ ? 1u : (mode == MEM_GROUP ? 2u : 0u);

  // ---- layout: segments in (group, round, local id) order ----
  u64* gseg = sim->gseg.as<u64>();
  u64* scan_total = sim->gl.as<u64>() + (offsetof(SimGlobals, ord) / 8);
  sim_group_seg_kernel<<<(unsigned)std::min<u64>((G + 255) / 256, 4096), 256, 0, st>>>(a, gseg);
  SCK(sim->scan_scratch.grow(aiwc::scan_scratch_elems(G + 1) * 8));
  u64 S = 0;
  SCK(cudaMemsetAsync(scan_total, 0, 8, st));
  aiwc::scan_exclusive_u64(gseg, G, sim->scan_scratch.as<u64>(), scan_total, st, nullptr);
  SCK(cudaMemcpyAsync(gseg + G, scan_total, 8, cudaMemcpyDeviceToDevice, st));
  SCK(cudaMemcpyAsync(&S, scan_total, 8, cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  a.gseg = gseg;
  SCK(sim->segv.grow((S + 1) * 8));
  u64* segv = sim->segv.as<u64>();
  sim_segv_kernel<<<(unsigned)std::min<u64>((a.n_wi + 255) / 256, 8192), 256, 0, st>>>(a, segv);
  u64 seg_total = 0;
  SCK(sim->scan_scratch.grow(aiwc::scan_scratch_elems(S + 1) * 8));
  SCK(cudaMemsetAsync(scan_total, 0, 8, st));
  aiwc::scan_exclusive_u64(segv, S, sim->scan_scratch.as<u64>(), scan_total, st, nullptr);
  SCK(cudaMemcpyAsync(segv + S, scan_total, 8, cudaMemcpyDeviceToDevice, st));
  SCK(cudaMemcpyAsync(&seg_total, scan_total, 8, cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  a.segpos = segv;
  sim->n_events = 2 + 2 * G + seg_total;
  out->n_events = sim->n_events;
  out->n_groups = G;
  out->n_instr = h.tot[0];
  out->n_reads = h.tot[1];
  out->n_writes = h.tot[2];
  out->n_branches = h.tot[3];
  out->n_barriers = h.tot[4];

  auto dev_u64 = [&](const u64* p, u64& v) -> int {
    SCK(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    return AIWC_OK;
  };
  auto dev_u32 = [&](const uint32_t* p, uint32_t& v) -> int {
    SCK(cudaMemcpyAsync(&v, p, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    return AIWC_OK;
  };
  // event index of the open event of segment (g, p, l): 2 + 2g + segpos[gseg[g] + pV + l]
  auto open_event = [&](u64 g, u64 p, u64 l, u64& ev) -> int {
    u64 gs = 0, sp = 0;
    if (int r = dev_u64(gseg + g, gs)) return r;
    if (int r = dev_u64(segv + gs + p * V + l, sp)) return r;
    ev = 2 + 2 * g + sp;
    return AIWC_OK;
  };
  auto fault_out = [&](const Fault& f) {
    out->error = f.code;
    out->line = f.line;
    out->reg = f.reg;
    out->lanes = f.lanes;
    out->width = f.width;
    out->buffer = f.buf;
    out->index = f.index;
  };
  auto fault_prefix = [&](u64 w, u64 p) -> int {  // events up to and including the faulting instruction
    u64 ev;
    if (int r = open_event(w / V, p, w % V, ev)) return r;
    uint32_t cnt = 0;
    if (int r = dev_u32(sim->segcnt.as<uint32_t>() + w * a.pcap + p, cnt)) return r;
    out->prefix_events = ev + 1 + cnt;
    out->wi = w;
    return AIWC_OK;
  };
  auto round_end = [&](u64 g, uint32_t r) -> int {  // events through barrier round r of group g
    u64 gs, sp;
    if (int e = dev_u64(gseg + g, gs)) return e;
    if (int e = dev_u64(segv + gs + (u64)(r + 1) * V, sp)) return e;
    out->prefix_events = 2 + 2 * g + sp;
    return AIWC_OK;
  };

  if (mode == MEM_SEQ) {
    if (h.s_stop == STOP_FAULT || h.s_stop == STOP_CAP) {
      if (int r = fault_prefix(h.s_wi, h.s_round)) return r;
      if (h.s_stop == STOP_FAULT) fault_out(h.f);
      else out->error = AIWC_SIM_STEP_LIMIT;
    } else if (h.s_stop == STOP_DIV) {
      if (int r = round_end(h.s_group, h.s_round)) return r;
      out->error = AIWC_SIM_DIVERGENCE;
      out->wi = h.culprit;
      out->wi2 = h.waiting;
      out->line = h.last_br;
      out->n_round = h.s_round;
    }
  } else {
    // earliest faulting segment, first divergent group, step limit: whichever comes first
    bool have_e = h.err_key != ~0ull, have_d = false;
    u64 eg = 0, ep = 0, el = 0, dg = 0;
    uint32_t dr = 0;
    if (have_e) {
      eg = h.err_key >> (a.kb_p + a.kb_l);
      ep = (h.err_key >> a.kb_l) & ((1ull << a.kb_p) - 1);
      el = h.err_key & ((1ull << a.kb_l) - 1);
    }
    sim_divergence_kernel<<<(unsigned)std::min<u64>((G + 255) / 256, 4096), 256, 0, st>>>(a);
    SimGlobals h2;
    if (int r = read_globals(sim, h2, st)) return r;
    if (h2.div_group != ~0u) {
      dg = h2.div_group;
      if (int r = dev_u32(a.gfin_min + dg, dr)) return r;
      have_d = true;
      if (have_e && (eg < dg || (eg == dg && ep <= dr))) have_d = false;
      else have_e = false;
    }
    auto ordinal = [&](u64 g, u64 p, u64 l, u64& o) -> int {
      SCK(cudaMemsetAsync(&a.gl->ord, 0, 8, st));
      sim_ordinal_kernel<<<(unsigned)std::min<u64>((a.n_wi + 255) / 256, 8192), 256, 0, st>>>(a, g, p, l);
      return dev_u64(&a.gl->ord, o);
    };
    bool step = false;
    if (have_e) {
      u64 o;
      if (int r = ordinal(eg, ep, el, o)) return r;
      uint32_t ni = 0;
      if (int r = dev_u32(sim->seginstr.as<uint32_t>() + (eg * V + el) * a.pcap + ep, ni)) return r;
      step = o + ni > limit;
    } else if (have_d) {
      u64 o;
      if (int r = ordinal(dg, (u64)dr + 1, 0, o)) return r;
      step = o > limit;
    } else {
      step = h.tot[0] > limit;
    }
    if (step) {
      out->error = AIWC_SIM_STEP_LIMIT;
      out->prefix_events = ~0ull;
    } else if (have_e || have_d) {
      SimGlobals hd;
      const u64 w_e = eg * V + el;
      if (mode == MEM_SPEC) {
        if (have_d) {
          sim_culprit_kernel<<<(unsigned)std::min<u64>((V + 255) / 256, 4096), 256, 0, st>>>(a);
          if (int r = read_globals(sim, hd, st)) return r;
        }
        const u64 culprit = have_d ? hd.culprit : 0, waiting = have_d ? hd.waiting : 0;
        sim_detail_kernel<<<1, 32, 0, st>>>(a, have_e ? w_e : culprit);
        if (int r = read_globals(sim, hd, st)) return r;
        hd.culprit = (uint32_t)culprit;
        hd.waiting = (uint32_t)waiting;
      } else {  // group mode: the group again, alone, from the initial memory
        if (int r = fresh_memory(sim, st)) return r;
        sim_group_kernel<MODE_DETAIL><<<1, 32, 0, st>>>(a, have_e ? eg : dg);
        if (int r = read_globals(sim, hd, st)) return r;
      }
      if (have_e) {
        fault_out(hd.f);
        if (int r = fault_prefix(w_e, ep)) return r;
      } else {
        if (int r = round_end(dg, dr)) return r;
        out->error = AIWC_SIM_DIVERGENCE;
        out->wi = hd.culprit;
        out->wi2 = hd.waiting;
        out->line = hd.last_br;
        out->n_round = dr;
      }
    }
  }
  sim->planned = true;
  return AIWC_OK;
}

extern "C" int aiwc_sim_emit(aiwc_sim* sim, uint8_t* kind_dev, uint64_t* payload_dev, uint64_t n_events,
                             void* stream) {
  if (!sim) return AIWC_ERR_ARGUMENT;
  if (!sim->planned) return sim_fail(sim, AIWC_ERR_ARGUMENT, "aiwc_sim_emit before aiwc_sim_plan");
  if (n_events != sim->n_events || !kind_dev || !payload_dev)
    return sim_fail(sim, AIWC_ERR_ARGUMENT, "output columns do not match the planned event count");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SimArgs a = sim->a;
  a.okind = kind_dev;
  a.opay = reinterpret_cast<u64*>(payload_dev);
  if (sim->mode == MEM_SPEC) {
    sim_spec_kernel<MODE_EMIT><<<(unsigned)sim->spec_grid, SPEC_TPB, 0, st>>>(a);
  } else {
    if (int r = fresh_memory(sim, st)) return r;
    if (sim->mode == MEM_GROUP) sim_group_kernel<MODE_EMIT><<<(unsigned)sim->group_grid, 32, 0, st>>>(a, ~0ull);
    else sim_seq_kernel<MODE_EMIT><<<1, 32, 0, st>>>(a);
  }
  sim_ends_kernel<<<1, 1, 0, st>>>(kind_dev, a.opay, n_events);
  SCK(cudaGetLastError());
  return AIWC_OK;
}
