// walker.cpp -- CPython extension `_walker`: TraceEvent iterable -> columnar trace.
//
// The object front door of consume(): it pulls events from any iterable
// (generators included, never materialised as a list), encodes them into the
// columnar layout of include/aiwc_b200.h and runs the reference's stream
// validation (StreamChecker, pkg/src/aiwc/trace.py:289-424) on the way, so
// InvalidStream carries the same event index, rule and detail text.
// Encoding stops at the first violation; the encoded prefix lets consume()
// decide whether the entry cap would have been crossed first
// (metrics.py:126-155).  No metric is computed here.
//
// Event classes are recognised by class name + tuple position, so both this
// package's NamedTuples and the reference's own aiwc.trace classes work.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <cstdint>
#include <thread>
#include <cstring>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/aiwc_b200.h"

namespace {

enum Ev { E_KB, E_KE, E_WGB, E_WGE, E_WIB, E_WIR, E_WIE, E_INS, E_BR, E_MEM, E_BAR, E_NONE };

PyObject* g_unsupported = nullptr;  // UnsupportedTrace class
PyObject* g_type_cache = nullptr;   // dict: type -> Ev code

int ev_code(PyObject* ev) {
  PyObject* t = reinterpret_cast<PyObject*>(Py_TYPE(ev));
  PyObject* c = PyDict_GetItem(g_type_cache, t);
  if (c) return (int)PyLong_AsLong(c);
  static const char* names[] = {"KernelBegin", "KernelEnd", "WorkGroupBegin", "WorkGroupEnd", "WorkItemBegin",
                                "WorkItemResume", "WorkItemEnd", "Instruction", "Branch", "Memory", "Barrier"};
  static const int sizes[] = {4, 0, 1, 1, 1, 1, 1, 2, 2, 2, 0};
  int code = E_NONE;
  if (PyTuple_Check(ev)) {
    const char* nm = Py_TYPE(ev)->tp_name;
    const char* dot = strrchr(nm, '.');
    if (dot) nm = dot + 1;
    for (int i = 0; i < 11; ++i)
      if (!strcmp(nm, names[i]) && PyTuple_GET_SIZE(ev) == sizes[i]) code = i;
  }
  PyObject* v = PyLong_FromLong(code);
  PyDict_SetItem(g_type_cache, t, v);
  Py_DECREF(v);
  return code;
}

struct V3 {
  long long v[3];
  bool operator==(const V3& o) const { return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2]; }
};
struct V3Hash {
  size_t operator()(const V3& a) const {
    uint64_t h = (uint64_t)a.v[0] * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)a.v[1] + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
    h ^= (uint64_t)a.v[2] + 0x94D049BB133111EBull + (h << 6) + (h >> 2);
    return (size_t)h;
  }
};

bool get_ll(PyObject* o, long long* out) {
  int ovf = 0;
  *out = PyLong_AsLongLongAndOverflow(o, &ovf);
  if (ovf || (*out == -1 && PyErr_Occurred())) {
    PyErr_Clear();
    return false;
  }
  return true;
}
bool get_u64(PyObject* o, uint64_t* out) {
  if (!PyLong_Check(o)) return false;
  unsigned long long v = PyLong_AsUnsignedLongLong(o);
  if (v == (unsigned long long)-1 && PyErr_Occurred()) {
    PyErr_Clear();
    return false;
  }
  *out = v;
  return true;
}
bool get_v3(PyObject* o, V3* out) {
  PyObject* seq = PySequence_Fast(o, "vec3");
  if (!seq) { PyErr_Clear(); return false; }
  bool ok = PySequence_Fast_GET_SIZE(seq) == 3;
  for (int d = 0; ok && d < 3; ++d) ok = get_ll(PySequence_Fast_GET_ITEM(seq, d), &out->v[d]);
  Py_DECREF(seq);
  return ok;
}
std::string v3s(const V3& a) {
  return "(" + std::to_string(a.v[0]) + ", " + std::to_string(a.v[1]) + ", " + std::to_string(a.v[2]) + ")";
}

enum WiStatus { ST_OPEN = 1, ST_AT_BARRIER = 2, ST_DONE = 3 };

struct Walker {
  std::vector<uint8_t> kind;
  std::vector<uint64_t> pay;
  // header
  bool have_header = false, ended = false;
  std::string kernel_name;
  PyObject* kernel_name_obj = nullptr;
  long long invocation = 0;
  V3 gsz{{1, 1, 1}}, lsz{{1, 1, 1}}, grid{{1, 1, 1}};
  PyObject* invocation_obj = nullptr;
  // dictionaries
  PyObject* opc_dict = nullptr;  // opcode object -> id
  PyObject* opc_list = nullptr;
  std::unordered_map<V3, uint32_t, V3Hash> extra;
  std::vector<V3> extra_list;
  // checker state (trace.py:297-307)
  bool group_open = false;
  V3 open_group{};
  bool seg_open = false;
  V3 seg_gid{};
  std::unordered_map<V3, size_t, V3Hash> wi_index;  // insertion-ordered status / barrier counts
  std::vector<V3> wi_order;
  std::vector<int> wi_status;
  std::vector<long long> wi_barriers;
  long long index = -1;
  // first violation
  bool violated = false;
  long long v_index = 0;
  std::string v_rule, v_detail;
  // address statistics
  uint64_t amin = ~0ull, amax = 0, aand = ~0ull, aor = 0;
  uint64_t n_mem = 0;
  // class totals (declared to the engine: one-pass ingest)
  uint64_t c_instr = 0, c_rd = 0, c_wr = 0, c_br = 0, c_wgb = 0, c_bres = 0;

  void flag(long long i, const char* rule, const std::string& detail) {
    if (violated) return;
    violated = true;
    v_index = i; v_rule = rule; v_detail = detail;
  }
  size_t wi_slot(const V3& key, bool create) {
    auto it = wi_index.find(key);
    if (it != wi_index.end()) return it->second;
    if (!create) return (size_t)-1;
    wi_index.emplace(key, wi_order.size());
    wi_order.push_back(key); wi_status.push_back(0); wi_barriers.push_back(-1);
    return wi_order.size() - 1;
  }
  void reset_group() { wi_index.clear(); wi_order.clear(); wi_status.clear(); wi_barriers.clear(); }
  uint64_t group_key(const V3& g) {
    bool in = true;
    for (int d = 0; d < 3; ++d) in = in && g.v[d] >= 0 && g.v[d] < grid.v[d];
    if (in) return (uint64_t)(g.v[0] + grid.v[0] * (g.v[1] + grid.v[1] * g.v[2]));
    auto it = extra.find(g);
    if (it != extra.end()) return it->second;
    const uint64_t base = (uint64_t)(grid.v[0] * grid.v[1] * grid.v[2]);
    const uint32_t k = (uint32_t)(base + extra_list.size());
    extra.emplace(g, k);
    extra_list.push_back(g);
    return k;
  }
  void push(uint8_t k, uint64_t p) {
    kind.push_back(k); pay.push_back(p);
    c_instr += k == AIWC_K_INSTR;
    c_rd += k == AIWC_K_LOAD || k == AIWC_K_ATOMIC_LOAD;
    c_wr += k == AIWC_K_STORE || k == AIWC_K_ATOMIC_STORE;
    c_br += k == AIWC_K_BRANCH;
    c_wgb += k == AIWC_K_WG_BEGIN;
    c_bres |= k == AIWC_K_BARRIER || k == AIWC_K_WI_RESUME;
  }
};

int unsupported(const char* msg) {
  PyErr_SetString(g_unsupported ? g_unsupported : PyExc_ValueError, msg);
  return -1;
}

// One event with native field values (both front doors fill it).
struct Rec {
  int c = E_NONE;
  uint64_t oid = 0, width = 0;         // instruction
  uint8_t memk = 0;                    // memory kind byte
  uint64_t addr = 0;
  uint64_t site = 0;                   // branch
  int taken = 0;
  V3 g{}, gid{}, lid{};                // group id (wg / wi events), global / local id (wi events)
  PyObject* name = nullptr;            // kernel_begin (borrowed)
  PyObject* inv = nullptr;
  V3 gsz{}, lsz{};
};

// opcode dictionary, shared by both front doors (ids in first-appearance order)
struct OpDict {
  std::unordered_map<std::string, uint64_t> str_ids;
};

int opcode_id_str(Walker& w, OpDict& d, const char* s, size_t n, uint64_t* oid) {
  std::string key(s, n);
  auto it = d.str_ids.find(key);
  if (it != d.str_ids.end()) { *oid = it->second; return 0; }
  PyObject* u = PyUnicode_DecodeUTF8(s, (Py_ssize_t)n, "strict");
  if (!u) return -1;
  const uint64_t id = (uint64_t)PyList_GET_SIZE(w.opc_list);
  PyObject* v = PyLong_FromUnsignedLongLong(id);
  const int rc = PyDict_SetItem(w.opc_dict, u, v);
  Py_DECREF(v);
  if (rc < 0 || PyList_Append(w.opc_list, u) < 0) { Py_DECREF(u); return -1; }
  Py_DECREF(u);
  d.str_ids.emplace(std::move(key), id);
  *oid = id;
  return 0;
}

int opcode_id_obj(Walker& w, OpDict& d, PyObject* op, uint64_t* oid) {
  if (PyUnicode_Check(op)) {
    Py_ssize_t n;
    const char* s = PyUnicode_AsUTF8AndSize(op, &n);
    if (s) return opcode_id_str(w, d, s, (size_t)n, oid);
    PyErr_Clear();  // not encodable: key it by object below
  }
  PyObject* id = PyDict_GetItemWithError(w.opc_dict, op);
  if (id) { *oid = PyLong_AsUnsignedLongLong(id); return 0; }
  if (PyErr_Occurred()) return -1;
  *oid = (uint64_t)PyList_GET_SIZE(w.opc_list);
  PyObject* v = PyLong_FromUnsignedLongLong(*oid);
  const int rc = PyDict_SetItem(w.opc_dict, op, v);
  Py_DECREF(v);
  if (rc < 0) return -1;
  return PyList_Append(w.opc_list, op);
}

// StreamChecker (trace.py:289-424) + columnar encoding of one event.
// returns 0 ok, 1 stop (violation), -1 Python error
int feed_rec(Walker& w, const Rec& r) {
  const long long i = ++w.index;
  const int c = r.c;
  if (w.ended) { w.flag(i, "kernel_end.last", "event after kernel_end"); return 1; }
  if (!w.have_header) {
    if (c == E_KB) {
      w.gsz = r.gsz; w.lsz = r.lsz;
      for (int d = 0; d < 3; ++d) {
        if (w.lsz.v[d] <= 0 || w.gsz.v[d] <= 0) return unsupported("launch sizes must be positive");
        w.grid.v[d] = (w.gsz.v[d] + w.lsz.v[d] - 1) / w.lsz.v[d];
      }
      if ((uint64_t)(w.grid.v[0] * w.grid.v[1] * w.grid.v[2]) >= (1ull << 31))
        return unsupported("more than 2^31 work-groups");
      if ((uint64_t)(w.lsz.v[0] * w.lsz.v[1] * w.lsz.v[2]) >= (1ull << 31))
        return unsupported("local size volume >= 2^31");
      Py_INCREF(r.name); w.kernel_name_obj = r.name;
      Py_INCREF(r.inv); w.invocation_obj = r.inv;
      w.have_header = true;
      w.push(AIWC_K_KERNEL_BEGIN, 0);
      return 0;
    }
    w.flag(i, "kernel_begin.first", "first event must be kernel_begin");
    return 1;
  }
  switch (c) {
    case E_INS: case E_MEM: case E_BR: {
      if (!w.seg_open) {
        static const char* nm[] = {"", "", "", "", "", "", "", "Instruction", "Branch", "Memory"};
        w.flag(i, "event.outside_segment", std::string(nm[c]) + " outside a work-item segment");
        return 1;
      }
      if (c == E_INS) {
        w.push(AIWC_K_INSTR, (r.oid << 32) | r.width);
      } else if (c == E_MEM) {
        w.push(r.memk, r.addr);
        w.amin = std::min(w.amin, r.addr); w.amax = std::max(w.amax, r.addr);
        w.aand &= r.addr; w.aor |= r.addr; ++w.n_mem;
      } else {
        w.push(AIWC_K_BRANCH, (r.site << 1) | (uint64_t)r.taken);
      }
      return 0;
    }
    case E_BAR: {
      if (!w.seg_open) { w.flag(i, "event.outside_segment", "Barrier outside a work-item segment"); return 1; }
      const size_t s = w.wi_slot(w.seg_gid, true);
      w.wi_status[s] = ST_AT_BARRIER;
      w.wi_barriers[s] = (w.wi_barriers[s] < 0 ? 0 : w.wi_barriers[s]) + 1;
      w.seg_open = false;
      w.push(AIWC_K_BARRIER, 0);
      return 0;
    }
    case E_KB: w.flag(i, "kernel_begin.first", "duplicate kernel_begin"); return 1;
    case E_KE:
      if (w.group_open) { w.flag(i, "wg.nesting", "kernel_end with open work-group"); return 1; }
      w.ended = true;
      w.push(AIWC_K_KERNEL_END, 0);
      return 0;
    case E_WGB: {
      if (w.group_open) { w.flag(i, "wg.nesting", "wg_begin while another group is open"); return 1; }
      w.group_open = true; w.open_group = r.g;
      w.reset_group();
      w.push(AIWC_K_WG_BEGIN, w.group_key(r.g));
      return 0;
    }
    case E_WGE: {
      if (!w.group_open || !(r.g == w.open_group)) { w.flag(i, "wg.nesting", "wg_end does not match open group"); return 1; }
      if (w.seg_open) { w.flag(i, "wi.nesting", "wg_end with open work-item segment"); return 1; }
      for (size_t s = 0; s < w.wi_order.size(); ++s)
        if (w.wi_status[s] != ST_DONE && w.wi_status[s] != 0) {
          w.flag(i, "wi.unfinished", "work-item " + v3s(w.wi_order[s]) + " never ended");
          return 1;
        }
      {
        std::vector<long long> counts;
        for (long long b : w.wi_barriers)
          if (b >= 0) counts.push_back(b);
        std::sort(counts.begin(), counts.end());
        counts.erase(std::unique(counts.begin(), counts.end()), counts.end());
        if (counts.size() > 1) {
          std::string lst = "[";
          for (size_t k = 0; k < counts.size(); ++k) lst += (k ? ", " : "") + std::to_string(counts[k]);
          lst += "]";
          w.flag(i, "barrier.divergence", "work-items of group " + v3s(w.open_group) + " hit differing barrier counts " + lst);
          return 1;
        }
      }
      w.group_open = false;
      w.reset_group();
      w.push(AIWC_K_WG_END, w.group_key(r.g));
      return 0;
    }
    default: {  // work-item events
      const V3 &gid = r.gid, &lid = r.lid, &grp = r.g;
      if (!w.group_open) { w.flag(i, "wi.nesting", "work-item event outside a work-group"); return 1; }
      if (!(grp == w.open_group)) { w.flag(i, "wi.nesting", "work-item belongs to a different group"); return 1; }
      for (int d = 0; d < 3; ++d) {  // _check_id (trace.py:410-418)
        if (lid.v[d] >= w.lsz.v[d]) {
          w.flag(i, "wi.id_arithmetic", "local_id[" + std::to_string(d) + "] >= local_size[" + std::to_string(d) + "]");
          return 1;
        }
        if (gid.v[d] != grp.v[d] * w.lsz.v[d] + lid.v[d]) {
          w.flag(i, "wi.id_arithmetic", "global_id != group_id*local_size + local_id");
          return 1;
        }
      }
      if (lid.v[0] < 0 || lid.v[1] < 0 || lid.v[2] < 0) return unsupported("negative local id");
      const uint64_t llin = (uint64_t)(lid.v[0] + w.lsz.v[0] * (lid.v[1] + w.lsz.v[1] * lid.v[2]));
      if (c == E_WIB) {
        if (w.seg_open) { w.flag(i, "wi.nesting", "segment opened while another is open"); return 1; }
        if (w.wi_index.count(gid)) { w.flag(i, "wi.nesting", "wi_begin for an already-started work-item"); return 1; }
        const size_t s = w.wi_slot(gid, true);
        w.wi_status[s] = ST_OPEN;
        if (w.wi_barriers[s] < 0) w.wi_barriers[s] = 0;
        w.seg_open = true; w.seg_gid = gid;
        w.push(AIWC_K_WI_BEGIN, llin);
      } else if (c == E_WIR) {
        if (w.seg_open) { w.flag(i, "wi.nesting", "segment opened while another is open"); return 1; }
        const size_t s = w.wi_slot(gid, false);
        if (s == (size_t)-1 || w.wi_status[s] != ST_AT_BARRIER) {
          w.flag(i, "wi.resume_without_barrier", "resume of a work-item not waiting at a barrier");
          return 1;
        }
        w.wi_status[s] = ST_OPEN;
        w.seg_open = true; w.seg_gid = gid;
        w.push(AIWC_K_WI_RESUME, llin);
      } else {
        if (!w.seg_open || !(w.seg_gid == gid)) { w.flag(i, "wi.nesting", "wi_end without matching open segment"); return 1; }
        w.seg_open = false;
        const size_t s = w.wi_slot(gid, true);
        w.wi_status[s] = ST_DONE;
        w.push(AIWC_K_WI_END, llin);
      }
      return 0;
    }
  }
}

// object front door: a TraceEvent (ours or the reference's NamedTuples)
int feed(Walker& w, OpDict& d, PyObject* ev) {
  const int c = ev_code(ev);
  if (c == E_NONE) {
    PyObject* r = PyObject_Repr(ev);
    PyErr_Format(PyExc_TypeError, "not a trace event: %U", r);
    Py_XDECREF(r);
    return -1;
  }
  Rec r;
  r.c = c;
  const bool open_or_header = !w.ended && w.have_header;
  switch (c) {
    case E_KB:
      if (w.have_header || w.ended) break;  // rule violation: fields are not looked at
      r.name = PyTuple_GET_ITEM(ev, 0);
      r.inv = PyTuple_GET_ITEM(ev, 1);
      if (!get_v3(PyTuple_GET_ITEM(ev, 2), &r.gsz) || !get_v3(PyTuple_GET_ITEM(ev, 3), &r.lsz))
        return unsupported("kernel_begin sizes must be 3 integers");
      break;
    case E_INS:
      if (!open_or_header || !w.seg_open) break;
      if (!get_u64(PyTuple_GET_ITEM(ev, 1), &r.width) || r.width >= (1ull << 32))
        return unsupported("instruction width must be an integer in [0, 2^32)");
      if (opcode_id_obj(w, d, PyTuple_GET_ITEM(ev, 0), &r.oid) < 0) return -1;
      break;
    case E_MEM: {
      if (!open_or_header || !w.seg_open) break;
      PyObject* op = PyTuple_GET_ITEM(ev, 0);
      if (!get_u64(PyTuple_GET_ITEM(ev, 1), &r.addr)) return unsupported("memory address must be an integer in [0, 2^64)");
      if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "load") == 0) r.memk = AIWC_K_LOAD;
      else if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "atomic_load") == 0) r.memk = AIWC_K_ATOMIC_LOAD;
      else if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "atomic_store") == 0) r.memk = AIWC_K_ATOMIC_STORE;
      else r.memk = AIWC_K_STORE;  // metrics.py:138: anything not in READ_OPS is a write
      break;
    }
    case E_BR: {
      if (!open_or_header || !w.seg_open) break;
      if (!get_u64(PyTuple_GET_ITEM(ev, 0), &r.site) || r.site >= (1ull << 32))
        return unsupported("branch site must be an integer in [0, 2^32)");
      const int t = PyObject_IsTrue(PyTuple_GET_ITEM(ev, 1));
      if (t < 0) return -1;
      r.taken = t;
      break;
    }
    case E_WGB:
      if (!open_or_header || w.group_open) break;
      if (!get_v3(PyTuple_GET_ITEM(ev, 0), &r.g)) return unsupported("group id must be 3 integers");
      break;
    case E_WGE:
      if (!open_or_header) break;
      if (!get_v3(PyTuple_GET_ITEM(ev, 0), &r.g)) return unsupported("group id must be 3 integers");
      break;
    case E_WIB: case E_WIR: case E_WIE: {
      if (!open_or_header) break;
      PyObject* wi = PyTuple_GET_ITEM(ev, 0);
      if (!PyTuple_Check(wi) || PyTuple_GET_SIZE(wi) != 3) return unsupported("work_item must be a WorkItemId");
      if (!get_v3(PyTuple_GET_ITEM(wi, 0), &r.gid) || !get_v3(PyTuple_GET_ITEM(wi, 1), &r.lid) ||
          !get_v3(PyTuple_GET_ITEM(wi, 2), &r.g))
        return unsupported("work-item ids must be 3 integers");
      break;
    }
    default: break;
  }
  return feed_rec(w, r);
}

// ---- .aiwctrace canonical lines (trace.py:100-138 writes exactly these) -------
// A line is taken natively only in the writer's canonical form (fixed key
// order, compact separators, plain strings without escapes, plain decimal
// integers); any other line goes to the Python decode_event restatement, so
// rejection rules and messages stay the reference's (trace.py:177-244).
struct Cur {
  const char* p;
  const char* e;
  bool lit(const char* s) {
    const size_t n = strlen(s);
    if ((size_t)(e - p) < n || memcmp(p, s, n) != 0) return false;
    p += n;
    return true;
  }
  bool uint(uint64_t* out) {  // 0 | [1-9][0-9]*, < 2^64
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0') { ++p; *out = 0; return p >= e || *p < '0' || *p > '9'; }
    uint64_t v = 0;
    while (p < e && *p >= '0' && *p <= '9') {
      const uint64_t dgt = (uint64_t)(*p - '0');
      if (v > (~0ull - dgt) / 10) return false;
      v = v * 10 + dgt;
      ++p;
    }
    *out = v;
    return true;
  }
  bool v3(V3* out) {  // [a,b,c] of non-negative ints < 2^62
    if (!lit("[")) return false;
    for (int d = 0; d < 3; ++d) {
      uint64_t x;
      if ((d && !lit(",")) || !uint(&x) || x >= (1ull << 62)) return false;
      out->v[d] = (long long)x;
    }
    return lit("]");
  }
  bool str(const char** s, size_t* n) {  // "..." without escapes / control chars, non-empty
    if (!lit("\"")) return false;
    const char* b = p;
    while (p < e && *p != '"') {
      if (*p == '\\' || (unsigned char)*p < 0x20) return false;
      ++p;
    }
    if (p >= e || p == b) return false;
    *s = b; *n = (size_t)(p - b);
    ++p;
    return true;
  }
  bool end() { return lit("}") && p == e; }
};

// 1 parsed, 0 not canonical (caller falls back), -1 Python error
int parse_canonical(Walker& w, OpDict& d, const char* b, const char* e, Rec* r, PyObject** tmp) {
  Cur c{b, e};
  if (!c.lit("{\"ev\":\"")) return 0;
  if (c.lit("instr\",\"opcode\":")) {
    const char* s; size_t n;
    if (!c.str(&s, &n) || !c.lit(",\"width\":") || !c.uint(&r->width) || !c.end()) return 0;
    if (r->width == 0 || r->width >= (1ull << 32)) return 0;
    // non-ASCII opcode bytes: let Python validate the UTF-8
    for (size_t k = 0; k < n; ++k) if ((unsigned char)s[k] >= 0x80) return 0;
    if (opcode_id_str(w, d, s, n, &r->oid) < 0) return -1;
    r->c = E_INS;
    return 1;
  }
  if (c.lit("mem\",\"op\":\"")) {
    if (c.lit("load\"")) r->memk = AIWC_K_LOAD;
    else if (c.lit("store\"")) r->memk = AIWC_K_STORE;
    else if (c.lit("atomic_load\"")) r->memk = AIWC_K_ATOMIC_LOAD;
    else if (c.lit("atomic_store\"")) r->memk = AIWC_K_ATOMIC_STORE;
    else return 0;
    if (!c.lit(",\"addr\":") || !c.uint(&r->addr) || !c.end()) return 0;
    r->c = E_MEM;
    return 1;
  }
  if (c.lit("branch\",\"site\":")) {
    if (!c.uint(&r->site) || r->site >= (1ull << 32) || !c.lit(",\"taken\":")) return 0;
    if (c.lit("true")) r->taken = 1;
    else if (c.lit("false")) r->taken = 0;
    else return 0;
    if (!c.end()) return 0;
    r->c = E_BR;
    return 1;
  }
  if (c.lit("barrier\"")) { if (!c.end()) return 0; r->c = E_BAR; return 1; }
  if (c.lit("kernel_end\"")) { if (!c.end()) return 0; r->c = E_KE; return 1; }
  int wi = -1;
  if (c.lit("wi_begin\"")) wi = E_WIB;
  else if (c.lit("wi_resume\"")) wi = E_WIR;
  else if (c.lit("wi_end\"")) wi = E_WIE;
  if (wi >= 0) {
    if (!c.lit(",\"global\":") || !c.v3(&r->gid) || !c.lit(",\"local\":") || !c.v3(&r->lid) ||
        !c.lit(",\"group\":") || !c.v3(&r->g) || !c.end())
      return 0;
    r->c = wi;
    return 1;
  }
  if (c.lit("wg_begin\",\"group\":")) { if (!c.v3(&r->g) || !c.end()) return 0; r->c = E_WGB; return 1; }
  if (c.lit("wg_end\",\"group\":")) { if (!c.v3(&r->g) || !c.end()) return 0; r->c = E_WGE; return 1; }
  if (c.lit("kernel_begin\",\"kernel\":")) {
    const char* s; size_t n;
    uint64_t inv;
    if (!c.str(&s, &n) || !c.lit(",\"invocation\":") || !c.uint(&inv) || !c.lit(",\"global_size\":") ||
        !c.v3(&r->gsz) || !c.lit(",\"local_size\":") || !c.v3(&r->lsz) || !c.end())
      return 0;
    for (int k = 0; k < 3; ++k) if (r->gsz.v[k] < 1 || r->lsz.v[k] < 1) return 0;
    for (size_t k = 0; k < n; ++k) if ((unsigned char)s[k] >= 0x80) return 0;
    tmp[0] = PyUnicode_DecodeUTF8(s, (Py_ssize_t)n, "strict");
    tmp[1] = PyLong_FromUnsignedLongLong(inv);
    if (!tmp[0] || !tmp[1]) return -1;
    r->name = tmp[0]; r->inv = tmp[1];
    r->c = E_KB;
    return 1;
  }
  return 0;
}

// ---- validate_stream (trace.py:427-437): every violation, reference state rules ----
// A separate, collect-everything restatement of StreamChecker.feed / finish
// (trace.py:309-424): it keeps going after a violation exactly as the
// reference does (which state each rule updates, several flags per event).
struct Checker {
  bool have_header = false, ended = false;
  V3 lsz{{1, 1, 1}};
  bool group_open = false;
  V3 open_group{};
  bool seg_open = false;
  V3 seg_gid{};
  std::unordered_map<V3, size_t, V3Hash> idx;  // insertion-ordered status dict
  std::vector<V3> order;
  std::vector<int> status;                      // 0 absent (never), ST_*
  std::unordered_map<V3, long long, V3Hash> barrier_counts;
  long long index = -1;
  std::vector<std::tuple<long long, std::string, std::string>> v;
  void flag(long long i, const char* rule, const std::string& d) { v.emplace_back(i, rule, d); }
  void clear_group() { idx.clear(); order.clear(); status.clear(); barrier_counts.clear(); }
  void set_status(const V3& k, int st) {
    auto it = idx.find(k);
    if (it == idx.end()) { idx.emplace(k, order.size()); order.push_back(k); status.push_back(st); }
    else status[it->second] = st;
  }
  int get_status(const V3& k) const {
    auto it = idx.find(k);
    return it == idx.end() ? 0 : status[it->second];
  }
};

void check_all(Checker& k, const Rec& r) {
  const long long i = ++k.index;
  const int t = r.c;
  if (k.ended) { k.flag(i, "kernel_end.last", "event after kernel_end"); return; }
  if (!k.have_header) {
    if (t == E_KB) { k.have_header = true; k.lsz = r.lsz; return; }
    k.flag(i, "kernel_begin.first", "first event must be kernel_begin");
    k.have_header = true;
    k.lsz = V3{{1, 1, 1}};
  }
  if (t == E_INS || t == E_MEM || t == E_BR) {
    static const char* nm[] = {"", "", "", "", "", "", "", "Instruction", "Branch", "Memory"};
    if (!k.seg_open) k.flag(i, "event.outside_segment", std::string(nm[t]) + " outside a work-item segment");
    return;
  }
  if (t == E_BAR) {
    if (!k.seg_open) { k.flag(i, "event.outside_segment", "Barrier outside a work-item segment"); return; }
    k.set_status(k.seg_gid, ST_AT_BARRIER);
    k.barrier_counts[k.seg_gid] += 1;
    k.seg_open = false;
    return;
  }
  if (t == E_KB) { k.flag(i, "kernel_begin.first", "duplicate kernel_begin"); return; }
  if (t == E_KE) {
    if (k.group_open) k.flag(i, "wg.nesting", "kernel_end with open work-group");
    k.ended = true;
    return;
  }
  if (t == E_WGB) {
    if (k.group_open) k.flag(i, "wg.nesting", "wg_begin while another group is open");
    k.group_open = true; k.open_group = r.g;
    k.clear_group();
    return;
  }
  if (t == E_WGE) {
    if (!k.group_open || !(r.g == k.open_group)) k.flag(i, "wg.nesting", "wg_end does not match open group");
    if (k.seg_open) { k.flag(i, "wi.nesting", "wg_end with open work-item segment"); k.seg_open = false; }
    for (size_t s = 0; s < k.order.size(); ++s)
      if (k.status[s] != ST_DONE) { k.flag(i, "wi.unfinished", "work-item " + v3s(k.order[s]) + " never ended"); break; }
    std::vector<long long> counts;
    for (auto& kv : k.barrier_counts) counts.push_back(kv.second);
    std::sort(counts.begin(), counts.end());
    counts.erase(std::unique(counts.begin(), counts.end()), counts.end());
    if (counts.size() > 1) {
      std::string lst = "[";
      for (size_t q = 0; q < counts.size(); ++q) lst += (q ? ", " : "") + std::to_string(counts[q]);
      lst += "]";
      k.flag(i, "barrier.divergence", "work-items of group " + (k.group_open ? v3s(k.open_group) : std::string("None")) +
                                          " hit differing barrier counts " + lst);
    }
    k.group_open = false;
    k.clear_group();
    return;
  }
  // work-item events
  if (!k.group_open) { k.flag(i, "wi.nesting", "work-item event outside a work-group"); return; }
  if (!(r.g == k.open_group)) k.flag(i, "wi.nesting", "work-item belongs to a different group");
  for (int d = 0; d < 3; ++d) {  // _check_id (trace.py:410-418)
    if (r.lid.v[d] >= k.lsz.v[d]) {
      k.flag(i, "wi.id_arithmetic", "local_id[" + std::to_string(d) + "] >= local_size[" + std::to_string(d) + "]");
      break;
    }
    if (r.gid.v[d] != r.g.v[d] * k.lsz.v[d] + r.lid.v[d]) {
      k.flag(i, "wi.id_arithmetic", "global_id != group_id*local_size + local_id");
      break;
    }
  }
  const V3& key = r.gid;
  if (t == E_WIB) {
    if (k.seg_open) k.flag(i, "wi.nesting", "segment opened while another is open");
    if (k.idx.count(key)) k.flag(i, "wi.nesting", "wi_begin for an already-started work-item");
    k.set_status(key, ST_OPEN);
    if (!k.barrier_counts.count(key)) k.barrier_counts[key] = 0;
    k.seg_open = true; k.seg_gid = key;
  } else if (t == E_WIR) {
    if (k.seg_open) k.flag(i, "wi.nesting", "segment opened while another is open");
    if (k.get_status(key) != ST_AT_BARRIER) k.flag(i, "wi.resume_without_barrier", "resume of a work-item not waiting at a barrier");
    k.set_status(key, ST_OPEN);
    k.seg_open = true; k.seg_gid = key;
  } else {
    if (!k.seg_open || !(k.seg_gid == key)) k.flag(i, "wi.nesting", "wi_end without matching open segment");
    else k.seg_open = false;
    k.set_status(key, ST_DONE);
  }
}

// full conversion of a TraceEvent for the checker (no rule short-cuts)
int rec_from_obj(PyObject* ev, Rec* r) {
  const int c = ev_code(ev);
  if (c == E_NONE) {
    PyObject* rp = PyObject_Repr(ev);
    PyErr_Format(PyExc_TypeError, "not a trace event: %U", rp);
    Py_XDECREF(rp);
    return -1;
  }
  r->c = c;
  switch (c) {
    case E_KB:
      if (!get_v3(PyTuple_GET_ITEM(ev, 3), &r->lsz) || !get_v3(PyTuple_GET_ITEM(ev, 2), &r->gsz))
        return unsupported("kernel_begin sizes must be 3 integers");
      break;
    case E_WGB: case E_WGE:
      if (!get_v3(PyTuple_GET_ITEM(ev, 0), &r->g)) return unsupported("group id must be 3 integers");
      break;
    case E_WIB: case E_WIR: case E_WIE: {
      PyObject* wi = PyTuple_GET_ITEM(ev, 0);
      if (!PyTuple_Check(wi) || PyTuple_GET_SIZE(wi) != 3) return unsupported("work_item must be a WorkItemId");
      if (!get_v3(PyTuple_GET_ITEM(wi, 0), &r->gid) || !get_v3(PyTuple_GET_ITEM(wi, 1), &r->lid) ||
          !get_v3(PyTuple_GET_ITEM(wi, 2), &r->g))
        return unsupported("work-item ids must be 3 integers");
      break;
    }
    default: break;
  }
  return 0;
}

PyObject* py_validate(PyObject*, PyObject* args) {
  PyObject* iterable;
  if (!PyArg_ParseTuple(args, "O", &iterable)) return nullptr;
  PyObject* it = PyObject_GetIter(iterable);
  if (!it) return nullptr;
  Checker k;
  PyObject* ev;
  while ((ev = PyIter_Next(it))) {
    Rec r;
    const int rc = rec_from_obj(ev, &r);
    Py_DECREF(ev);
    if (rc < 0) { Py_DECREF(it); return nullptr; }
    check_all(k, r);
  }
  Py_DECREF(it);
  if (PyErr_Occurred()) return nullptr;
  if (!k.have_header) k.flag(0, "kernel_begin.first", "empty stream");  // finish() (trace.py:420-424)
  else if (!k.ended) k.flag(std::max(k.index, 0LL), "kernel_end.last", "stream has no kernel_end");
  PyObject* out = PyList_New((Py_ssize_t)k.v.size());
  for (size_t q = 0; q < k.v.size(); ++q)
    PyList_SET_ITEM(out, q, Py_BuildValue("(Lss)", std::get<0>(k.v[q]), std::get<1>(k.v[q]).c_str(),
                                          std::get<2>(k.v[q]).c_str()));
  return out;
}

// the result dict of both front doors; consumes the walker's references
PyObject* finish(Walker& w, int rc, long long last_line, PyObject* pending) {
  auto cleanup = [&]() {
    Py_XDECREF(w.opc_dict); Py_XDECREF(w.opc_list);
    Py_XDECREF(w.kernel_name_obj); Py_XDECREF(w.invocation_obj);
  };
  if (rc < 0 && !pending) { cleanup(); return nullptr; }
  if (rc == 0) {  // finish() (trace.py:420-424)
    if (!w.have_header) w.flag(0, "kernel_begin.first", "empty stream");
    else if (!w.ended) w.flag(std::max(w.index, 0LL), "kernel_end.last", "stream has no kernel_end");
  }
  PyObject* violation = Py_None;
  Py_INCREF(Py_None);
  if (w.violated) {
    Py_DECREF(Py_None);
    violation = Py_BuildValue("(Lss)", w.v_index, w.v_rule.c_str(), w.v_detail.c_str());
  }
  PyObject* kinds = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(w.kind.data()), (Py_ssize_t)w.kind.size());
  PyObject* pays = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(w.pay.data()), (Py_ssize_t)(w.pay.size() * 8));
  PyObject* extras = PyList_New((Py_ssize_t)w.extra_list.size());
  for (size_t k = 0; k < w.extra_list.size(); ++k)
    PyList_SET_ITEM(extras, k, Py_BuildValue("(LLL)", w.extra_list[k].v[0], w.extra_list[k].v[1], w.extra_list[k].v[2]));
  PyObject* stats = Py_None;
  Py_INCREF(Py_None);
  if (w.n_mem) {
    Py_DECREF(Py_None);
    stats = Py_BuildValue("(KKKK)", (unsigned long long)w.amin, (unsigned long long)w.amax,
                          (unsigned long long)w.aand, (unsigned long long)w.aor);
  }
  PyObject* name = w.kernel_name_obj ? w.kernel_name_obj : Py_None;
  PyObject* inv = w.invocation_obj ? w.invocation_obj : Py_None;
  PyObject* err = pending ? pending : Py_None;
  PyObject* counts = Py_BuildValue("(KKKKKK)", (unsigned long long)w.c_instr, (unsigned long long)w.c_rd,
                                   (unsigned long long)w.c_wr, (unsigned long long)w.c_br, (unsigned long long)w.c_wgb,
                                   (unsigned long long)w.c_bres);
  PyObject* out = Py_BuildValue("{s:N,s:N,s:O,s:O,s:(LLL),s:(LLL),s:O,s:N,s:N,s:N,s:O,s:L,s:O,s:N}", "kind", kinds,
                                "payload", pays, "kernel_name", name, "invocation", inv, "global_size", w.gsz.v[0],
                                w.gsz.v[1], w.gsz.v[2], "local_size", w.lsz.v[0], w.lsz.v[1], w.lsz.v[2], "opcodes",
                                w.opc_list, "extra_groups", extras, "addr_stats", stats, "violation", violation,
                                "have_header", w.have_header ? Py_True : Py_False, "last_line", last_line, "error",
                                err, "counts", counts);
  Py_XDECREF(pending);
  cleanup();
  return out;
}

PyObject* py_encode(PyObject*, PyObject* args) {
  PyObject* iterable;
  if (!PyArg_ParseTuple(args, "O", &iterable)) return nullptr;
  PyObject* it = PyObject_GetIter(iterable);
  if (!it) return nullptr;
  Walker w;
  OpDict d;
  w.opc_dict = PyDict_New();
  w.opc_list = PyList_New(0);
  int rc = 0;
  PyObject* ev;
  while ((ev = PyIter_Next(it))) {
    rc = feed(w, d, ev);
    Py_DECREF(ev);
    if (rc) break;
  }
  Py_DECREF(it);
  if (PyErr_Occurred()) rc = -1;
  return finish(w, rc, -1, nullptr);
}

// encode_lines(data: bytes, decode_event) -- the lines of an .aiwctrace file
// (iter_trace, trace.py:246-256): '#' lines are comments, canonical lines are
// parsed natively, every other line is decoded by decode_event(line, line_no)
// (the reference's json.loads path, with its MalformedEvent rules).  Stops at
// the first violation; a MalformedEvent (or decode error) is returned in
// "error" with the encoded prefix, so the caller can order it against the
// entry cap exactly as the reference's lazy consume() would.
PyObject* py_encode_lines(PyObject*, PyObject* args) {
  Py_buffer buf;
  PyObject* decode;
  if (!PyArg_ParseTuple(args, "y*O", &buf, &decode)) return nullptr;
  Walker w;
  OpDict d;
  w.opc_dict = PyDict_New();
  w.opc_list = PyList_New(0);
  const char* p = static_cast<const char*>(buf.buf);
  const char* end = p + buf.len;
  long long line_no = 0, last_line = -1;
  int rc = 0;
  PyObject* pending = nullptr;
  while (p < end && rc == 0) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    const char* le = nl ? nl : end;
    ++line_no;
    const char* b = p;
    p = nl ? nl + 1 : end;
    if (le > b && *b == '#') continue;
    last_line = line_no;
    Rec r;
    PyObject* tmp[2] = {nullptr, nullptr};
    int got = parse_canonical(w, d, b, le, &r, tmp);
    if (got == 1) {
      rc = feed_rec(w, r);
    } else if (got == 0) {
      PyObject* ev = nullptr;
      PyObject* line = PyUnicode_DecodeUTF8(b, (Py_ssize_t)(le - b), "strict");
      if (line) {
        ev = PyObject_CallFunction(decode, "OL", line, line_no);
        Py_DECREF(line);
      }
      if (!ev) {  // MalformedEvent / UnicodeDecodeError: hand back with the prefix
        PyObject *t, *v, *tb;
        PyErr_Fetch(&t, &v, &tb);
        PyErr_NormalizeException(&t, &v, &tb);
        pending = v ? v : (Py_INCREF(Py_None), Py_None);
        Py_XDECREF(t); Py_XDECREF(tb);
        rc = -1;
      } else {
        rc = feed(w, d, ev);
        Py_DECREF(ev);
      }
    } else {
      rc = -1;
    }
    Py_XDECREF(tmp[0]); Py_XDECREF(tmp[1]);
  }
  PyBuffer_Release(&buf);
  if (rc < 0 && !pending) return finish(w, -1, last_line, nullptr);
  return finish(w, pending ? 2 : rc, last_line, pending);
}

// ---- encode_lines_fast: the canonical lines of an .aiwctrace file on all host threads ----
// Every line after the header must be a canonical, decodable event line (no
// comments, no other forms) and pass the per-event checks that the columnar
// layout cannot carry (id arithmetic, a work-item's group = the open group);
// then chunks of lines are parsed in parallel into columns with chunk-local
// opcode / out-of-grid group dictionaries, merged in first-appearance order.
// The stream invariants are NOT checked here: the columns are handed to the
// engine as untrusted (the in-pass check / device validator).  Returns None
// whenever the sequential walker must decide (its errors are exact).
struct FastChunk {
  std::vector<uint8_t> kind;
  std::vector<uint64_t> pay;
  std::unordered_map<std::string, uint32_t> opc;
  std::vector<std::string> opc_order;
  std::unordered_map<V3, uint32_t, V3Hash> extra;
  std::vector<V3> extra_order;
  bool failed = false;
  bool has_gb = false, pre = false, pre_mismatch = false;
  V3 last_gb{}, pre_g{};
  uint64_t amin = ~0ull, amax = 0, aand = ~0ull, aor = 0, n_mem = 0;
  uint64_t c_instr = 0, c_rd = 0, c_wr = 0, c_br = 0, c_wgb = 0, c_bres = 0;
};

constexpr uint64_t EXTRA_TAG = 1ull << 63;  // chunk-local out-of-grid group key, remapped at the merge

void parse_chunk(const char* b, const char* e, const V3& lsz, const V3& grid, FastChunk* out) {
  FastChunk& ch = *out;
  auto gkey = [&](const V3& g) -> uint64_t {
    bool in = true;
    for (int d = 0; d < 3; ++d) in = in && g.v[d] < grid.v[d];
    if (in) return (uint64_t)(g.v[0] + grid.v[0] * (g.v[1] + grid.v[1] * g.v[2]));
    auto it = ch.extra.find(g);
    if (it != ch.extra.end()) return EXTRA_TAG | it->second;
    const uint32_t k = (uint32_t)ch.extra_order.size();
    ch.extra.emplace(g, k);
    ch.extra_order.push_back(g);
    return EXTRA_TAG | k;
  };
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* le = nl ? nl : e;
    Cur c{p, le};
    p = nl ? nl + 1 : e;
    if (!c.lit("{\"ev\":\"")) { ch.failed = true; return; }
    if (c.lit("instr\",\"opcode\":")) {
      const char* s; size_t n; uint64_t width;
      if (!c.str(&s, &n) || !c.lit(",\"width\":") || !c.uint(&width) || !c.end() || width == 0 || width >= (1ull << 32)) {
        ch.failed = true; return;
      }
      for (size_t k = 0; k < n; ++k) if ((unsigned char)s[k] >= 0x80) { ch.failed = true; return; }
      std::string key(s, n);
      auto it = ch.opc.find(key);
      uint32_t id;
      if (it == ch.opc.end()) {
        id = (uint32_t)ch.opc_order.size();
        ch.opc.emplace(key, id);
        ch.opc_order.push_back(std::move(key));
      } else {
        id = it->second;
      }
      ch.kind.push_back(AIWC_K_INSTR); ch.pay.push_back(((uint64_t)id << 32) | width);
      ++ch.c_instr;
    } else if (c.lit("mem\",\"op\":\"")) {
      uint8_t k;
      if (c.lit("load\"")) k = AIWC_K_LOAD;
      else if (c.lit("store\"")) k = AIWC_K_STORE;
      else if (c.lit("atomic_load\"")) k = AIWC_K_ATOMIC_LOAD;
      else if (c.lit("atomic_store\"")) k = AIWC_K_ATOMIC_STORE;
      else { ch.failed = true; return; }
      uint64_t addr;
      if (!c.lit(",\"addr\":") || !c.uint(&addr) || !c.end()) { ch.failed = true; return; }
      ch.kind.push_back(k); ch.pay.push_back(addr);
      ch.amin = std::min(ch.amin, addr); ch.amax = std::max(ch.amax, addr); ch.aand &= addr; ch.aor |= addr;
      ++ch.n_mem;
      if (k & 0x02) ++ch.c_rd; else ++ch.c_wr;
    } else if (c.lit("branch\",\"site\":")) {
      uint64_t site; int taken;
      if (!c.uint(&site) || site >= (1ull << 32) || !c.lit(",\"taken\":")) { ch.failed = true; return; }
      if (c.lit("true")) taken = 1;
      else if (c.lit("false")) taken = 0;
      else { ch.failed = true; return; }
      if (!c.end()) { ch.failed = true; return; }
      ch.kind.push_back(AIWC_K_BRANCH); ch.pay.push_back((site << 1) | (uint64_t)taken);
      ++ch.c_br;
    } else if (c.lit("barrier\"")) {
      if (!c.end()) { ch.failed = true; return; }
      ch.kind.push_back(AIWC_K_BARRIER); ch.pay.push_back(0);
      ch.c_bres = 1;
    } else if (c.lit("kernel_end\"")) {
      if (!c.end()) { ch.failed = true; return; }
      ch.kind.push_back(AIWC_K_KERNEL_END); ch.pay.push_back(0);
    } else if (c.lit("wg_")) {
      bool begin;
      if (c.lit("begin\",\"group\":")) begin = true;
      else if (c.lit("end\",\"group\":")) begin = false;
      else { ch.failed = true; return; }
      V3 g;
      if (!c.v3(&g) || !c.end()) { ch.failed = true; return; }
      ch.kind.push_back(begin ? AIWC_K_WG_BEGIN : AIWC_K_WG_END); ch.pay.push_back(gkey(g));
      if (begin) { ch.has_gb = true; ch.last_gb = g; ++ch.c_wgb; }
    } else {
      uint8_t k;
      if (c.lit("wi_begin\"")) k = AIWC_K_WI_BEGIN;
      else if (c.lit("wi_resume\"")) k = AIWC_K_WI_RESUME;
      else if (c.lit("wi_end\"")) k = AIWC_K_WI_END;
      else { ch.failed = true; return; }  // kernel_begin in the body, unknown events: the walker decides
      V3 gid, lid, g;
      if (!c.lit(",\"global\":") || !c.v3(&gid) || !c.lit(",\"local\":") || !c.v3(&lid) || !c.lit(",\"group\":") ||
          !c.v3(&g) || !c.end()) {
        ch.failed = true; return;
      }
      for (int d = 0; d < 3; ++d)  // wi.id_arithmetic (trace.py:406-418): the columns keep only the local id
        if (lid.v[d] >= lsz.v[d] || gid.v[d] != g.v[d] * lsz.v[d] + lid.v[d]) { ch.failed = true; return; }
      // the work-item's group must be the open group: the last wg_begin (in an earlier chunk: checked at the merge)
      if (ch.has_gb) {
        if (!(g == ch.last_gb)) { ch.failed = true; return; }
      } else if (!ch.pre) {
        ch.pre = true; ch.pre_g = g;
      } else if (!(g == ch.pre_g)) {
        ch.pre_mismatch = true;
      }
      ch.kind.push_back(k); ch.pay.push_back((uint64_t)(lid.v[0] + lsz.v[0] * (lid.v[1] + lsz.v[1] * lid.v[2])));
      if (k == AIWC_K_WI_RESUME) ch.c_bres = 1;
    }
  }
}

PyObject* py_encode_lines_fast(PyObject*, PyObject* args) {
  Py_buffer buf;
  int threads;
  if (!PyArg_ParseTuple(args, "y*i", &buf, &threads)) return nullptr;
  const char* b = static_cast<const char*>(buf.buf);
  const char* end = b + buf.len;
  auto none = [&]() { PyBuffer_Release(&buf); Py_RETURN_NONE; };
  if (buf.len == 0) return none();
  // the header: a canonical kernel_begin on line 1
  const char* nl = static_cast<const char*>(memchr(b, '\n', (size_t)(end - b)));
  if (!nl) return none();
  Walker w;
  OpDict d;
  w.opc_dict = PyDict_New();
  w.opc_list = PyList_New(0);
  Rec hr;
  PyObject* tmp[2] = {nullptr, nullptr};
  const int got = parse_canonical(w, d, b, nl, &hr, tmp);
  auto bail = [&]() -> PyObject* {
    Py_XDECREF(tmp[0]); Py_XDECREF(tmp[1]);
    Py_XDECREF(w.opc_dict); Py_XDECREF(w.opc_list);
    PyBuffer_Release(&buf);
    Py_RETURN_NONE;
  };
  if (got != 1 || hr.c != E_KB) { PyErr_Clear(); return bail(); }
  V3 lsz = hr.lsz, grid;
  for (int dd = 0; dd < 3; ++dd) grid.v[dd] = (hr.gsz.v[dd] + lsz.v[dd] - 1) / lsz.v[dd];
  if ((uint64_t)(grid.v[0] * grid.v[1] * grid.v[2]) >= (1ull << 31) || (uint64_t)(lsz.v[0] * lsz.v[1] * lsz.v[2]) >= (1ull << 31))
    return bail();
  // chunks of whole lines
  const char* body = nl + 1;
  const int T = std::max(1, std::min(threads, 64));
  std::vector<const char*> cuts{body};
  for (int t = 1; t < T; ++t) {
    const char* q = body + (end - body) * t / T;
    if (q <= cuts.back()) continue;
    const char* n2 = static_cast<const char*>(memchr(q, '\n', (size_t)(end - q)));
    if (!n2) break;
    if (n2 + 1 > cuts.back() && n2 + 1 < end) cuts.push_back(n2 + 1);
  }
  cuts.push_back(end);
  const size_t C = cuts.size() - 1;
  std::vector<FastChunk> ch(C);
  Py_BEGIN_ALLOW_THREADS
  std::vector<std::thread> th;
  for (size_t i = 0; i < C; ++i) th.emplace_back(parse_chunk, cuts[i], cuts[i + 1], std::cref(lsz), std::cref(grid), &ch[i]);
  for (auto& t : th) t.join();
  Py_END_ALLOW_THREADS
  // a trailing newline leaves an empty last line: the reference's iterator skips nothing else
  bool fail = false;
  bool have_gb = false;
  V3 open_g{};
  for (size_t i = 0; i < C && !fail; ++i) {
    fail = ch[i].failed || ch[i].pre_mismatch || (ch[i].pre && (!have_gb || !(ch[i].pre_g == open_g)));
    if (ch[i].has_gb) { have_gb = true; open_g = ch[i].last_gb; }
  }
  if (fail) return bail();
  // dictionaries in first-appearance order, then the remap of each chunk
  std::unordered_map<std::string, uint64_t>& gop = d.str_ids;
  std::vector<std::vector<uint64_t>> omap(C), xmap(C);
  std::unordered_map<V3, uint64_t, V3Hash> gx;
  std::vector<V3> gx_order;
  const uint64_t n_grid = (uint64_t)(grid.v[0] * grid.v[1] * grid.v[2]);
  for (size_t i = 0; i < C; ++i) {
    for (auto& o : ch[i].opc_order) {
      uint64_t id;
      if (opcode_id_str(w, d, o.data(), o.size(), &id) < 0) { PyErr_Clear(); return bail(); }
      omap[i].push_back(id);
    }
    for (auto& g : ch[i].extra_order) {
      auto it = gx.find(g);
      if (it == gx.end()) { it = gx.emplace(g, n_grid + gx_order.size()).first; gx_order.push_back(g); }
      xmap[i].push_back(it->second);
    }
  }
  (void)gop;
  std::vector<size_t> off(C + 1, 1);
  for (size_t i = 0; i < C; ++i) off[i + 1] = off[i] + ch[i].kind.size();
  const size_t N = off[C];
  PyObject* kinds = PyBytes_FromStringAndSize(nullptr, (Py_ssize_t)N);
  PyObject* pays = PyBytes_FromStringAndSize(nullptr, (Py_ssize_t)(N * 8));
  if (!kinds || !pays) { Py_XDECREF(kinds); Py_XDECREF(pays); return bail(); }
  uint8_t* K = reinterpret_cast<uint8_t*>(PyBytes_AS_STRING(kinds));
  uint64_t* P = reinterpret_cast<uint64_t*>(PyBytes_AS_STRING(pays));
  K[0] = AIWC_K_KERNEL_BEGIN; P[0] = 0;
  Py_BEGIN_ALLOW_THREADS
  std::vector<std::thread> th;
  for (size_t i = 0; i < C; ++i)
    th.emplace_back([&, i]() {
      const FastChunk& c = ch[i];
      uint8_t* k = K + off[i];
      uint64_t* q = P + off[i];
      memcpy(k, c.kind.data(), c.kind.size());
      for (size_t j = 0; j < c.kind.size(); ++j) {
        uint64_t v = c.pay[j];
        if (c.kind[j] == AIWC_K_INSTR) v = (omap[i][v >> 32] << 32) | (v & 0xFFFFFFFFull);
        else if ((c.kind[j] & 0x40) && (v & EXTRA_TAG)) v = xmap[i][v & 0xFFFFFFFFull];
        q[j] = v;
      }
    });
  for (auto& t : th) t.join();
  Py_END_ALLOW_THREADS
  uint64_t amin = ~0ull, amax = 0, aand = ~0ull, aor = 0, n_mem = 0, cnt[6] = {0, 0, 0, 0, 0, 0};
  for (auto& c : ch) {
    if (c.n_mem) { amin = std::min(amin, c.amin); amax = std::max(amax, c.amax); aand &= c.aand; aor |= c.aor; }
    n_mem += c.n_mem;
    cnt[0] += c.c_instr; cnt[1] += c.c_rd; cnt[2] += c.c_wr; cnt[3] += c.c_br; cnt[4] += c.c_wgb;
    cnt[5] |= c.c_bres;
  }
  PyObject* extras = PyList_New((Py_ssize_t)gx_order.size());
  for (size_t k = 0; k < gx_order.size(); ++k)
    PyList_SET_ITEM(extras, k, Py_BuildValue("(LLL)", gx_order[k].v[0], gx_order[k].v[1], gx_order[k].v[2]));
  PyObject* stats = Py_None;
  Py_INCREF(Py_None);
  if (n_mem) {
    Py_DECREF(Py_None);
    stats = Py_BuildValue("(KKKK)", (unsigned long long)amin, (unsigned long long)amax, (unsigned long long)aand,
                          (unsigned long long)aor);
  }
  PyObject* counts = Py_BuildValue("(KKKKKK)", (unsigned long long)cnt[0], (unsigned long long)cnt[1],
                                   (unsigned long long)cnt[2], (unsigned long long)cnt[3], (unsigned long long)cnt[4],
                                   (unsigned long long)cnt[5]);
  PyObject* out = Py_BuildValue("{s:N,s:N,s:O,s:O,s:(LLL),s:(LLL),s:O,s:N,s:N,s:N,s:L}", "kind", kinds, "payload",
                                pays, "kernel_name", hr.name, "invocation", hr.inv, "global_size", hr.gsz.v[0],
                                hr.gsz.v[1], hr.gsz.v[2], "local_size", lsz.v[0], lsz.v[1], lsz.v[2], "opcodes",
                                w.opc_list, "extra_groups", extras, "addr_stats", stats, "counts", counts, "lines",
                                (long long)N);
  Py_XDECREF(tmp[0]); Py_XDECREF(tmp[1]);
  Py_XDECREF(w.opc_dict); Py_XDECREF(w.opc_list);
  PyBuffer_Release(&buf);
  return out;
}

PyObject* py_init(PyObject*, PyObject* args) {
  PyObject* cls;
  if (!PyArg_ParseTuple(args, "O", &cls)) return nullptr;
  Py_XDECREF(g_unsupported);
  Py_INCREF(cls);
  g_unsupported = cls;
  Py_RETURN_NONE;
}

PyMethodDef methods[] = {
    {"encode", py_encode, METH_VARARGS, "encode(iterable) -> dict of columns, dictionaries and first violation"},
    {"encode_lines", py_encode_lines, METH_VARARGS,
     "encode_lines(data, decode_event) -> the same for the lines of an .aiwctrace file"},
    {"validate", py_validate, METH_VARARGS, "validate(iterable) -> [(event_index, rule, detail)] (every violation)"},
    {"encode_lines_fast", py_encode_lines_fast, METH_VARARGS,
     "encode_lines_fast(data, threads) -> columns of an all-canonical .aiwctrace file (unchecked stream) or None"},
    {"init", py_init, METH_VARARGS, "init(UnsupportedTrace class)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_walker", "TraceEvent iterable -> columnar trace", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__walker(void) {
  g_type_cache = PyDict_New();
  return PyModule_Create(&module);
}
