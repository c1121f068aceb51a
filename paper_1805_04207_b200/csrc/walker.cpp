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
#include <cstring>
#include <string>
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
  void push(uint8_t k, uint64_t p) { kind.push_back(k); pay.push_back(p); }
};

int unsupported(const char* msg) {
  PyErr_SetString(g_unsupported ? g_unsupported : PyExc_ValueError, msg);
  return -1;
}

// returns 0 ok, 1 stop (violation), -1 Python error
int feed(Walker& w, PyObject* ev) {
  const long long i = ++w.index;
  const int c = ev_code(ev);
  if (c == E_NONE) {
    PyObject* r = PyObject_Repr(ev);
    PyErr_Format(PyExc_TypeError, "not a trace event: %U", r);
    Py_XDECREF(r);
    return -1;
  }
  if (w.ended) { w.flag(i, "kernel_end.last", "event after kernel_end"); return 1; }
  if (!w.have_header) {
    if (c == E_KB) {
      PyObject* name = PyTuple_GET_ITEM(ev, 0);
      PyObject* inv = PyTuple_GET_ITEM(ev, 1);
      if (!get_v3(PyTuple_GET_ITEM(ev, 2), &w.gsz) || !get_v3(PyTuple_GET_ITEM(ev, 3), &w.lsz))
        return unsupported("kernel_begin sizes must be 3 integers");
      for (int d = 0; d < 3; ++d) {
        if (w.lsz.v[d] <= 0 || w.gsz.v[d] <= 0) return unsupported("launch sizes must be positive");
        w.grid.v[d] = (w.gsz.v[d] + w.lsz.v[d] - 1) / w.lsz.v[d];
      }
      if ((uint64_t)(w.grid.v[0] * w.grid.v[1] * w.grid.v[2]) >= (1ull << 31))
        return unsupported("more than 2^31 work-groups");
      if ((uint64_t)(w.lsz.v[0] * w.lsz.v[1] * w.lsz.v[2]) >= (1ull << 31))
        return unsupported("local size volume >= 2^31");
      Py_INCREF(name); w.kernel_name_obj = name;
      Py_INCREF(inv); w.invocation_obj = inv;
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
        PyObject* op = PyTuple_GET_ITEM(ev, 0);
        uint64_t width;
        if (!get_u64(PyTuple_GET_ITEM(ev, 1), &width) || width >= (1ull << 32))
          return unsupported("instruction width must be an integer in [0, 2^32)");
        PyObject* id = PyDict_GetItemWithError(w.opc_dict, op);
        uint64_t oid;
        if (id) {
          oid = PyLong_AsUnsignedLongLong(id);
        } else {
          if (PyErr_Occurred()) return -1;
          oid = (uint64_t)PyList_GET_SIZE(w.opc_list);
          PyObject* v = PyLong_FromUnsignedLongLong(oid);
          if (PyDict_SetItem(w.opc_dict, op, v) < 0) { Py_DECREF(v); return -1; }
          Py_DECREF(v);
          PyList_Append(w.opc_list, op);
        }
        w.push(AIWC_K_INSTR, (oid << 32) | width);
      } else if (c == E_MEM) {
        PyObject* op = PyTuple_GET_ITEM(ev, 0);
        uint64_t addr;
        if (!get_u64(PyTuple_GET_ITEM(ev, 1), &addr)) return unsupported("memory address must be an integer in [0, 2^64)");
        uint8_t k;
        if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "load") == 0) k = AIWC_K_LOAD;
        else if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "atomic_load") == 0) k = AIWC_K_ATOMIC_LOAD;
        else if (PyUnicode_Check(op) && PyUnicode_CompareWithASCIIString(op, "atomic_store") == 0) k = AIWC_K_ATOMIC_STORE;
        else k = AIWC_K_STORE;  // metrics.py:138: anything not in READ_OPS is a write
        w.push(k, addr);
        w.amin = std::min(w.amin, addr); w.amax = std::max(w.amax, addr);
        w.aand &= addr; w.aor |= addr; ++w.n_mem;
      } else {
        uint64_t site;
        if (!get_u64(PyTuple_GET_ITEM(ev, 0), &site) || site >= (1ull << 32))
          return unsupported("branch site must be an integer in [0, 2^32)");
        const int t = PyObject_IsTrue(PyTuple_GET_ITEM(ev, 1));
        if (t < 0) return -1;
        w.push(AIWC_K_BRANCH, (site << 1) | (uint64_t)t);
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
      V3 g;
      if (!get_v3(PyTuple_GET_ITEM(ev, 0), &g)) return unsupported("group id must be 3 integers");
      w.group_open = true; w.open_group = g;
      w.reset_group();
      w.push(AIWC_K_WG_BEGIN, w.group_key(g));
      return 0;
    }
    case E_WGE: {
      V3 g;
      if (!get_v3(PyTuple_GET_ITEM(ev, 0), &g)) return unsupported("group id must be 3 integers");
      if (!w.group_open || !(g == w.open_group)) { w.flag(i, "wg.nesting", "wg_end does not match open group"); return 1; }
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
      w.push(AIWC_K_WG_END, w.group_key(g));
      return 0;
    }
    default: {  // work-item events
      PyObject* wi = PyTuple_GET_ITEM(ev, 0);
      if (!PyTuple_Check(wi) || PyTuple_GET_SIZE(wi) != 3) return unsupported("work_item must be a WorkItemId");
      V3 gid, lid, grp;
      if (!get_v3(PyTuple_GET_ITEM(wi, 0), &gid) || !get_v3(PyTuple_GET_ITEM(wi, 1), &lid) ||
          !get_v3(PyTuple_GET_ITEM(wi, 2), &grp))
        return unsupported("work-item ids must be 3 integers");
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

PyObject* py_encode(PyObject*, PyObject* args) {
  PyObject* iterable;
  if (!PyArg_ParseTuple(args, "O", &iterable)) return nullptr;
  PyObject* it = PyObject_GetIter(iterable);
  if (!it) return nullptr;
  Walker w;
  w.opc_dict = PyDict_New();
  w.opc_list = PyList_New(0);
  int rc = 0;
  PyObject* ev;
  while ((ev = PyIter_Next(it))) {
    rc = feed(w, ev);
    Py_DECREF(ev);
    if (rc) break;
  }
  Py_DECREF(it);
  auto cleanup = [&]() {
    Py_XDECREF(w.opc_dict); Py_XDECREF(w.opc_list);
    Py_XDECREF(w.kernel_name_obj); Py_XDECREF(w.invocation_obj);
  };
  if (rc < 0 || PyErr_Occurred()) { cleanup(); return nullptr; }
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
  PyObject* out = Py_BuildValue("{s:N,s:N,s:O,s:O,s:(LLL),s:(LLL),s:O,s:N,s:N,s:N,s:O}", "kind", kinds, "payload", pays,
                                "kernel_name", name, "invocation", inv, "global_size", w.gsz.v[0], w.gsz.v[1],
                                w.gsz.v[2], "local_size", w.lsz.v[0], w.lsz.v[1], w.lsz.v[2], "opcodes", w.opc_list,
                                "extra_groups", extras, "addr_stats", stats, "violation", violation, "have_header",
                                w.have_header ? Py_True : Py_False);
  cleanup();
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
    {"init", py_init, METH_VARARGS, "init(UnsupportedTrace class)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_walker", "TraceEvent iterable -> columnar trace", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__walker(void) {
  g_type_cache = PyDict_New();
  return PyModule_Create(&module);
}
