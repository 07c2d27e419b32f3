/* hostenc.c - native host-side encoding of foreign ScheduleState objects
 * (the reference's own states, handed to the V-callable, search.py:3-8) into
 * the 16-byte ts_decision records of the C-ABI.
 *
 * schedule_space.encode_states spent its time in Python per decision.  Here
 * one C call walks a group of states: a state that already carries its
 * records (state._cache["ts_records"], featurizer.py:72-73's cache idiom)
 * is copied; otherwise every decision object is looked up by identity in an
 * open-addressing table (pointer -> schedule index + record; the table holds
 * a reference, so the pointer stays valid); an unseen object is looked up by
 * value ((index, its seven fields) -> record: the same action built again by
 * candidate_actions) in the pipeline's own value dict (_PipelineInfo.val_cache,
 * filled by the Python encoder), and only unseen values call back into Python
 * (_PipelineInfo.encode: validation + encoding) - unless the pipeline's
 * stage table is given, in which case the common case (a legal decision with
 * plain int / str / tuple fields) is validated and packed here
 * (encode_native, the same checks and layout as _PipelineInfo._encode_fields,
 * schedule_space.py) and anything it does not accept goes to the Python
 * encoder, which raises the reference's error.  Both caches are per
 * pipeline: a record depends on the stage's loop table and its sole consumer,
 * so the same (index, fields) can encode differently - or be illegal - in
 * another pipeline.  Identity slots carry their owner (the value dict).  Search
 * children share all but their last decision object with their parent, so a
 * child costs one identity probe per decision and one value lookup.
 *
 * Module _hostenc (CPython C API, built in-tree by build.py):
 *   encode_group(states, idxs, T, fallback, vcache[, stab]) -> (records: bytes, offsets: bytes [int64 n+1])
 *     stab: per schedule index (stage name, pure dim names, reduction dim
 *     names, sole consumer name or None), or None for a stage whose loop
 *     names could collide (always the Python encoder)
 *   clear() -> None   (drop the identity table)
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  PyObject* obj;   /* strong reference; NULL = empty slot */
  PyObject* owner; /* strong reference: the pipeline's value dict */
  int32_t idx;
  uint8_t rec[16];
} Slot;

#define CAP_LOG2 18
#define CAP (1u << CAP_LOG2)
static Slot* table = NULL;
static size_t used = 0;
static PyObject* s_cache = NULL;   /* "_cache" */
static PyObject* s_records = NULL; /* "ts_records" */
static PyObject* s_decisions = NULL;
/* decision fields: the value key of a decision object (its dataclass fields,
 * search.py / schedule_space.py LayerSchedule) */
static PyObject* s_fields[7] = {NULL};
static const char* field_names[7] = {"stage", "splits", "order", "vectorize_width", "parallel", "compute_at",
                                     "store_at"};

static void table_clear(void) {
  if (!table) return;
  for (size_t i = 0; i < CAP; ++i) {
    if (table[i].obj) {
      Py_DECREF(table[i].obj);
      Py_DECREF(table[i].owner);
      table[i].obj = NULL;
      table[i].owner = NULL;
    }
  }
  used = 0;
}

static inline size_t slot_of(const void* p, const void* owner) {
  uint64_t h = (uint64_t)(uintptr_t)p ^ ((uint64_t)(uintptr_t)owner << 7);
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  return (size_t)(h & (CAP - 1));
}

/* UTF-8 view of a str (cached in the object); NULL (no error set) otherwise */
static const char* utf8(PyObject* o, Py_ssize_t* n) {
  if (!PyUnicode_Check(o)) return NULL;
  const char* c = PyUnicode_AsUTF8AndSize(o, n);
  if (!c) PyErr_Clear();
  return c;
}

/* exact int in [lo, hi] (bool and other int subclasses: not accepted) */
static int small_int(PyObject* o, long lo, long hi, long* v) {
  if (!PyLong_CheckExact(o)) return 0;
  int ovf = 0;
  const long x = PyLong_AsLongAndOverflow(o, &ovf);
  if (ovf || (x == -1 && PyErr_Occurred())) {
    PyErr_Clear();
    return 0;
  }
  if (x < lo || x > hi) return 0;
  *v = x;
  return 1;
}

/* The 16-byte record of a legal decision from its fields (f[0..6]: stage,
 * splits, order, vectorize_width, parallel, compute_at, store_at) and its
 * stage's entry (name, pure, red, sole): split[4], order[8], n_loops, vec,
 * flags, anchor - the checks and packing of _encode_fields.  1 = packed,
 * 0 = not accepted here (the Python encoder decides), -1 = error. */
static int encode_native(PyObject* const* f, PyObject* ent, uint8_t* out) {
  if (!PyTuple_Check(ent) || PyTuple_GET_SIZE(ent) != 4) return 0;
  PyObject *name = PyTuple_GET_ITEM(ent, 0), *pure = PyTuple_GET_ITEM(ent, 1), *red = PyTuple_GET_ITEM(ent, 2),
           *sole = PyTuple_GET_ITEM(ent, 3);
  if (!PyTuple_Check(pure) || !PyTuple_Check(red)) return 0;
  const Py_ssize_t np_ = PyTuple_GET_SIZE(pure), nr = PyTuple_GET_SIZE(red);
  if (np_ < 1 || np_ > 4 || nr > 4) return 0;
  const char* pn[4];
  Py_ssize_t pl[4];
  for (Py_ssize_t k = 0; k < np_; ++k)
    if (!(pn[k] = utf8(PyTuple_GET_ITEM(pure, k), &pl[k]))) return 0;
  /* stage */
  PyObject* stage = f[0];
  if (!PyUnicode_Check(stage) || !PyUnicode_Check(name)) return 0;
  if (stage != name) {
    const int c = PyUnicode_Compare(stage, name);
    if (c == -1 && PyErr_Occurred()) return -1;
    if (c != 0) return 0;
  }
  memset(out, 0, 16);
  /* splits: ((dim, factor), ...), each pure dim at most once, 2 <= f <= 255 */
  unsigned split_mask = 0;
  {
    PyObject* sq = PySequence_Fast(f[1], "");
    if (!sq) {
      PyErr_Clear();
      return 0;
    }
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(sq);
    PyObject* const* it = PySequence_Fast_ITEMS(sq);
    int ok = 1;
    for (Py_ssize_t i = 0; ok && i < n; ++i) {
      PyObject* pr = it[i];
      if (!PyTuple_Check(pr) || PyTuple_GET_SIZE(pr) != 2) {
        ok = 0;
        break;
      }
      Py_ssize_t dl;
      const char* dn = utf8(PyTuple_GET_ITEM(pr, 0), &dl);
      long f;
      if (!dn || !small_int(PyTuple_GET_ITEM(pr, 1), 2, 255, &f)) {
        ok = 0;
        break;
      }
      int k = -1;
      for (Py_ssize_t q = 0; q < np_; ++q)
        if (pl[q] == dl && !memcmp(pn[q], dn, (size_t)dl)) k = (int)q;
      if (k < 0 || (split_mask >> k & 1u)) ok = 0;
      else {
        split_mask |= 1u << k;
        out[k] = (uint8_t)f;
      }
    }
    Py_DECREF(sq);
    if (!ok) return 0;
  }
  /* order: a permutation of the loop table's names */
  {
    PyObject* oq = PySequence_Fast(f[2], "");
    if (!oq) {
      PyErr_Clear();
      return 0;
    }
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(oq);
    Py_ssize_t n_table = np_ + nr;
    for (Py_ssize_t k = 0; k < np_; ++k) n_table += split_mask >> k & 1u;
    int ok = n == n_table && n <= 8;
    unsigned seen = 0;
    PyObject* const* it = PySequence_Fast_ITEMS(oq);
    for (Py_ssize_t i = 0; ok && i < n; ++i) {
      Py_ssize_t l;
      const char* c = utf8(it[i], &l);
      int code = -1;
      if (c) {
        for (Py_ssize_t k = 0; code < 0 && k < np_; ++k) {
          if (split_mask >> k & 1u) {
            if (l == pl[k] + 1 && !memcmp(c, pn[k], (size_t)pl[k]) && (c[l - 1] == 'o' || c[l - 1] == 'i'))
              code = 2 * (int)k + (c[l - 1] == 'i');
          } else if (l == pl[k] && !memcmp(c, pn[k], (size_t)l)) {
            code = 2 * (int)k;
          }
        }
        for (Py_ssize_t r = 0; code < 0 && r < nr; ++r) {
          Py_ssize_t rl;
          const char* rn = utf8(PyTuple_GET_ITEM(red, r), &rl);
          if (rn && rl == l && !memcmp(rn, c, (size_t)l)) code = 8 + (int)r;
        }
      }
      if (code < 0 || (seen >> code & 1u)) ok = 0;
      else {
        seen |= 1u << code;
        out[4 + i] = (uint8_t)code;
      }
    }
    for (Py_ssize_t i = n; ok && i < 8; ++i) out[4 + i] = 0xFF;
    Py_DECREF(oq);
    if (!ok) return 0;
    out[12] = (uint8_t)n;
  }
  long vw;
  if (!small_int(f[3], 1, 255, &vw)) return 0;
  out[13] = (uint8_t)vw;
  const int par = PyObject_IsTrue(f[4]);
  if (par < 0) {
    PyErr_Clear();
    return 0;
  }
  uint8_t flags = par ? 1 : 0; /* FLAG_PARALLEL */
  PyObject *cat = f[5], *sat = f[6];
  int8_t anchor = -1;
  if (cat == Py_None) {
    if (sat != Py_None) return 0;
  } else {
    if (!PyTuple_Check(cat) || PyTuple_GET_SIZE(cat) != 2 || sole == Py_None || !PyUnicode_Check(sole))
      return 0;
    PyObject* cname = PyTuple_GET_ITEM(cat, 0);
    if (!PyUnicode_Check(cname)) return 0;
    const int c = PyUnicode_Compare(cname, sole);
    if (c == -1 && PyErr_Occurred()) return -1;
    long lvl;
    if (c != 0 || !small_int(PyTuple_GET_ITEM(cat, 1), 0, 7, &lvl)) return 0;
    anchor = (int8_t)lvl;
    if (sat != Py_None) {
      const int eq = PyObject_RichCompareBool(sat, cat, Py_EQ);
      if (eq < 0) {
        PyErr_Clear();
        return 0;
      }
      if (!eq) return 0;
      flags |= 2; /* FLAG_STORE_AT */
    }
  }
  out[14] = flags;
  out[15] = (uint8_t)anchor;
  return 1;
}

/* identity slot for d (held: its pointer stays valid while cached) */
static void remember(PyObject* d, int j, PyObject* vcache, const uint8_t* rec) {
  if (used >= CAP / 2) table_clear(); /* bounded: foreign callers bring new objects */
  size_t s = slot_of(d, vcache);
  while (table[s].obj) s = (s + 1) & (CAP - 1);
  Py_INCREF(d);
  Py_INCREF(vcache);
  table[s].obj = d;
  table[s].owner = vcache;
  table[s].idx = j;
  memcpy(table[s].rec, rec, 16);
  ++used;
}

/* record of decision d at schedule index j of the pipeline whose value dict
 * is vcache: table hit, native encoding, value hit or Python fallback */
static int record_of(PyObject* d, int j, PyObject* fallback, PyObject* vcache, PyObject* stab, uint8_t* out) {
  size_t s = slot_of(d, vcache);
  for (;;) {
    Slot* e = &table[s];
    if (!e->obj) break;
    if (e->obj == d && e->idx == j && e->owner == vcache) {
      memcpy(out, e->rec, 16);
      return 0;
    }
    s = (s + 1) & (CAP - 1);
  }
  /* a new object of a legal value: validated and packed here, no value
   * lookup (hashing the nested field tuples costs more than encoding) */
  if (stab != Py_None && PyTuple_GET_ITEM(stab, j) != Py_None) {
    PyObject* f[7];
    int nf = 0;
    for (; nf < 7; ++nf)
      if (!(f[nf] = PyObject_GetAttr(d, s_fields[nf]))) {
        PyErr_Clear();
        break;
      }
    int ok = 0;
    if (nf == 7) ok = encode_native(f, PyTuple_GET_ITEM(stab, j), out);
    for (int q = 0; q < nf; ++q) Py_DECREF(f[q]);
    if (ok < 0) return -1;
    if (ok) {
      remember(d, j, vcache, out);
      return 0;
    }
  }
  PyObject* jj = PyLong_FromLong(j); /* a cached small int */
  if (!jj) return -1;
  /* a new object: look its value up (a decision equal to one already
   * encoded at this index - candidate_actions builds new objects for the
   * same actions), else the Python encoder validates and encodes it */
  PyObject* key = PyTuple_New(8);
  if (!key) {
    Py_DECREF(jj);
    return -1;
  }
  Py_INCREF(jj);
  PyTuple_SET_ITEM(key, 0, jj);
  int have_key = 1;
  for (int f = 0; f < 7; ++f) {
    PyObject* v = PyObject_GetAttr(d, s_fields[f]);
    if (!v) { /* not decision-like: the fallback reports it */
      PyErr_Clear();
      have_key = 0;
      break;
    }
    PyTuple_SET_ITEM(key, 1 + f, v);
  }
  PyObject* r = NULL;
  if (have_key) {
    r = PyDict_GetItemWithError(vcache, key); /* borrowed */
    if (r) {
      Py_INCREF(r);
    } else if (PyErr_Occurred()) { /* unhashable fields: the fallback decides */
      PyErr_Clear();
      have_key = 0;
    }
  }
  if (!r) {
    PyObject* argv[2] = {jj, d}; /* fills vcache itself */
    r = PyObject_Vectorcall(fallback, argv, 2, NULL);
  }
  Py_DECREF(key);
  Py_DECREF(jj);
  if (!r) return -1;
  if (!PyBytes_Check(r) || PyBytes_GET_SIZE(r) != 16) {
    Py_DECREF(r);
    PyErr_SetString(PyExc_TypeError, "encode fallback must return 16 bytes");
    return -1;
  }
  memcpy(out, PyBytes_AS_STRING(r), 16);
  Py_DECREF(r);
  remember(d, j, vcache, out);
  return 0;
}

static PyObject* encode_group(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *states, *idxs, *fallback, *vcache, *stab = Py_None;
  Py_ssize_t T;
  if (!PyArg_ParseTuple(args, "OOnOO!|O", &states, &idxs, &T, &fallback, &PyDict_Type, &vcache, &stab)) return NULL;
  if (stab != Py_None && (!PyTuple_Check(stab) || PyTuple_GET_SIZE(stab) != T)) {
    PyErr_SetString(PyExc_TypeError, "stage table must be a tuple of T entries or None");
    return NULL;
  }
  if (!table) {
    table = (Slot*)PyMem_Calloc(CAP, sizeof(Slot));
    if (!table) return PyErr_NoMemory();
  }
  PyObject* sq = PySequence_Fast(states, "states must be a sequence");
  if (!sq) return NULL;
  PyObject* iq = PySequence_Fast(idxs, "indices must be a sequence");
  if (!iq) {
    Py_DECREF(sq);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(iq);
  PyObject* offs = PyBytes_FromStringAndSize(NULL, (n + 1) * (Py_ssize_t)sizeof(int64_t));
  Py_ssize_t cap = n * 20 + 16, len = 0;
  uint8_t* buf = (uint8_t*)PyMem_Malloc((size_t)cap * 16);
  if (!offs || !buf) {
    Py_XDECREF(offs);
    PyMem_Free(buf);
    Py_DECREF(sq);
    Py_DECREF(iq);
    return PyErr_NoMemory();
  }
  int64_t* off = (int64_t*)PyBytes_AS_STRING(offs);
  off[0] = 0;
  PyObject* const* sv = PySequence_Fast_ITEMS(sq);
  const Py_ssize_t ns = PySequence_Fast_GET_SIZE(sq);
  for (Py_ssize_t q = 0; q < n; ++q) {
    const Py_ssize_t i = PyLong_AsSsize_t(PySequence_Fast_GET_ITEM(iq, q));
    if (i < 0 || i >= ns) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_IndexError, "state index out of range");
      goto fail;
    }
    PyObject* st = sv[i];
    /* a state carrying its records (state._cache["ts_records"]) */
    PyObject* cache = PyObject_GetAttr(st, s_cache);
    if (!cache) PyErr_Clear();
    if (cache && PyDict_Check(cache)) {
      PyObject* hit = PyDict_GetItemWithError(cache, s_records); /* borrowed */
      if (hit && PyBytes_Check(hit) && PyBytes_GET_SIZE(hit) % 16 == 0) {
        const Py_ssize_t m = PyBytes_GET_SIZE(hit) / 16;
        if (m > T) {
          Py_DECREF(cache);
          PyErr_SetString(PyExc_ValueError, "state has more decisions than stages");
          goto fail;
        }
        if (len + m > cap) {
          cap = 2 * (len + m) + 16;
          uint8_t* nb = (uint8_t*)PyMem_Realloc(buf, (size_t)cap * 16);
          if (!nb) {
            Py_DECREF(cache);
            PyErr_NoMemory();
            goto fail;
          }
          buf = nb;
        }
        memcpy(buf + len * 16, PyBytes_AS_STRING(hit), (size_t)m * 16);
        len += m;
        off[q + 1] = len;
        Py_DECREF(cache);
        continue;
      }
      if (PyErr_Occurred()) {
        Py_DECREF(cache);
        goto fail;
      }
    }
    PyObject* dec = PyObject_GetAttr(st, s_decisions);
    if (!dec) {
      Py_XDECREF(cache);
      goto fail;
    }
    PyObject* dq = PySequence_Fast(dec, "decisions must be a sequence");
    Py_DECREF(dec);
    if (!dq) {
      Py_XDECREF(cache);
      goto fail;
    }
    const Py_ssize_t m = PySequence_Fast_GET_SIZE(dq);
    if (m > T) {
      Py_DECREF(dq);
      Py_XDECREF(cache);
      PyErr_SetString(PyExc_ValueError, "state has more decisions than stages");
      goto fail;
    }
    if (len + m > cap) {
      cap = 2 * (len + m) + 16;
      uint8_t* nb = (uint8_t*)PyMem_Realloc(buf, (size_t)cap * 16);
      if (!nb) {
        Py_DECREF(dq);
        Py_XDECREF(cache);
        PyErr_NoMemory();
        goto fail;
      }
      buf = nb;
    }
    PyObject* const* dv = PySequence_Fast_ITEMS(dq);
    for (Py_ssize_t j = 0; j < m; ++j) {
      if (record_of(dv[j], (int)j, fallback, vcache, stab, buf + (len + j) * 16)) {
        Py_DECREF(dq);
        Py_XDECREF(cache);
        goto fail;
      }
    }
    if (cache && PyDict_Check(cache)) { /* cache the records on the state, like records_of */
      PyObject* rb = PyBytes_FromStringAndSize((const char*)(buf + len * 16), m * 16);
      if (!rb || PyDict_SetItem(cache, s_records, rb) < 0) {
        Py_XDECREF(rb);
        Py_DECREF(dq);
        Py_DECREF(cache);
        goto fail;
      }
      Py_DECREF(rb);
    }
    Py_XDECREF(cache);
    Py_DECREF(dq);
    len += m;
    off[q + 1] = len;
  }
  Py_DECREF(sq);
  Py_DECREF(iq);
  PyObject* recs = PyBytes_FromStringAndSize((const char*)buf, len * 16);
  PyMem_Free(buf);
  if (!recs) {
    Py_DECREF(offs);
    return NULL;
  }
  PyObject* res = PyTuple_Pack(2, recs, offs);
  Py_DECREF(recs);
  Py_DECREF(offs);
  return res;
fail:
  Py_DECREF(sq);
  Py_DECREF(iq);
  Py_DECREF(offs);
  PyMem_Free(buf);
  return NULL;
}

static PyObject* clear(PyObject* self, PyObject* args) {
  (void)self;
  (void)args;
  table_clear();
  Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"encode_group", encode_group, METH_VARARGS, "records + offsets of states[idxs] (see hostenc.c)"},
    {"clear", clear, METH_NOARGS, "drop the decision identity table"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostenc", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostenc(void) {
  s_cache = PyUnicode_InternFromString("_cache");
  s_records = PyUnicode_InternFromString("ts_records");
  s_decisions = PyUnicode_InternFromString("decisions");
  if (!s_cache || !s_records || !s_decisions) return NULL;
  for (int f = 0; f < 7; ++f)
    if (!(s_fields[f] = PyUnicode_InternFromString(field_names[f]))) return NULL;
  return PyModule_Create(&module);
}
