// _fvhost: the batch front end's two per-row host loops as a CPython
// extension, so a 1e8-row call is not dominated by them
// once the solvers run on the device:
//
//   parse_flags_u(arr)          batch.py:78-88 parse_flags on a numpy 'U' array:
//                               case-insensitive 'c' / 'p' -> int8 +1 / -1.
//                               Returns (flags, first_bad) with first_bad = -1
//                               or the lowest index of an element that is not
//                               exactly one of c C p P (the caller raises
//                               BadFlag for it, as the reference does).
//   status_objects(names, codes) batch.py:217/:259 status column: an object
//                               array with element i = names[codes[i]] (the
//                               same str objects, so the same values and dtype
//                               as np.array(names, dtype=object)[codes]).
//
// Both run over the rows on several threads with the GIL released.  The
// object array is allocated through the numpy C API (zero-filled, no None
// pass) and its pointers are written by the threads; each name's reference
// count is then raised by its number of occurrences under the GIL (a no-op
// for immortal objects).
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

namespace {

const int64_t kRowsPerThread = 1 << 20;

template <class F>
void par_rows(int64_t n, F fn) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt > 16) nt = 16;
  int64_t parts = n / kRowsPerThread;
  if (parts > (int64_t)nt) parts = nt;
  if (parts < 2) { fn(0, 0, n); return; }
  const int64_t per = (n + parts - 1) / parts;
  std::vector<std::thread> th;
  for (int64_t k = 1; k < parts; ++k) {
    const int64_t a = k * per, b = std::min(n, a + per);
    if (a >= b) break;
    th.emplace_back([=] { fn((int)k, a, b); });
  }
  fn(0, 0, std::min(n, per));
  for (auto& t : th) t.join();
}

PyObject* parse_flags_u(PyObject*, PyObject* args) {
  PyArrayObject* arr;
  if (!PyArg_ParseTuple(args, "O!", &PyArray_Type, &arr)) return nullptr;
  if (PyArray_NDIM(arr) != 1 || PyArray_TYPE(arr) != NPY_UNICODE || !PyArray_IS_C_CONTIGUOUS(arr)) {
    PyErr_SetString(PyExc_TypeError, "parse_flags_u: 1-d C-contiguous numpy 'U' array expected");
    return nullptr;
  }
  const int64_t n = PyArray_DIM(arr, 0);
  const int64_t width = PyArray_ITEMSIZE(arr) / 4;      // UCS-4 code points per element
  npy_intp dims[1] = {(npy_intp)n};
  PyArrayObject* out = (PyArrayObject*)PyArray_SimpleNew(1, dims, NPY_INT8);
  if (!out) return nullptr;
  const uint32_t* cp = (const uint32_t*)PyArray_DATA(arr);
  int8_t* o = (int8_t*)PyArray_DATA(out);
  std::vector<int64_t> first(17, -1);
  Py_BEGIN_ALLOW_THREADS
  par_rows(n, [&](int k, int64_t a, int64_t b) {
    int64_t bad = -1;
    for (int64_t i = a; i < b; ++i) {
      const uint32_t* e = cp + i * width;
      const uint32_t low = e[0] | 0x20u;
      bool ok = (low == 0x63u || low == 0x70u);
      for (int64_t j = 1; j < width; ++j) ok = ok && e[j] == 0;
      o[i] = (int8_t)(low == 0x63u ? 1 : -1);
      if (!ok) { bad = i; break; }
    }
    first[k] = bad;
  });
  Py_END_ALLOW_THREADS
  int64_t bad = -1;
  for (int64_t v : first)
    if (v >= 0 && (bad < 0 || v < bad)) bad = v;
  return Py_BuildValue("NL", (PyObject*)out, (long long)bad);
}

PyObject* status_objects(PyObject*, PyObject* args) {
  PyObject* names;
  PyArrayObject* codes;
  if (!PyArg_ParseTuple(args, "O!O!", &PyTuple_Type, &names, &PyArray_Type, &codes)) return nullptr;
  if (PyArray_NDIM(codes) != 1 || PyArray_TYPE(codes) != NPY_INT8 || !PyArray_IS_C_CONTIGUOUS(codes)) {
    PyErr_SetString(PyExc_TypeError, "status_objects: 1-d C-contiguous int8 codes expected");
    return nullptr;
  }
  const Py_ssize_t m = PyTuple_GET_SIZE(names);
  if (m < 1 || m > 127) {
    PyErr_SetString(PyExc_ValueError, "status_objects: 1..127 names expected");
    return nullptr;
  }
  std::vector<PyObject*> tab(m);
  for (Py_ssize_t j = 0; j < m; ++j) tab[j] = PyTuple_GET_ITEM(names, j);
  const int64_t n = PyArray_DIM(codes, 0);
  npy_intp dims[1] = {(npy_intp)n};
  // PyArray_SimpleNew zero-fills object arrays (NPY_NEEDS_INIT); every slot
  // is written below before the array is returned
  PyArrayObject* out = (PyArrayObject*)PyArray_SimpleNew(1, dims, NPY_OBJECT);
  if (!out) return nullptr;
  const int8_t* c = (const int8_t*)PyArray_DATA(codes);
  PyObject** o = (PyObject**)PyArray_DATA(out);
  std::vector<std::vector<int64_t>> counts(17, std::vector<int64_t>(m, 0));
  std::vector<int64_t> first_bad(17, -1);
  Py_BEGIN_ALLOW_THREADS
  par_rows(n, [&](int k, int64_t a, int64_t b) {
    int64_t* cnt = counts[k].data();
    for (int64_t i = a; i < b; ++i) {
      const int8_t v = c[i];
      if (v < 0 || v >= m) { first_bad[k] = i; for (int64_t j = i; j < b; ++j) o[j] = tab[0]; cnt[0] += b - i; break; }
      o[i] = tab[v];
      ++cnt[v];
    }
  });
  Py_END_ALLOW_THREADS
  for (Py_ssize_t j = 0; j < m; ++j) {
    int64_t total = 0;
    for (auto& v : counts) total += v[j];
    if (total) Py_SET_REFCNT(tab[j], Py_REFCNT(tab[j]) + total);   // ignored for immortal objects
  }
  for (int64_t v : first_bad) {
    if (v >= 0) {
      Py_DECREF(out);
      PyErr_Format(PyExc_ValueError, "status_objects: code out of range at row %lld", (long long)v);
      return nullptr;
    }
  }
  return (PyObject*)out;
}

PyMethodDef kMethods[] = {
    {"parse_flags_u", parse_flags_u, METH_VARARGS, "case-insensitive c/p -> int8 +1/-1; (flags, first_bad)"},
    {"status_objects", status_objects, METH_VARARGS, "object array names[codes]"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_fvhost", "fastvol_b200 batch front-end host loops", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__fvhost(void) {
  import_array();
  return PyModule_Create(&kModule);
}
