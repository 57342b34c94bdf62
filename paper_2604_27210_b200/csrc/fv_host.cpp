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

#include <errno.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <memory>
#include <string>
#include <thread>
#include <vector>

namespace {

// rows per host thread: a thread costs ~30-50 us to start, a row ~1-3 ns, so
// a 1M-row column (the reference bench harness's size) already splits 8 ways
const int64_t kRowsPerThread = 1 << 17;

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
    if (width == 1) {                          // 'U1': a branch-free pass, then the first bad row if any
      uint32_t any_bad = 0;
      for (int64_t i = a; i < b; ++i) {
        const uint32_t low = cp[i] | 0x20u;
        o[i] = (int8_t)(low == 0x63u ? 1 : -1);
        any_bad |= (uint32_t)(low != 0x63u) & (uint32_t)(low != 0x70u);
      }
      if (any_bad)
        for (int64_t i = a; i < b; ++i) {
          const uint32_t low = cp[i] | 0x20u;
          if (low != 0x63u && low != 0x70u) { bad = i; break; }
        }
      first[k] = bad;
      return;
    }
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

// ---- CSV serialisation (batch.py:287-306 format_output(table, "csv")) -------
// Cell text: float columns -> repr(float(v)) (shortest round trip), integer
// columns -> 'c' if v > 0 else 'p', str objects -> the string itself.  The
// shortest digits come from std::to_chars (C++17: the shortest string that
// round-trips, nearest to the value on ties -- the digits of CPython's
// repr); the layout is CPython's float_repr_style 'short' rule: positional
// when -4 < decpt <= 16, else d[.ddd]e+XX with at least two exponent digits.
int repr_double(double v, char* out) {
  if (v != v) { memcpy(out, "nan", 3); return 3; }
  char buf[40];
  auto res = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  const char* p = buf;
  const char* end = res.ptr;
  int o = 0;
  if (*p == '-') { out[o++] = '-'; ++p; }
  if (*p == 'i') { memcpy(out + o, "inf", 3); return o + 3; }
  char dig[24];
  int nd = 0;
  while (p < end && *p != 'e') { if (*p != '.') dig[nd++] = *p; ++p; }
  int e10 = 0;
  if (p < end) {                                   // 'e' [+-] digits
    ++p;
    const bool neg = *p == '-';
    ++p;
    while (p < end) e10 = e10 * 10 + (*p++ - '0');
    if (neg) e10 = -e10;
  }
  const int decpt = e10 + 1;                       // value = 0.d1d2... x 10^decpt
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      out[o++] = '0'; out[o++] = '.';
      for (int i = 0; i < -decpt; ++i) out[o++] = '0';
      memcpy(out + o, dig, nd); o += nd;
    } else if (decpt < nd) {
      memcpy(out + o, dig, decpt); o += decpt;
      out[o++] = '.';
      memcpy(out + o, dig + decpt, nd - decpt); o += nd - decpt;
    } else {
      memcpy(out + o, dig, nd); o += nd;
      for (int i = nd; i < decpt; ++i) out[o++] = '0';
      out[o++] = '.'; out[o++] = '0';
    }
    return o;
  }
  out[o++] = dig[0];
  if (nd > 1) { out[o++] = '.'; memcpy(out + o, dig + 1, nd - 1); o += nd - 1; }
  out[o++] = 'e';
  int x = decpt - 1;
  out[o++] = x < 0 ? '-' : '+';
  if (x < 0) x = -x;
  char xe[8];
  int nx = 0;
  do { xe[nx++] = (char)('0' + x % 10); x /= 10; } while (x);
  if (nx < 2) xe[nx++] = '0';
  while (nx) out[o++] = xe[--nx];
  return o;
}

PyObject* repr_doubles(PyObject*, PyObject* args) {       // test hook: list of repr strings
  PyArrayObject* arr;
  if (!PyArg_ParseTuple(args, "O!", &PyArray_Type, &arr)) return nullptr;
  if (PyArray_NDIM(arr) != 1 || PyArray_TYPE(arr) != NPY_FLOAT64) {
    PyErr_SetString(PyExc_TypeError, "repr_doubles: 1-d float64 array expected");
    return nullptr;
  }
  const int64_t n = PyArray_DIM(arr, 0);
  PyObject* lst = PyList_New(n);
  if (!lst) return nullptr;
  char buf[48];
  for (int64_t i = 0; i < n; ++i) {
    const double v = *(const double*)PyArray_GETPTR1(arr, i);
    const int k = repr_double(v, buf);
    PyList_SET_ITEM(lst, i, PyUnicode_FromStringAndSize(buf, k));
  }
  return lst;
}

enum ColKind { COL_F64, COL_INT, COL_STR };
struct CsvCol {
  ColKind kind;
  const char* base;
  int64_t stride;          // bytes
  int isize;               // integer item size
  bool is_signed;
  std::vector<PyObject*> objs;          // COL_STR: distinct objects ...
  std::vector<std::string> text;        // ... and their UTF-8
  size_t maxlen = 0;                    // longest text
};

// ---- threaded text output ---------------------------------------------------
// Workers for `work` units with at least `min_per` units each (<= 16).
int parts_for(int64_t work, int64_t min_per) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt > 16) nt = 16;
  if (nt < 1) nt = 1;
  int64_t p = work / min_per;
  if (p > (int64_t)nt) p = nt;
  if (p < 1) p = 1;
  return (int)p;
}
template <class F>
void run_parts(int parts, F fn) {
  std::vector<std::thread> th;
  for (int k = 1; k < parts; ++k) th.emplace_back(fn, k);
  fn(0);
  for (auto& t : th) t.join();
}
// A growable byte buffer written through a raw pointer: reserve() the bound
// of the next record, then append with put()/ptr (no per-character capacity
// checks; the std::string appends of the first form ran at ~250 MB/s).
struct OutBuf {
  std::unique_ptr<char[]> b;
  size_t cap = 0, n = 0;
  void reserve(size_t more) {
    if (n + more <= cap) return;
    size_t nc = cap ? cap : 1 << 16;
    while (nc < n + more) nc *= 2;
    std::unique_ptr<char[]> nb(new char[nc]);
    if (n) memcpy(nb.get(), b.get(), n);
    b.swap(nb);
    cap = nc;
  }
  char* ptr() { return b.get() + n; }
  void put(const char* p, size_t k) { memcpy(b.get() + n, p, k); n += k; }
  void put(char c) { b[n++] = c; }
};
bool ascii_text(const char* p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if ((unsigned char)p[i] >= 0x80) return false;
  return true;
}
// The pieces, in order, as one str: ASCII text becomes a compact 1-byte
// PyUnicode filled by parallel copies (no concatenated copy, no UTF-8
// decode pass); anything else goes through the UTF-8 decoder.
PyObject* str_from_pieces(const std::vector<std::pair<const char*, size_t>>& pcs, bool ascii) {
  size_t total = 0;
  for (auto& pc : pcs) total += pc.second;
  if (!ascii) {
    std::string all;
    all.reserve(total);
    for (auto& pc : pcs) all.append(pc.first, pc.second);
    return PyUnicode_DecodeUTF8(all.data(), (Py_ssize_t)all.size(), "strict");
  }
  PyObject* out = PyUnicode_New((Py_ssize_t)total, 127);
  if (!out) return nullptr;
  char* dst = (char*)PyUnicode_1BYTE_DATA(out);
  std::vector<size_t> off(pcs.size() + 1, 0);
  for (size_t i = 0; i < pcs.size(); ++i) off[i + 1] = off[i] + pcs[i].second;
  const int parts = parts_for((int64_t)total, 1 << 22);
  Py_BEGIN_ALLOW_THREADS
  run_parts(parts, [&](int k) {                      // byte range [a, b) of the output
    const size_t a = total * k / parts, b = total * (k + 1) / parts;
    for (size_t i = 0; i < pcs.size(); ++i) {
      const size_t lo = std::max(a, off[i]), hi = std::min(b, off[i + 1]);
      if (lo < hi) memcpy(dst + lo, pcs[i].first + (lo - off[i]), hi - lo);
    }
  });
  Py_END_ALLOW_THREADS
  return out;
}
// Column setup shared by the CSV and JSON formatters: false -> the caller
// returns None (Python path); sets an exception and returns false with
// `err` when the C API failed.
bool setup_col(PyObject* o, int64_t& n, CsvCol& c, bool int_ok, bool& err) {
  err = false;
  if (!PyArray_Check(o)) return false;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_NDIM(a) != 1) return false;
  if (n < 0) n = PyArray_DIM(a, 0);
  if (PyArray_DIM(a, 0) != n) return false;
  c.base = (const char*)PyArray_DATA(a);
  c.stride = PyArray_STRIDE(a, 0);
  const int t = PyArray_TYPE(a);
  if (t == NPY_FLOAT64 && PyArray_ISNOTSWAPPED(a)) {
    c.kind = COL_F64;
    c.maxlen = 24;                                   // -d.ddddddddddddddddde-308
    return true;
  }
  if (PyArray_ISFLOAT(a)) return false;              // other float widths: Python path
  if (int_ok && PyArray_ISINTEGER(a) && PyArray_ISNOTSWAPPED(a) && PyArray_ITEMSIZE(a) <= 8) {
    c.kind = COL_INT;
    c.isize = (int)PyArray_ITEMSIZE(a);
    c.is_signed = PyArray_ISSIGNED(a);
    c.maxlen = 1;
    return true;
  }
  if (t != NPY_OBJECT) return false;
  c.kind = COL_STR;
  for (int64_t i = 0; i < n; ++i) {                  // distinct objects (a status column has <= 5)
    PyObject* v = *(PyObject* const*)(c.base + i * c.stride);
    bool seen = false;
    for (PyObject* w : c.objs) if (w == v) { seen = true; break; }
    if (seen) continue;
    if (c.objs.size() >= 16 || !v || !PyUnicode_CheckExact(v)) return false;
    Py_ssize_t len;
    const char* u = PyUnicode_AsUTF8AndSize(v, &len);
    if (!u) { err = true; return false; }
    c.objs.push_back(v);
    c.text.emplace_back(u, len);
    c.maxlen = std::max(c.maxlen, (size_t)len);
  }
  return true;
}
inline bool int_pos(const CsvCol& c, const char* p) {
  switch (c.isize) {
    case 1: return c.is_signed ? *(const int8_t*)p > 0 : *(const uint8_t*)p > 0;
    case 2: return c.is_signed ? *(const int16_t*)p > 0 : *(const uint16_t*)p > 0;
    case 4: return c.is_signed ? *(const int32_t*)p > 0 : *(const uint32_t*)p > 0;
    default: return c.is_signed ? *(const int64_t*)p > 0 : *(const uint64_t*)p > 0;
  }
}
inline const std::string& str_of(const CsvCol& c, const char* p) {
  PyObject* v = *(PyObject* const*)p;
  size_t w = 0;
  while (c.objs[w] != v) ++w;
  return c.text[w];
}

// format_csv(names, columns) -> str, or None when a column is outside the
// fast path (the caller then runs the Python loop).
PyObject* format_csv(PyObject*, PyObject* args) {
  PyObject* names;
  PyObject* cols;
  if (!PyArg_ParseTuple(args, "O!O!", &PyTuple_Type, &names, &PyTuple_Type, &cols)) return nullptr;
  const Py_ssize_t m = PyTuple_GET_SIZE(names);
  if (m != PyTuple_GET_SIZE(cols) || m == 0) Py_RETURN_NONE;
  std::string header;
  for (Py_ssize_t j = 0; j < m; ++j) {
    PyObject* nm = PyTuple_GET_ITEM(names, j);
    if (!PyUnicode_CheckExact(nm)) Py_RETURN_NONE;
    Py_ssize_t len;
    const char* u = PyUnicode_AsUTF8AndSize(nm, &len);
    if (!u) return nullptr;
    if (j) header += ',';
    header.append(u, len);
  }
  header += '\n';
  bool ascii = ascii_text(header.data(), header.size());
  int64_t n = -1;
  std::vector<CsvCol> cc(m);
  size_t rowmax = (size_t)m;                         // separators
  for (Py_ssize_t j = 0; j < m; ++j) {
    bool err;
    if (!setup_col(PyTuple_GET_ITEM(cols, j), n, cc[j], true, err)) {
      if (err) return nullptr;
      Py_RETURN_NONE;
    }
    rowmax += cc[j].maxlen;
    for (auto& t : cc[j].text) ascii = ascii && ascii_text(t.data(), t.size());
  }
  const int parts = parts_for(n, 65536);
  std::vector<OutBuf> buf(parts);
  Py_BEGIN_ALLOW_THREADS
  run_parts(parts, [&](int k) {
    const int64_t a = n * k / parts, b = n * (k + 1) / parts;
    OutBuf& s = buf[k];
    s.reserve((size_t)(b - a) * (size_t)m * 18);
    for (int64_t i = a; i < b; ++i) {
      s.reserve(rowmax);
      char* w = s.ptr();                 // a local cursor: stores through char*
                                         // would otherwise reload s.n each time
      for (Py_ssize_t j = 0; j < m; ++j) {
        const CsvCol& c = cc[j];
        const char* p = c.base + i * c.stride;
        if (c.kind == COL_F64) {
          double v;
          memcpy(&v, p, 8);
          w += repr_double(v, w);
        } else if (c.kind == COL_INT) {
          *w++ = int_pos(c, p) ? 'c' : 'p';
        } else {
          const std::string& t = str_of(c, p);
          memcpy(w, t.data(), t.size());
          w += t.size();
        }
        *w++ = (j + 1 < m) ? ',' : '\n';
      }
      s.n = (size_t)(w - s.b.get());
    }
  });
  Py_END_ALLOW_THREADS
  std::vector<std::pair<const char*, size_t>> pcs;
  pcs.emplace_back(header.data(), header.size());
  for (auto& s : buf) pcs.emplace_back(s.b.get(), s.n);
  return str_from_pieces(pcs, ascii);
}

// ---- CSV chain input (cli.py:140-173 _read_chain + _numeric) ---------------
// parse_chain_csv(data) -> None when the text is outside the fast path (any
// '"' or '\r', a ragged row, a non-ASCII byte, a non-flag text column), else
// (header, columns, bad) with columns[j] a float64 array (numeric columns:
// every cell that is a plain decimal -- [-]digits[.digits][(e|E)[+-]digits] --
// parsed by std::from_chars, correctly rounded like float()) or, for the
// 'flag' column, a numpy 'U1' array; bad = list of (row, column) cells the
// strict form did not take (the caller applies float() to them, which either
// parses them or raises the reference's error).  csv.reader semantics for
// this subset: lines end at '\n', a final '\n' ends the last row, an empty
// line is a row of 0 cells.
bool plain_decimal(const char* p, const char* e) {
  if (p < e && *p == '-') ++p;
  const char* d0 = p;
  while (p < e && *p >= '0' && *p <= '9') ++p;
  bool digits = p > d0;
  if (p < e && *p == '.') {
    ++p;
    const char* f0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    digits = digits || p > f0;
  }
  if (!digits) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* x0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == x0) return false;
  }
  return p == e;
}

PyObject* parse_chain_csv(PyObject*, PyObject* args) {
  Py_buffer buf;
  if (!PyArg_ParseTuple(args, "y*", &buf)) return nullptr;
  struct Release { Py_buffer* b; ~Release() { PyBuffer_Release(b); } } rel{&buf};
  const char* d = (const char*)buf.buf;
  const int64_t len = buf.len;
  if (len == 0) Py_RETURN_NONE;
  // the byte screen and the line starts, on byte ranges in parallel
  const int sparts = parts_for(len, 1 << 22);
  std::vector<std::vector<int64_t>> nl(sparts);
  std::vector<char> odd(sparts, 0);
  Py_BEGIN_ALLOW_THREADS
  run_parts(sparts, [&](int k) {
    const int64_t a = len * k / sparts, b = len * (k + 1) / sparts;
    std::vector<int64_t>& v = nl[k];
    v.reserve((size_t)((b - a) / 48 + 16));
    unsigned char acc = 0;
    for (int64_t i = a; i < b; ++i) {
      const unsigned char ch = (unsigned char)d[i];
      acc |= (unsigned char)(ch == '"' || ch == '\r' || ch >= 0x80);
      if (ch == '\n') v.push_back(i);
    }
    odd[k] = (char)acc;
  });
  Py_END_ALLOW_THREADS
  for (char o : odd) if (o) Py_RETURN_NONE;
  std::vector<int64_t> ls;
  {
    size_t cnt = 1;
    for (auto& v : nl) cnt += v.size();
    ls.reserve(cnt);
  }
  ls.push_back(0);
  for (auto& v : nl)
    for (int64_t i : v)
      if (i + 1 < len) ls.push_back(i + 1);
  std::vector<std::vector<int64_t>>().swap(nl);
  auto line_end = [&](size_t k) {
    int64_t e = (k + 1 < ls.size()) ? ls[k + 1] - 1 : len;
    if (e > ls[k] && d[e - 1] == '\n') --e;         // the final line's '\n'
    return e;
  };
  // header
  std::vector<std::pair<int64_t, int64_t>> hcells;
  {
    int64_t a = ls[0], e = line_end(0);
    if (a == e) Py_RETURN_NONE;                         // csv gives [] for an empty header line
    int64_t c0 = a;
    for (int64_t i = a; i <= e; ++i)
      if (i == e || d[i] == ',') { hcells.emplace_back(c0, i); c0 = i + 1; }
  }
  const int64_t m = (int64_t)hcells.size();
  const int64_t n = (int64_t)ls.size() - 1;
  int flag_col = -1;
  for (int64_t j = 0; j < m; ++j)
    if (hcells[j].second - hcells[j].first == 4 && memcmp(d + hcells[j].first, "flag", 4) == 0) flag_col = (int)j;
  std::vector<double*> out(m, nullptr);
  std::vector<PyObject*> arrays(m, nullptr);
  npy_intp dims[1] = {(npy_intp)n};
  for (int64_t j = 0; j < m; ++j) {
    arrays[j] = (j == flag_col) ? PyArray_New(&PyArray_Type, 1, dims, NPY_UNICODE, nullptr, nullptr, 4, 0, nullptr)
                                : PyArray_SimpleNew(1, dims, NPY_FLOAT64);
    if (!arrays[j]) { for (auto* o : arrays) Py_XDECREF(o); return nullptr; }
  }
  uint32_t* flag_out = flag_col >= 0 ? (uint32_t*)PyArray_DATA((PyArrayObject*)arrays[flag_col]) : nullptr;
  for (int64_t j = 0; j < m; ++j)
    if (j != flag_col) out[j] = (double*)PyArray_DATA((PyArrayObject*)arrays[j]);
  const int parts = parts_for(n, 65536);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> bad(parts);
  std::vector<char> fallback(parts, 0);
  Py_BEGIN_ALLOW_THREADS
  run_parts(parts, [&](int k) {
    const int64_t r0 = n * k / parts, r1 = n * (k + 1) / parts;
    for (int64_t r = r0; r < r1 && !fallback[k]; ++r) {
      const int64_t a = ls[r + 1], e = line_end(r + 1);
      if (a == e) { fallback[k] = 1; break; }            // empty line: csv gives a 0-cell row
      int64_t j = 0, c0 = a;
      for (int64_t i = a; i <= e; ++i) {
        if (i != e && d[i] != ',') continue;
        if (j >= m) { fallback[k] = 1; break; }          // ragged row: the Python path reports it
        if (j == flag_col) {
          if (i - c0 != 1) { fallback[k] = 1; break; }   // flag cells other than one character
          flag_out[r] = (unsigned char)d[c0];
        } else if (plain_decimal(d + c0, d + i)) {
          double v;
          auto res = std::from_chars(d + c0, d + i, v);
          if (res.ec == std::errc::result_out_of_range) {
            bad[k].emplace_back(r, j);                   // float() gives inf / 0 here: let it
            v = 0.0;
          }
          out[j][r] = v;
        } else {
          out[j][r] = 0.0;
          bad[k].emplace_back(r, j);
        }
        ++j;
        c0 = i + 1;
      }
      if (j != m) fallback[k] = 1;
    }
  });
  Py_END_ALLOW_THREADS
  bool fb = false;
  for (char f : fallback) fb = fb || f;
  if (fb) { for (auto* o : arrays) Py_XDECREF(o); Py_RETURN_NONE; }
  PyObject* hdr = PyTuple_New(m);
  PyObject* cols = PyTuple_New(m);
  PyObject* badl = PyList_New(0);
  for (int64_t j = 0; j < m; ++j) {
    PyTuple_SET_ITEM(hdr, j, PyUnicode_DecodeASCII(d + hcells[j].first, hcells[j].second - hcells[j].first, "strict"));
    PyTuple_SET_ITEM(cols, j, arrays[j]);
  }
  for (auto& v : bad)
    for (auto& rc : v) {
      PyObject* t = Py_BuildValue("(LL)", (long long)rc.first, (long long)rc.second);
      PyList_Append(badl, t);
      Py_DECREF(t);
    }
  return Py_BuildValue("(NNN)", hdr, cols, badl);
}

// format_json(keys, columns, flag_index) -> str or None: batch.py:307-317
// json.dumps({name: [...]}) with float64 columns as repr / null (non-finite),
// the integer 'flag' column as "c" / "p", str-object columns as their text;
// keys arrive JSON-encoded from the caller.  Strings that would need JSON
// escapes (quote, backslash, control or non-ASCII characters) -> None.
bool json_plain(const std::string& s) {
  for (unsigned char ch : s)
    if (ch < 0x20 || ch >= 0x7f || ch == '"' || ch == '\\') return false;
  return true;
}

PyObject* format_json(PyObject*, PyObject* args) {
  PyObject* keys;
  PyObject* cols;
  int flag_index;
  if (!PyArg_ParseTuple(args, "O!O!i", &PyTuple_Type, &keys, &PyTuple_Type, &cols, &flag_index)) return nullptr;
  const Py_ssize_t m = PyTuple_GET_SIZE(keys);
  if (m != PyTuple_GET_SIZE(cols)) Py_RETURN_NONE;
  std::vector<std::string> kenc(m);
  bool ascii = true;
  for (Py_ssize_t j = 0; j < m; ++j) {
    PyObject* k = PyTuple_GET_ITEM(keys, j);
    if (!PyUnicode_CheckExact(k)) Py_RETURN_NONE;
    Py_ssize_t len;
    const char* u = PyUnicode_AsUTF8AndSize(k, &len);
    if (!u) return nullptr;
    kenc[j].assign(u, len);
    ascii = ascii && ascii_text(u, (size_t)len);
  }
  int64_t n = -1;
  std::vector<CsvCol> cc(m);
  for (Py_ssize_t j = 0; j < m; ++j) {
    bool err;
    PyObject* o = PyTuple_GET_ITEM(cols, j);
    if (j != flag_index && PyArray_Check(o) && PyArray_TYPE((PyArrayObject*)o) != NPY_FLOAT64 &&
        PyArray_TYPE((PyArrayObject*)o) != NPY_OBJECT)
      Py_RETURN_NONE;
    if (!setup_col(o, n, cc[j], j == flag_index, err)) {
      if (err) return nullptr;
      Py_RETURN_NONE;
    }
    if (j == flag_index && cc[j].kind == COL_STR) Py_RETURN_NONE;   // Python's "c" / "p" mapping
    for (auto& t : cc[j].text) {
      if (!json_plain(t)) Py_RETURN_NONE;
      t = "\"" + t + "\"";
    }
    cc[j].maxlen += 2;
    if (cc[j].kind == COL_INT) cc[j].maxlen = 3;
  }
  if (n < 0) n = 0;
  const int parts = parts_for(n, 65536);
  std::vector<OutBuf> chunk((size_t)m * parts);
  Py_BEGIN_ALLOW_THREADS
  run_parts(parts, [&](int k) {
    const int64_t a = n * k / parts, b = n * (k + 1) / parts;
    for (Py_ssize_t j = 0; j < m; ++j) {
      const CsvCol& c = cc[j];
      OutBuf& s = chunk[(size_t)j * parts + k];
      s.reserve((size_t)(b - a) * (c.kind == COL_F64 ? 20 : c.maxlen + 2));
      const int64_t blk = 4096;
      for (int64_t i0 = a; i0 < b; i0 += blk) {
        const int64_t i1 = std::min(b, i0 + blk);
        s.reserve((size_t)(i1 - i0) * (c.maxlen + 2));
        char* w = s.ptr();
        for (int64_t i = i0; i < i1; ++i) {
          if (i) { *w++ = ','; *w++ = ' '; }
          const char* p = c.base + i * c.stride;
          if (c.kind == COL_F64) {
            double v;
            memcpy(&v, p, 8);
            if (v - v != 0.0) { memcpy(w, "null", 4); w += 4; }   // nan, inf
            else w += repr_double(v, w);
          } else if (c.kind == COL_INT) {
            memcpy(w, int_pos(c, p) ? "\"c\"" : "\"p\"", 3);
            w += 3;
          } else {
            const std::string& t = str_of(c, p);
            memcpy(w, t.data(), t.size());
            w += t.size();
          }
        }
        s.n = (size_t)(w - s.b.get());
      }
    }
  });
  Py_END_ALLOW_THREADS
  std::vector<std::string> glue((size_t)m + 1);
  std::vector<std::pair<const char*, size_t>> pcs;
  for (Py_ssize_t j = 0; j < m; ++j) {
    glue[j] = (j ? std::string(", ") : std::string("{")) + kenc[j] + ": [";
    pcs.emplace_back(glue[j].data(), glue[j].size());
    for (int k = 0; k < parts; ++k) {
      OutBuf& s = chunk[(size_t)j * parts + k];
      pcs.emplace_back(s.b.get(), s.n);
    }
    pcs.emplace_back("]", 1);
  }
  glue[m] = m ? "}" : "{}";
  pcs.emplace_back(glue[m].data(), glue[m].size());
  return str_from_pieces(pcs, ascii);
}

// write_text(path, text) -> True, or None for text that is not compact ASCII
// (the caller writes it itself): the bytes of an ASCII str are its UTF-8, so
// they go to the file as they are, without the text layer's encode copy,
// with the GIL released.  Same file contents as open(path, "w").write(text).
PyObject* write_text(PyObject*, PyObject* args) {
  PyObject* path;
  PyObject* text;
  if (!PyArg_ParseTuple(args, "O&U", PyUnicode_FSConverter, &path, &text)) return nullptr;
  struct Drop { PyObject* o; ~Drop() { Py_DECREF(o); } } drop{path};
  if (!PyUnicode_IS_COMPACT_ASCII(text)) Py_RETURN_NONE;
  const char* p = (const char*)PyUnicode_DATA(text);
  size_t left = (size_t)PyUnicode_GET_LENGTH(text);
  const char* fn = PyBytes_AS_STRING(path);
  int rc = 0, e = 0;
  Py_BEGIN_ALLOW_THREADS
  const int fd = open(fn, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0666);
  if (fd < 0) { rc = -1; e = errno; }
  while (fd >= 0 && left) {
    const ssize_t w = write(fd, p, left > (1u << 30) ? (1u << 30) : left);
    if (w < 0) { if (errno == EINTR) continue; rc = -1; e = errno; break; }
    p += w;
    left -= (size_t)w;
  }
  if (fd >= 0 && close(fd) != 0 && rc == 0) { rc = -1; e = errno; }
  Py_END_ALLOW_THREADS
  if (rc) {
    errno = e;
    return PyErr_SetFromErrnoWithFilenameObject(PyExc_OSError, PyTuple_GET_ITEM(args, 0));
  }
  Py_RETURN_TRUE;
}

PyMethodDef kMethods[] = {
    {"format_json", format_json, METH_VARARGS, "format_output(table, 'json') for float / flag / str columns, or None"},
    {"parse_chain_csv", parse_chain_csv, METH_VARARGS, "fast path of the chain CSV reader, or None"},
    {"format_csv", format_csv, METH_VARARGS, "format_output(table, 'csv') for float / integer-flag / str columns, or None"},
    {"repr_doubles", repr_doubles, METH_VARARGS, "repr(float(v)) for each element (test hook)"},
    {"parse_flags_u", parse_flags_u, METH_VARARGS, "case-insensitive c/p -> int8 +1/-1; (flags, first_bad)"},
    {"status_objects", status_objects, METH_VARARGS, "object array names[codes]"},
    {"write_text", write_text, METH_VARARGS, "write an ASCII str to a file (GIL released), or None"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_fvhost", "fastvol_b200 batch front-end host loops", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__fvhost(void) {
  import_array();
  return PyModule_Create(&kModule);
}
