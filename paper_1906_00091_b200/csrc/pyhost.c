/* Host-side packing entry for Python callers (libdlrmpy.so, loaded with
 * ctypes.PyDLL so it runs holding the GIL).
 *
 * InputLayout._pack_native used to build its per-table pointer arrays in
 * Python (arr.ctypes.data per offsets / indices array: ~1 us each, 2T + 4
 * per batch, ~180 us of interpreter time per c2 batch of 26 tables).  The
 * Prefetcher's packing workers held the GIL that long per batch, and the
 * training thread's own per-step calls (graph replay, input hand-over,
 * result ring) waited behind them: e2e at c2 was host-bound at 0.27 ms
 * against a 0.18 ms device step.  Here the same validation (dtype, shape,
 * contiguity, capacity) and pointer extraction are done through the buffer
 * protocol in C, then dlrm_pack_batch (randsrc.cu) runs with the GIL
 * released.
 *
 * Return codes: 0 packed; 1 the arrays are not the reference's dtypes /
 * layout (caller falls back to the numpy path); 2 + t: table t holds more
 * indices than its capacity (caller raises the OverflowError); -1 a Python
 * error is set.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

#include "dlrm_b200.h"

#define MAXT 1024

static int is_fmt(const Py_buffer* v, char a, char b) {
  const char* f = v->format ? v->format : "B";
  if (*f == '<' || *f == '=' || *f == '@') ++f;
  return f[1] == 0 && (f[0] == a || f[0] == b);
}

/* 1-D C-contiguous buffer of 8-byte items of format a|b, n elements (n < 0:
 * any).  0 ok, 1 mismatch, -1 error set. */
static int get_vec(PyObject* o, Py_buffer* v, char a, char b, Py_ssize_t n) {
  if (PyObject_GetBuffer(o, v, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
    PyErr_Clear();
    return 1;
  }
  if (v->ndim != 1 || v->itemsize != 8 || !is_fmt(v, a, b) || (n >= 0 && v->shape[0] != n)) {
    PyBuffer_Release(v);
    return 1;
  }
  return 0;
}

/* The staging half (optional): after packing, still without the GIL, the
 * block's H2D copy is issued on `stream` (after wait_ev) and ev1 / ev2
 * recorded (dlrm_h2d_async); nnz_out (optional) receives the per-table index
 * counts. */
static int pack_impl(PyObject* dense, PyObject* labels, PyObject* offsets, PyObject* indices,
                     PyObject* weights, uint8_t* dst, const int64_t* sec, int64_t batch,
                     int64_t k0, int64_t ldx, int32_t nt, const int64_t* cap_base,
                     int32_t nthreads, void* dev_dst, size_t bytes, void* wait_ev, void* ev1,
                     void* ev2, void* stream, int64_t* nnz_out);

int dlrm_pack_batch_py(PyObject* dense, PyObject* labels, PyObject* offsets, PyObject* indices,
                       PyObject* weights, uint8_t* dst, const int64_t* sec, int64_t batch,
                       int64_t k0, int64_t ldx, int32_t nt, const int64_t* cap_base,
                       int32_t nthreads) {
  return pack_impl(dense, labels, offsets, indices, weights, dst, sec, batch, k0, ldx, nt,
                   cap_base, nthreads, NULL, 0, NULL, NULL, NULL, NULL, NULL);
}

int dlrm_pack_stage_py(PyObject* dense, PyObject* labels, PyObject* offsets, PyObject* indices,
                       PyObject* weights, uint8_t* dst, const int64_t* sec, int64_t batch,
                       int64_t k0, int64_t ldx, int32_t nt, const int64_t* cap_base,
                       int32_t nthreads, void* dev_dst, size_t bytes, void* wait_ev, void* ev1,
                       void* ev2, void* stream, int64_t* nnz_out) {
  return pack_impl(dense, labels, offsets, indices, weights, dst, sec, batch, k0, ldx, nt,
                   cap_base, nthreads, dev_dst, bytes, wait_ev, ev1, ev2, stream, nnz_out);
}

static int pack_impl(PyObject* dense, PyObject* labels, PyObject* offsets, PyObject* indices,
                     PyObject* weights, uint8_t* dst, const int64_t* sec, int64_t batch,
                     int64_t k0, int64_t ldx, int32_t nt, const int64_t* cap_base,
                     int32_t nthreads, void* dev_dst, size_t bytes, void* wait_ev, void* ev1,
                     void* ev2, void* stream, int64_t* nnz_out) {
  if (nt < 1 || nt > MAXT) return 1;
  PyObject* fo = PySequence_Fast(offsets, "offsets");
  PyObject* fi = fo ? PySequence_Fast(indices, "indices") : NULL;
  PyObject* fw = NULL;
  if (!fo || !fi) {
    Py_XDECREF(fo);
    PyErr_Clear();
    return 1;
  }
  if (weights != Py_None) {
    fw = PySequence_Fast(weights, "weights");
    if (!fw) {
      Py_DECREF(fo);
      Py_DECREF(fi);
      PyErr_Clear();
      return 1;
    }
  }
  int rc = 1;
  Py_buffer bd, bl;
  Py_buffer* bo = PyMem_Calloc(3 * (size_t)nt, sizeof(Py_buffer));
  const int64_t** po = PyMem_Calloc(3 * (size_t)nt, sizeof(void*));
  int64_t* nnz = PyMem_Calloc((size_t)nt, sizeof(int64_t));
  char* held = PyMem_Calloc(3 * (size_t)nt, 1);
  int have_d = 0, have_l = 0;
  const int64_t** pi = po ? po + nt : NULL;
  const double** pw = po ? (const double**)(po + 2 * nt) : NULL;
  if (!bo || !po || !nnz || !held) {
    PyErr_NoMemory();
    rc = -1;
    goto out;
  }
  if (PySequence_Fast_GET_SIZE(fo) != nt || PySequence_Fast_GET_SIZE(fi) != nt ||
      (fw && PySequence_Fast_GET_SIZE(fw) != nt))
    goto out;
  /* dense: 2-D float64, unit column stride */
  if (PyObject_GetBuffer(dense, &bd, PyBUF_STRIDES | PyBUF_FORMAT) != 0) {
    PyErr_Clear();
    goto out;
  }
  have_d = 1;
  if (bd.ndim != 2 || bd.itemsize != 8 || !is_fmt(&bd, 'd', 'd') || bd.shape[0] != batch ||
      bd.shape[1] != k0 || bd.strides[1] != 8 || bd.strides[0] % 8 != 0 || bd.strides[0] < 0)
    goto out;
  if (get_vec(labels, &bl, 'd', 'd', batch)) goto out;
  have_l = 1;
  for (int t = 0; t < nt; ++t) {
    if (get_vec(PySequence_Fast_GET_ITEM(fo, t), &bo[t], 'l', 'q', batch + 1)) goto out;
    held[t] = 1;
    po[t] = (const int64_t*)bo[t].buf;
    if (get_vec(PySequence_Fast_GET_ITEM(fi, t), &bo[nt + t], 'l', 'q', -1)) goto out;
    held[nt + t] = 1;
    pi[t] = (const int64_t*)bo[nt + t].buf;
    nnz[t] = bo[nt + t].shape[0];
    if (fw) {
      PyObject* w = PySequence_Fast_GET_ITEM(fw, t);
      if (w != Py_None) {
        if (get_vec(w, &bo[2 * nt + t], 'd', 'd', nnz[t])) goto out;
        held[2 * nt + t] = 1;
        pw[t] = (const double*)bo[2 * nt + t].buf;
      }
    }
  }
  for (int t = 0; t < nt; ++t)
    if (nnz[t] > cap_base[t + 1] - cap_base[t]) {
      rc = 2 + t;
      goto out;
    }
  {
    const double* dp = (const double*)bd.buf;
    const int64_t ldd = bd.strides[0] / 8;
    const double* lp = (const double*)bl.buf;
    int r, h = 0;
    Py_BEGIN_ALLOW_THREADS
    r = dlrm_pack_batch(dst, sec, batch, k0, ldx, nt, cap_base, dp, ldd, lp, po, pi, nnz,
                        fw ? pw : NULL, nthreads);
    if (r == 0 && dev_dst) h = dlrm_h2d_async(dev_dst, dst, bytes, wait_ev, ev1, ev2, stream);
    Py_END_ALLOW_THREADS
    if (r == 0 && h != 0) {
      PyErr_SetString(PyExc_RuntimeError, dlrm_last_error());
      rc = -1;
      goto out;
    }
    if (r == 0 && nnz_out) memcpy(nnz_out, nnz, sizeof(int64_t) * (size_t)nt);
    rc = r == 0 ? 0 : 1;
  }
out:
  if (held)
    for (int i = 0; i < 3 * nt; ++i)
      if (held[i]) PyBuffer_Release(&bo[i]);
  if (have_l) PyBuffer_Release(&bl);
  if (have_d) PyBuffer_Release(&bd);
  PyMem_Free(bo);
  PyMem_Free(po);
  PyMem_Free(nnz);
  PyMem_Free(held);
  Py_DECREF(fo);
  Py_DECREF(fi);
  Py_XDECREF(fw);
  return rc;
}
