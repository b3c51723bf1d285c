"""ctypes binding of libdlrmb200.so (the C ABI in include/dlrm_b200.h).

There is no CPU fallback: if the library is missing, or a tensor handed to a
kernel is not a CUDA tensor, the call fails loudly.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DLRM_B200_LIB") or os.path.join(_HERE, "libdlrmb200.so")

MAX_TABLES = 128
MAX_FEATURES = 129
ACT = {"identity": 0, "relu": 1}

_i64, _i32, _f32, _vp, _sz = C.c_int64, C.c_int32, C.c_float, C.c_void_p, C.c_size_t


class TableDesc(C.Structure):
    _fields_ = [("offsets", _vp), ("indices", _vp), ("weights", _vp),
                ("row_base", _i64), ("num_rows", _i64), ("out_offset", _i64),
                ("capacity", _i64), ("table_id", _i64)]


class Update(C.Structure):
    """dlrm_update: SGD / Adagrad rule; accumulator = parameter + accum_delta."""
    _fields_ = [("kind", _i32), ("lr", _f32), ("eps", _f32), ("accum_delta", _i64)]


UPD_SGD, UPD_ADAGRAD = 0, 1


class Features(C.Structure):
    _fields_ = [("feat", _vp * MAX_FEATURES),
                ("feat_stride", _i64 * MAX_FEATURES)]


_SIGS = {
    "dlrm_err_reset": [_vp, _i32, _vp, _vp],
    "dlrm_err_resolve": [_vp, _i32, _vp, _vp, _vp, _vp],
    "dlrm_emb_fwd": [_vp, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp],
    "dlrm_emb_bwd_sgd": [_vp, _i64, _vp, _i32, _i64, _vp, _i64, _f32, _vp,
                         _i64, _vp, _sz, _vp],
    "dlrm_emb_bwd_prepare": [_i64, _vp, _i32, _i64, _i64, _vp, _sz, _vp],
    "dlrm_emb_bwd_apply_sgd": [_vp, _i64, _vp, _i32, _i64, _vp, _i64, _f32,
                               _vp, _i64, _vp, _sz, _vp],
    "dlrm_emb_bwd_apply": [_vp, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _i64,
                           _vp, _sz, _vp],
    "dlrm_update_rows": [_vp, _i64, _vp, _vp, _i64, _vp, _vp],
    "dlrm_linear_bwd_weight_upd": [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp,
                                   _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                   _sz, _vp],
    "dlrm_head_bwd_upd": [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp,
                          _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
    "dlrm_update_dense": [_vp, _vp, _i64, _vp, _vp, _vp],
    "dlrm_head_step": [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _f32, _vp, _vp, _vp,
                       _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
    "dlrm_head_step_partials": [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _f32, _vp, _vp, _vp,
                                _i64, _i32, _vp, _sz, _vp],
    "dlrm_head_step_reduce": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
    "dlrm_emb_bwd_coalesce": [_i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp,
                              _vp, _vp, _sz, _vp],
    "dlrm_sgd_rows": [_vp, _i64, _vp, _vp, _i64, _f32, _vp],
    "dlrm_interact_fwd": [_vp, _i32, _i64, _i64, _vp, _i64, _i64, _vp],
    "dlrm_interact_bwd": [_vp, _i32, _i64, _i64, _vp, _i64, _vp, _vp, _i32,
                          _vp],
    "dlrm_linear_fwd": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _i64,
                        _i64, _i64, _i32, _vp],
    "dlrm_linear_bwd_data": [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                             _i64, _i64, _i64, _vp],
    "dlrm_linear_fwd_wlo": [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _i64,
                            _i64, _i64, _i32, _vp],
    "dlrm_linear_bwd_data_wlo": [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                                 _i64, _i64, _i64, _vp],
    "dlrm_tf32_split_lo": [_vp, _vp, _i64, _vp],
    "dlrm_h2d_async": [_vp, _vp, C.c_size_t, _vp, _vp, _vp, _vp],
    "dlrm_step_result_copy": [_vp, _vp, C.c_size_t, _vp, _vp, C.c_size_t, _vp, _vp],
    "dlrm_d2d_async": [_vp, _vp, C.c_size_t, _vp, _vp, _vp],
    "dlrm_linear_bwd_weight": [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp,
                               _i64, _vp, _vp, _i64, _vp, _f32, _vp, _vp,
                               _sz, _vp],
    "dlrm_bce_head": [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _f32, _vp, _vp,
                      _vp, _vp, _vp, _vp, _sz, _vp],
    "dlrm_head_bwd": [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp,
                      _vp, _vp, _vp, _f32, _vp, _vp, _sz, _vp],
    "dlrm_relu_grad": [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _vp],
    "dlrm_sgd_dense": [_vp, _vp, _i64, _f32, _vp, _vp],
    "dlrm_gemm_mode": [_i32],
}
_SIZE_FNS = {
    "dlrm_emb_bwd_workspace_size": [_i64, _i64, _i64],
    "dlrm_linear_bwd_weight_workspace_size": [_i64, _i64, _i64],
    "dlrm_bce_head_workspace_size": [_i64],
    "dlrm_head_bwd_workspace_size": [_i64, _i64],
    "dlrm_head_step_workspace_size": [_i64, _i64],
}

# every symbol include/dlrm_b200.h declares (checked by tests/test_abi.py)
EXPORTS = sorted(list(_SIGS) + list(_SIZE_FNS) + [
    "dlrm_launch_count", "dlrm_last_error", "dlrm_build_info", "dlrm_criteo_parse",
    "dlrm_blake2b64", "dlrm_random_bags", "dlrm_pack_batch", "dlrm_gemm_mode_get"])

_lib = None


def lib():
    """Load libdlrmb200.so once; raise if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with "
                "`python -m paper_1906_00091_b200.build` (there is no CPU "
                "fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, _i32
        for name, args in _SIZE_FNS.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, _sz
        L.dlrm_launch_count.argtypes, L.dlrm_launch_count.restype = [], _i64
        # host-side input pipeline (no GPU needed)
        L.dlrm_criteo_parse.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64,
                                        _i64, _vp, _i32]
        L.dlrm_criteo_parse.restype = _i64
        L.dlrm_blake2b64.argtypes, L.dlrm_blake2b64.restype = [_vp, _i64], C.c_uint64
        L.dlrm_random_bags.argtypes = [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp]
        L.dlrm_random_bags.restype = _i32
        L.dlrm_pack_batch.argtypes = [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _i64, _vp,
                                      _vp, _vp, _vp, _vp, _i32]
        L.dlrm_pack_batch.restype = _i32
        L.dlrm_gemm_mode_get.argtypes, L.dlrm_gemm_mode_get.restype = [], _i32
        L.dlrm_last_error.restype = C.c_char_p
        L.dlrm_build_info.restype = C.c_char_p
        _lib = L
    return _lib


PYLIB_PATH = os.path.join(_HERE, "libdlrmpy.so")
_pylib = None


def pylib():
    """libdlrmpy.so (csrc/pyhost.c: batch packing straight from the Python
    arrays, buffer protocol in C, GIL released around dlrm_pack_batch),
    loaded with ctypes.PyDLL; None when it was not built."""
    global _pylib
    if _pylib is None:
        lib()
        if not os.path.exists(PYLIB_PATH):
            _pylib = False
        else:
            L = C.PyDLL(PYLIB_PATH)
            f = L.dlrm_pack_batch_py
            po = C.py_object
            f.argtypes = [po, po, po, po, po, _vp, _vp, _i64, _i64, _i64, _i32, _vp, _i32]
            f.restype = C.c_int
            g = L.dlrm_pack_stage_py
            g.argtypes = f.argtypes + [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp]
            g.restype = C.c_int
            _pylib = L
    return _pylib or None


class KernelError(RuntimeError):
    pass


@contextlib.contextmanager
def accurate_gemms(enable: bool):
    """The enclosed launches and graph captures use the SIMT fp32 GEMMs and
    interaction (``dlrm_gemm_mode(1)``) when ``enable`` and the caller left
    the default mode; the caller's mode is restored.  Used by Adagrad steps:
    Adagrad divides every gradient component by its own running magnitude,
    so the error of tiny components — larger with 3xTF32's truncating
    tensor-core accumulation than with fp32 FMA chains — reaches the weights
    (DESIGN.md §2)."""
    if not enable:
        yield
        return
    L = lib()
    prev = int(L.dlrm_gemm_mode_get())
    if prev != 0:
        yield
        return
    L.dlrm_gemm_mode(1)
    try:
        yield
    finally:
        L.dlrm_gemm_mode(prev)


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().dlrm_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise KernelError(f"{name}: {msg}")


def size(name, *args) -> int:
    return int(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().dlrm_launch_count())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t) -> C.c_void_p:
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    if not t.is_cuda:
        raise TypeError("libdlrmb200 kernels take CUDA tensors only "
                        "(no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1906_00091_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def make_features(ptrs_strides):
    f = Features()
    if len(ptrs_strides) > MAX_FEATURES:
        raise ValueError(f"at most {MAX_FEATURES} interaction features")
    for i, (p, s) in enumerate(ptrs_strides):
        f.feat[i] = p
        f.feat_stride[i] = s
    return f


def table_array(descs):
    if len(descs) > MAX_TABLES:
        raise ValueError(f"at most {MAX_TABLES} tables per kernel call")
    arr = (TableDesc * len(descs))()
    for i, d in enumerate(descs):
        arr[i] = d
    return arr


class capture_guard:
    """Around a CUDA-graph capture: collect garbage first and keep the cyclic
    collector off while capturing.  A model and its cached step engine
    reference each other, so dead engines (and their CUDA graphs) are freed
    by the cyclic GC — which may otherwise run in the middle of a capture,
    where destroying a graph is an illegal operation that invalidates it."""

    def __enter__(self):
        import gc
        gc.collect()
        self._was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()
        return False
