"""Thin ctypes binding of include/gft.h (argument marshalling only).

Every function here has the name of the C entry point it wraps and does nothing but
convert arguments, call the library and raise GFTError on a non-OK status.  All
computation happens in libgft.so: the host planner in C++ and the transforms in the
generated sm_100a kernels.  There is no CPU or PyTorch fallback: if the library or a
CUDA device is missing the call raises.

`Plan` is a convenience owner of a gft_plan handle whose methods are the same calls.
torch is used only to hand device pointers and the current stream to the library.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_size_t, c_uint32, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFT_LIB", os.path.join(_HERE, "_lib", "libgft.so"))

GFT_F32, GFT_F64 = 0, 1
GFT_FLAG_HOST_ONLY, GFT_FLAG_NO_CUBIN_CACHE, GFT_FLAG_NO_TENSOR_CORES, GFT_FLAG_NORMALIZED = 1, 2, 4, 8
GFT_FLAG_DENSE_TC = 16
GFT_FLAG_NO_RIGHT_HAAR = 32
K_FAST_FWD, K_FAST_INV, K_DENSE_FWD, K_DENSE_INV = 0, 1, 2, 3
GFT_MAX_LEVELS = 64

STATUS = {0: "GFT_OK", 1: "GFT_ERR_INVALID_ARG", 2: "GFT_ERR_NOT_INVOLUTION",
          3: "GFT_ERR_NOT_SYMMETRIC", 4: "GFT_ERR_EIG_NOCONVERGE", 5: "GFT_ERR_ALIGNMENT",
          6: "GFT_ERR_UNSUPPORTED", 7: "GFT_ERR_CUDA", 8: "GFT_ERR_NOMEM", 9: "GFT_ERR_COMPILE",
          10: "GFT_ERR_NO_DEVICE"}

# every symbol include/gft.h declares (checked by tests/test_abi.py)
EXPORTS = ["gft_plan_opts_default", "gft_plan_create", "gft_plan_destroy", "gft_forward",
           "gft_inverse", "gft_dense_forward", "gft_dense_inverse", "gft_execute_host",
           "gft_plan_compile", "gft_plan_info_get", "gft_plan_eigenvalues", "gft_plan_basis",
           "gft_plan_leaf_sizes", "gft_plan_kernel_source", "gft_plan_kernel_name",
           "gft_plan_launch_config", "gft_laplacian", "gft_decompose", "gft_find_involution",
           "gft_status_str", "gft_last_error", "gft_abi_version", "gft_filter_create",
           "gft_filter_apply", "gft_filter_kernel_name", "gft_filter_kernel_source", "gft_filter_destroy",
           "gft_plan_serialize", "gft_plan_deserialize", "gft_plan_tune", "gft_filter_tune",
           "gft_plan_tuning_get", "gft_plan_tuning_set"]


class GFTError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__("%s: %s" % (self.name, msg))


class gft_plan_opts(ctypes.Structure):
    _fields_ = [("max_depth", c_int32), ("min_leaf", c_int32), ("search_budget", c_int64),
                ("sym_rtol", c_double), ("dtypes", c_uint32), ("flags", c_uint32),
                ("approx_layers", c_int32), ("approx_min_leaf", c_int32)]


class gft_plan_info(ctypes.Structure):
    _fields_ = [("n", c_int32), ("depth", c_int32), ("n_units", c_int32),
                ("units_per_level", c_int32 * GFT_MAX_LEVELS), ("n_leaves", c_int32),
                ("max_leaf", c_int32), ("n_scale_fix", c_int32), ("n_vz_total", c_int32),
                ("sum_k2", c_int64), ("adds", c_int64), ("mults", c_int64), ("paper_mults", c_int64),
                ("dense_adds", c_int64), ("dense_mults", c_int64), ("n_clusters", c_int32),
                ("kernels_ready", c_int32), ("residual", c_double), ("orth_error", c_double),
                ("n_right_stages", c_int32), ("n_right_pairs", c_int32),
                ("n_approx_leaves", c_int32), ("n_givens", c_int32)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "units_per_level"}
        d["units_per_level"] = list(self.units_per_level[: self.depth])
        return d


_lib = None


def lib():
    """Load libgft.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libgft.so not built: run `python -m paper_1907_07875_b200.build` "
                          "(or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    P = c_void_p
    sig = {
        "gft_plan_opts_default": (None, [POINTER(gft_plan_opts)]),
        "gft_plan_create": (c_int32, [POINTER(c_void_p), c_int32, c_int64, P, P, P, P, P,
                                      POINTER(gft_plan_opts)]),
        "gft_plan_destroy": (c_int32, [P]),
        "gft_forward": (c_int32, [P, P, P, c_int64, c_int32, P]),
        "gft_inverse": (c_int32, [P, P, P, c_int64, c_int32, P]),
        "gft_dense_forward": (c_int32, [P, P, P, c_int64, c_int32, P]),
        "gft_dense_inverse": (c_int32, [P, P, P, c_int64, c_int32, P]),
        "gft_execute_host": (c_int32, [P, c_int32, P, P, c_int64, c_int32, P, c_size_t, c_int64, P]),
        "gft_plan_compile": (c_int32, [P, c_int32, c_uint32]),
        "gft_plan_tune": (c_int32, [P, c_int32, c_uint32, c_uint32, P, P, c_int64, c_int32, P, P]),
        "gft_filter_tune": (c_int32, [P, c_int32, c_uint32, P, P, c_int64, c_int32, P, P]),
        "gft_plan_tuning_get": (c_int32, [P, c_int32, c_int32, P]),
        "gft_plan_tuning_set": (c_int32, [P, c_int32, c_int32, P]),
        "gft_plan_info_get": (c_int32, [P, POINTER(gft_plan_info)]),
        "gft_plan_eigenvalues": (c_int32, [P, P]),
        "gft_plan_basis": (c_int32, [P, P]),
        "gft_plan_leaf_sizes": (c_int32, [P, P, c_int32, POINTER(c_int32)]),
        "gft_plan_kernel_source": (c_int32, [P, c_int32, c_int32, c_char_p, c_size_t, POINTER(c_size_t)]),
        "gft_plan_kernel_name": (c_int32, [P, c_int32, c_int32, c_char_p, c_size_t]),
        "gft_plan_launch_config": (c_int32, [P, c_int32, c_int32, c_int64, POINTER(c_int32),
                                             POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
        "gft_laplacian": (c_int32, [c_int32, c_int64, P, P, P, P, P]),
        "gft_decompose": (c_int32, [c_int32, P, P, c_double, P, P, POINTER(c_int32)]),
        "gft_find_involution": (c_int32, [c_int32, P, c_double, c_int64, P, POINTER(c_int32),
                                          POINTER(c_int32)]),
        "gft_status_str": (c_char_p, [c_int32]),
        "gft_last_error": (c_char_p, []),
        "gft_abi_version": (c_int32, []),
        "gft_filter_create": (c_int32, [POINTER(c_void_p), P, P, c_uint32, c_uint32]),
        "gft_filter_apply": (c_int32, [P, P, P, c_int64, c_int32, P]),
        "gft_filter_kernel_name": (c_int32, [P, c_int32, c_char_p, c_size_t]),
        "gft_filter_kernel_source": (c_int32, [P, c_int32, c_char_p, c_size_t, POINTER(c_size_t)]),
        "gft_filter_destroy": (c_int32, [P]),
        "gft_plan_serialize": (c_int32, [P, P, c_size_t, POINTER(c_size_t)]),
        "gft_plan_deserialize": (c_int32, [POINTER(c_void_p), P, c_size_t, POINTER(gft_plan_opts)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status):
    if status != 0:
        raise GFTError(status, lib().gft_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


def _dev_ptr(t):
    """Device address of a torch tensor (or an int address), as an int (ctypes converts it
    for c_void_p arguments)."""
    if isinstance(t, int):
        return t
    return t.data_ptr()



def _check_pair(a, b, n, cuda):
    """The output tensor `b` of a call must mirror the input `a`: same device kind, shape
    [batch, n], dtype, contiguous -- the library writes batch x n elements through its raw
    pointer, so a smaller / strided / host-vs-device mismatch would corrupt memory."""
    import torch
    where = "CUDA" if cuda else "host"
    for t, nm in ((a, "input"), (b, "output")):
        if not isinstance(t, torch.Tensor) or t.is_cuda != cuda:
            raise ValueError("%s: a %s tensor is required" % (nm, where))
        if t.dim() != 2 or t.shape[1] != n or not t.is_contiguous():
            raise ValueError("%s: expected a contiguous [batch, %d] tensor" % (nm, n))
        if t.dtype is not torch.float32 and t.dtype is not torch.float64:
            raise ValueError("%s: float32 / float64 tensors only" % nm)
    if b.shape != a.shape or b.dtype != a.dtype:
        raise ValueError("input and output must have the same shape and dtype")
    if cuda and a.device != b.device:
        raise ValueError("input and output must be on the same device")

_raw_stream = None


def _stream_handle(stream, device_index=None):
    """CUstream handle (int): the given torch stream / raw handle, else the current stream of
    `device_index` (default: the current device)."""
    global _raw_stream
    if stream is None:
        import torch
        if _raw_stream is None:
            # the raw-handle query avoids building a torch.cuda.Stream object per call (~2 us)
            _raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", False)
        if device_index is None:
            device_index = torch.cuda.current_device()
        if _raw_stream:
            return _raw_stream(device_index)
        return torch.cuda.current_stream(device_index).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dtype_code(dtype):
    if dtype in (GFT_F32, GFT_F64):
        return dtype
    s = str(dtype)
    if "64" in s or s in ("f64", "double"):
        return GFT_F64
    return GFT_F32


# ----------------------------------------------------------------------------- C names
def gft_abi_version():
    return lib().gft_abi_version()


def gft_status_str(s):
    return lib().gft_status_str(s).decode()


def gft_last_error():
    return lib().gft_last_error().decode()


def gft_plan_opts_default():
    o = gft_plan_opts()
    lib().gft_plan_opts_default(ctypes.byref(o))
    return o


def _edges_arrays(src, dst, w):
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    if not (len(src) == len(dst) == len(w)):
        raise ValueError("src, dst, w must have equal length")
    return src, dst, w


def gft_plan_create(n, src, dst, w, self_loops=None, phi=None, opts=None):
    src, dst, w = _edges_arrays(src, dst, w)
    s = None if self_loops is None else np.ascontiguousarray(self_loops, dtype=np.float64)
    if s is not None and len(s) != n:
        raise ValueError("self_loops must have length n")
    p = None if phi is None else np.ascontiguousarray(phi, dtype=np.int32)
    if p is not None and len(p) != n:
        raise ValueError("phi must have length n")
    h = c_void_p()
    _check(lib().gft_plan_create(ctypes.byref(h), int(n), len(src), _ptr(src), _ptr(dst), _ptr(w),
                                 _ptr(s), _ptr(p), None if opts is None else ctypes.byref(opts)))
    return h


def gft_plan_destroy(h):
    _check(lib().gft_plan_destroy(h))


def gft_plan_serialize(h):
    size = c_size_t()
    _check(lib().gft_plan_serialize(h, None, 0, ctypes.byref(size)))
    buf = ctypes.create_string_buffer(size.value)
    _check(lib().gft_plan_serialize(h, buf, size.value, ctypes.byref(size)))
    return buf.raw[: size.value]


def gft_plan_deserialize(data, opts=None):
    data = bytes(data)
    buf = ctypes.create_string_buffer(data, len(data))
    h = c_void_p()
    _check(lib().gft_plan_deserialize(ctypes.byref(h), buf, len(data),
                                      None if opts is None else ctypes.byref(opts)))
    return h


def _run(fn, h, a, b, batch, dtype, stream):
    dev = None if isinstance(a, int) else a.get_device()
    st = fn(h, _dev_ptr(a), _dev_ptr(b), int(batch), _dtype_code(dtype), _stream_handle(stream, dev))
    if st:
        _check(st)


def gft_forward(h, X, Y, batch, dtype=GFT_F32, stream=None):
    _run(lib().gft_forward, h, X, Y, batch, dtype, stream)


def gft_inverse(h, Y, X, batch, dtype=GFT_F32, stream=None):
    _run(lib().gft_inverse, h, Y, X, batch, dtype, stream)


def gft_dense_forward(h, X, Y, batch, dtype=GFT_F32, stream=None):
    _run(lib().gft_dense_forward, h, X, Y, batch, dtype, stream)


def gft_dense_inverse(h, Y, X, batch, dtype=GFT_F32, stream=None):
    _run(lib().gft_dense_inverse, h, Y, X, batch, dtype, stream)


def gft_execute_host(h, direction, in_host, out_host, batch, dtype, workspace, workspace_bytes,
                     chunk_rows, stream=None):
    _check(lib().gft_execute_host(h, int(direction), c_void_p(in_host.data_ptr()),
                                  c_void_p(out_host.data_ptr()), int(batch), _dtype_code(dtype),
                                  _dev_ptr(workspace), int(workspace_bytes), int(chunk_rows),
                                  _stream_handle(stream)))


def gft_plan_compile(h, dtype, kinds_mask=0):
    _check(lib().gft_plan_compile(h, _dtype_code(dtype), int(kinds_mask)))


GFT_TUNE_GEOMETRY = 1
GFT_TUNE_SUSTAINED = 2


def gft_plan_tune(h, dtype, kinds_mask, X, Y, batch, reps=0, stream=None, flags=0):
    """Returns {kind: (R, stages, warps, pace_ns)} for the kinds tuned (FMA-skeleton kernels)."""
    out = (ctypes.c_int32 * 16)()
    _check(lib().gft_plan_tune(h, _dtype_code(dtype), int(kinds_mask), int(flags), _dev_ptr(X),
                               _dev_ptr(Y), int(batch), int(reps), _stream_handle(stream), out))
    return {k: tuple(out[4 * k: 4 * k + 4]) for k in range(4) if out[4 * k] >= 0}


def gft_filter_tune(f, dtype, X, Y, batch, reps=0, stream=None, flags=0):
    """Returns (R, stages, warps, pace_ns) of the kept filter kernel, or None (tensor cores)."""
    out = (ctypes.c_int32 * 4)()
    _check(lib().gft_filter_tune(f, _dtype_code(dtype), int(flags), _dev_ptr(X), _dev_ptr(Y),
                                 int(batch), int(reps), _stream_handle(stream), out))
    return tuple(out) if out[0] >= 0 else None


def gft_plan_tuning_get(h, dtype, kind):
    """(R, stages, warps, pace_ns, tc_variant) of the kernel (see include/gft.h)."""
    out = (ctypes.c_int32 * 5)()
    _check(lib().gft_plan_tuning_get(h, _dtype_code(dtype), int(kind), out))
    return tuple(out)


def gft_plan_tuning_set(h, dtype, kind, rec):
    """rec: (R, stages, warps, pace_ns[, tc_variant]) -- a 4-tuple means tc_variant -1."""
    if len(rec) not in (4, 5):
        raise ValueError("tuning record: (R, stages, warps, pace_ns[, tc_variant])")
    vals = [int(v) for v in rec] + ([-1] if len(rec) == 4 else [])
    _check(lib().gft_plan_tuning_set(h, _dtype_code(dtype), int(kind), (ctypes.c_int32 * 5)(*vals)))


def gft_plan_info_get(h):
    info = gft_plan_info()
    _check(lib().gft_plan_info_get(h, ctypes.byref(info)))
    return info


def gft_plan_eigenvalues(h, n):
    lam = np.empty(n, dtype=np.float64)
    _check(lib().gft_plan_eigenvalues(h, _ptr(lam)))
    return lam


def gft_plan_basis(h, n):
    U = np.empty((n, n), dtype=np.float64)
    _check(lib().gft_plan_basis(h, _ptr(U)))
    return U


def gft_plan_leaf_sizes(h):
    cnt = c_int32()
    _check(lib().gft_plan_leaf_sizes(h, None, 0, ctypes.byref(cnt)))
    out = np.zeros(cnt.value, dtype=np.int32)
    _check(lib().gft_plan_leaf_sizes(h, _ptr(out), cnt.value, ctypes.byref(cnt)))
    return out.tolist()


def gft_plan_kernel_source(h, kind, dtype=GFT_F32):
    ln = c_size_t()
    _check(lib().gft_plan_kernel_source(h, int(kind), _dtype_code(dtype), None, 0, ctypes.byref(ln)))
    buf = ctypes.create_string_buffer(ln.value + 1)
    _check(lib().gft_plan_kernel_source(h, int(kind), _dtype_code(dtype), buf, ln.value + 1,
                                        ctypes.byref(ln)))
    return buf.value.decode()


def gft_plan_kernel_name(h, kind, dtype=GFT_F32):
    buf = ctypes.create_string_buffer(256)
    _check(lib().gft_plan_kernel_name(h, int(kind), _dtype_code(dtype), buf, 256))
    return buf.value.decode()


def gft_plan_launch_config(h, kind, dtype, batch):
    g, b, s, r = c_int32(), c_int32(), c_int32(), c_int32()
    _check(lib().gft_plan_launch_config(h, int(kind), _dtype_code(dtype), int(batch), ctypes.byref(g),
                                        ctypes.byref(b), ctypes.byref(s), ctypes.byref(r)))
    return {"grid": g.value, "block": b.value, "smem": s.value, "regs": r.value}


def gft_laplacian(n, src, dst, w, self_loops=None):
    src, dst, w = _edges_arrays(src, dst, w)
    s = None if self_loops is None else np.ascontiguousarray(self_loops, dtype=np.float64)
    if s is not None and s.shape != (n,):
        raise ValueError("self_loops must have length n")
    L = np.empty((n, n), dtype=np.float64)
    _check(lib().gft_laplacian(int(n), len(src), _ptr(src), _ptr(dst), _ptr(w), _ptr(s), _ptr(L)))
    return L


def gft_decompose(L, phi, sym_rtol=1e-12):
    L = np.ascontiguousarray(L, dtype=np.float64)
    n = L.shape[0]
    phi = np.ascontiguousarray(phi, dtype=np.int32)
    if L.ndim != 2 or L.shape != (n, n) or phi.shape != (n,):
        raise ValueError("L must be n x n and phi of length n")
    p = int(np.sum(phi > np.arange(n)))
    Lp = np.empty((n - p, n - p), dtype=np.float64)
    Lm = np.empty((p, p), dtype=np.float64)
    pout = c_int32()
    _check(lib().gft_decompose(n, _ptr(L), _ptr(phi), float(sym_rtol), _ptr(Lp), _ptr(Lm),
                               ctypes.byref(pout)))
    return Lp, Lm


def gft_find_involution(L, rtol=1e-10, budget=1000000):
    L = np.ascontiguousarray(L, dtype=np.float64)
    n = L.shape[0]
    if L.ndim != 2 or L.shape != (n, n):
        raise ValueError("L must be n x n")
    phi = np.empty(n, dtype=np.int32)
    p, comp = c_int32(), c_int32()
    _check(lib().gft_find_involution(n, _ptr(L), float(rtol), int(budget), _ptr(phi), ctypes.byref(p),
                                     ctypes.byref(comp)))
    return phi, p.value, bool(comp.value)


def gft_filter_create(plan_h, h, dtypes=("f32", "f64"), flags=0):
    h = np.ascontiguousarray(h, dtype=np.float64)
    mask = 0
    for d in dtypes:
        mask |= 1 << _dtype_code(d)
    fh = c_void_p()
    _check(lib().gft_filter_create(ctypes.byref(fh), plan_h, _ptr(h), mask, int(flags)))
    return fh


def gft_filter_apply(fh, X, Y, batch, dtype=GFT_F32, stream=None):
    _run(lib().gft_filter_apply, fh, X, Y, batch, dtype, stream)


def gft_filter_kernel_name(fh, dtype=GFT_F32):
    buf = ctypes.create_string_buffer(256)
    _check(lib().gft_filter_kernel_name(fh, _dtype_code(dtype), buf, 256))
    return buf.value.decode()


def gft_filter_kernel_source(fh, dtype=GFT_F32):
    ln = c_size_t()
    _check(lib().gft_filter_kernel_source(fh, _dtype_code(dtype), None, 0, ctypes.byref(ln)))
    buf = ctypes.create_string_buffer(ln.value + 1)
    _check(lib().gft_filter_kernel_source(fh, _dtype_code(dtype), buf, ln.value + 1, ctypes.byref(ln)))
    return buf.value.decode()


def gft_filter_destroy(fh):
    _check(lib().gft_filter_destroy(fh))


class Filter:
    """Owner of a gft_filter: fused y = U diag(h) U^T x (one HBM pass)."""

    def __init__(self, plan, h, dtypes=("f32", "f64"), no_cubin_cache=False, no_tensor_cores=False):
        if len(h) != plan.n:
            raise ValueError("h must have length n")
        self.n = plan.n
        flags = (GFT_FLAG_NO_CUBIN_CACHE if no_cubin_cache else 0) | \
                (GFT_FLAG_NO_TENSOR_CORES if no_tensor_cores else 0)
        self._h = gft_filter_create(plan.handle, h, dtypes, flags)

    def apply(self, X, Y=None, stream=None):
        import torch
        if not X.is_cuda or X.dim() != 2 or X.shape[1] != self.n or not X.is_contiguous():
            raise ValueError("expected a contiguous CUDA [batch, %d] tensor" % self.n)
        if Y is None:
            Y = torch.empty_like(X)
        _check_pair(X, Y, self.n, cuda=True)
        dt = GFT_F64 if X.dtype == torch.float64 else GFT_F32
        gft_filter_apply(self._h, X, Y, X.shape[0], dt, stream)
        return Y

    def tune(self, X, Y=None, dtype="f32", reps=0, stream=None, geometry=False, sustained=False):
        """gft_filter_tune on the device tensors X -> Y: (R, stages, warps, pace_ns) kept, or
        None for a tensor-core filter kernel.  sustained=True: GFT_TUNE_SUSTAINED."""
        import torch
        if Y is None:
            Y = torch.empty_like(X)
        _check_pair(X, Y, self.n, cuda=True)
        return gft_filter_tune(self._h, dtype, X, Y, X.shape[0], reps, stream,
                               (GFT_TUNE_GEOMETRY if geometry else 0) | (GFT_TUNE_SUSTAINED if sustained else 0))

    def kernel_name(self, dtype="f32"):
        return gft_filter_kernel_name(self._h, dtype)

    def kernel_source(self, dtype="f32"):
        return gft_filter_kernel_source(self._h, dtype)

    def close(self):
        if getattr(self, "_h", None):
            gft_filter_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- Plan
class Plan:
    """Owner of a gft_plan.  Methods are the C calls of the same name."""

    def __init__(self, n, src, dst, w, self_loops=None, phi=None, *, max_depth=-1, min_leaf=1,
                 search_budget=1000000, sym_rtol=1e-12, dtypes=("f32", "f64"), host_only=False,
                 no_cubin_cache=False, no_tensor_cores=False, normalized=False, dense_tc=False,
                 right_haar=True, approx_layers=-1, approx_min_leaf=2):
        o = gft_plan_opts_default()
        o.approx_layers = approx_layers
        o.approx_min_leaf = approx_min_leaf
        o.max_depth = max_depth
        o.min_leaf = min_leaf
        o.search_budget = search_budget
        o.sym_rtol = sym_rtol
        o.dtypes = 0
        for d in dtypes:
            o.dtypes |= 1 << _dtype_code(d)
        o.flags = ((GFT_FLAG_HOST_ONLY if host_only else 0) | (GFT_FLAG_NO_CUBIN_CACHE if no_cubin_cache else 0)
                   | (GFT_FLAG_NO_TENSOR_CORES if no_tensor_cores else 0)
                   | (GFT_FLAG_NORMALIZED if normalized else 0) | (GFT_FLAG_DENSE_TC if dense_tc else 0)
                   | (0 if right_haar else GFT_FLAG_NO_RIGHT_HAAR))
        self.n = int(n)
        self._h = gft_plan_create(n, src, dst, w, self_loops, phi, o)

    def save(self):
        """The plan as bytes (gft_plan_serialize)."""
        return gft_plan_serialize(self._h)

    @classmethod
    def load(cls, data, *, dtypes=("f32", "f64"), host_only=False, no_cubin_cache=False,
             no_tensor_cores=False, dense_tc=False):
        """Rebuild a plan from Plan.save() bytes (gft_plan_deserialize): no search, no
        eigensolve; kernels regenerated for `dtypes`."""
        o = gft_plan_opts_default()
        o.dtypes = 0
        for d in dtypes:
            o.dtypes |= 1 << _dtype_code(d)
        o.flags = ((GFT_FLAG_HOST_ONLY if host_only else 0) | (GFT_FLAG_NO_CUBIN_CACHE if no_cubin_cache else 0)
                   | (GFT_FLAG_NO_TENSOR_CORES if no_tensor_cores else 0) | (GFT_FLAG_DENSE_TC if dense_tc else 0))
        self = cls.__new__(cls)
        self._h = gft_plan_deserialize(data, o)
        self.n = self.info()["n"]
        return self

    @classmethod
    def from_config(cls, cfg, **kw):
        kw.setdefault("max_depth", cfg.max_depth)
        kw.setdefault("dtypes", cfg.dtypes)
        return cls(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops, cfg.phi, **kw)

    def close(self):
        if getattr(self, "_h", None):
            gft_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # hot path: torch CUDA tensors [batch, n], float32 or float64
    def forward(self, X, Y=None, stream=None):
        return self._apply(gft_forward, X, Y, stream)

    def inverse(self, Y, X=None, stream=None):
        return self._apply(gft_inverse, Y, X, stream)

    def dense_forward(self, X, Y=None, stream=None):
        return self._apply(gft_dense_forward, X, Y, stream)

    def dense_inverse(self, Y, X=None, stream=None):
        return self._apply(gft_dense_inverse, Y, X, stream)

    def _apply(self, fn, a, b, stream):
        import torch
        if not a.is_cuda:
            raise ValueError("device tensors required (use execute_host for host buffers)")
        shape = a.shape
        if len(shape) != 2 or shape[1] != self.n or not a.is_contiguous():
            raise ValueError("expected a contiguous [batch, %d] tensor" % self.n)
        if b is None:
            b = torch.empty_like(a)
        adt = a.dtype
        if b.dtype != adt or (adt is not torch.float32 and adt is not torch.float64):
            raise ValueError("float32/float64 tensors of equal dtype required")
        _check_pair(a, b, self.n, cuda=True)
        fn(self._h, a, b, shape[0], GFT_F64 if adt is torch.float64 else GFT_F32, stream)
        return b

    def execute_host(self, direction, in_host, out_host, workspace, chunk_rows, stream=None):
        import torch
        _check_pair(in_host, out_host, self.n, cuda=False)
        if not isinstance(workspace, torch.Tensor) or not workspace.is_cuda or not workspace.is_contiguous():
            raise ValueError("workspace: a contiguous CUDA tensor is required")
        dt = GFT_F64 if in_host.dtype == torch.float64 else GFT_F32
        gft_execute_host(self._h, direction, in_host, out_host, in_host.shape[0], dt, workspace,
                         workspace.numel() * workspace.element_size(), chunk_rows, stream)
        return out_host

    def compile(self, dtype="f32", kinds=(0, 1, 2, 3)):
        gft_plan_compile(self._h, dtype, sum(1 << k for k in kinds))

    def tune(self, dtype="f32", kinds=(0, 1), X=None, Y=None, batch=None, reps=0, stream=None,
             geometry=False, sustained=False):
        """gft_plan_tune on the device tensors X -> Y (or on scratch buffers of `batch` rows,
        default 256 MiB of rows, > L2); geometry=True also searches the warp-tile geometry;
        sustained=True (GFT_TUNE_SUSTAINED) times the candidates after >= 1 s of load.
        Returns {kind: (R, stages, warps, pace_ns)} for the kinds on the FMA skeleton."""
        import torch
        tdt = torch.float64 if dtype == "f64" else torch.float32
        if X is None:
            if batch is None:
                batch = max(1 << 16, (256 << 20) // (self.n * (8 if dtype == "f64" else 4)))
            X = torch.randn(batch, self.n, device="cuda", dtype=tdt)
        if Y is None:
            Y = torch.empty_like(X)
        if X.dtype != tdt or Y.dtype != tdt or X.shape[1] != self.n or Y.shape != X.shape:
            raise ValueError("X, Y: [batch, %d] tensors of the tuned dtype" % self.n)
        _check_pair(X, Y, self.n, cuda=True)
        return gft_plan_tune(self._h, dtype, sum(1 << k for k in kinds), X, Y, X.shape[0], reps, stream,
                             (GFT_TUNE_GEOMETRY if geometry else 0) | (GFT_TUNE_SUSTAINED if sustained else 0))

    def tuning(self, dtype="f32", kinds=(0, 1, 2, 3)):
        """Tuning records {kind: (R, stages, warps, pace_ns, tc_variant)}."""
        return {k: gft_plan_tuning_get(self._h, dtype, k) for k in kinds}

    def set_tuning(self, record, dtype="f32"):
        """Re-apply records from tuning() (4-tuples: FMA geometry with tc_variant -1)."""
        for k, rec in record.items():
            gft_plan_tuning_set(self._h, dtype, int(k), rec)

    def info(self):
        return gft_plan_info_get(self._h).as_dict()

    def eigenvalues(self):
        return gft_plan_eigenvalues(self._h, self.n)

    def basis(self):
        return gft_plan_basis(self._h, self.n)

    def leaf_sizes(self):
        return gft_plan_leaf_sizes(self._h)

    def kernel_source(self, kind, dtype="f32"):
        return gft_plan_kernel_source(self._h, kind, dtype)

    def kernel_name(self, kind, dtype="f32"):
        return gft_plan_kernel_name(self._h, kind, dtype)

    def launch_config(self, kind, dtype, batch):
        return gft_plan_launch_config(self._h, kind, dtype, batch)
