"""Thin Python binding of libmaddness (include/maddness.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels. There is no CPU fallback -- importing this package without
the built ``libmaddness.so`` raises, and calls without a CUDA device fail.

Names mirror the C ABI: ``mdn_model_load``, ``mdn_build_luts``,
``mdn_luts_serialize``, ``mdn_luts_load``, ``mdn_encode``, ``mdn_scan``,
``mdn_amm``, ``mdn_exec_create``, ``mdn_amm_host``.
Device buffers are torch CUDA tensors (PyTorch is used for device memory and
streams only); host buffers are numpy arrays or CPU tensors.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# MDN_LIB: an in-tree variant build (build.py --variant NAME) for A/B experiments
LIB_PATH = os.path.join(_PKG, os.environ.get("MDN_LIB", "libmaddness.so"))

MDN_SUM_EXACT = 0
MDN_SUM_AVG = 1
K = 16

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libmaddness.so not built at {LIB_PATH}; run `python paper_2106_10860_b200/build.py` "
        "(there is no CPU fallback)")

_lib = ct.CDLL(LIB_PATH)

_vp, _sz, _i64, _i32 = ct.c_void_p, ct.c_size_t, ct.c_int64, ct.c_int
_SIGS = {
    "mdn_model_load": (_i32, [_vp, _sz, _i32, ct.POINTER(_vp), ct.POINTER(_sz)]),
    "mdn_model_free": (None, [_vp]),
    "mdn_model_info": (_i32, [_vp, ct.POINTER(_i32), ct.POINTER(_i32), ct.POINTER(ct.c_uint64)]),
    "mdn_build_luts": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, ct.POINTER(_vp)]),
    "mdn_luts_serialize": (_i32, [_vp, _vp, ct.POINTER(_sz)]),
    "mdn_luts_load": (_i32, [_vp, _sz, _i32, ct.POINTER(_vp), ct.POINTER(_sz)]),
    "mdn_luts_free": (None, [_vp]),
    "mdn_luts_info": (_i32, [_vp, ct.POINTER(_i32), ct.POINTER(_i32), ct.POINTER(_i32),
                             ct.POINTER(_i32), ct.POINTER(_i32), ct.POINTER(ct.c_float),
                             ct.POINTER(ct.c_float), ct.POINTER(ct.c_uint64)]),
    "mdn_encode": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "mdn_scan": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "mdn_amm": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "mdn_exec_create": (_i32, [_vp, _vp, _i64, _i32, ct.POINTER(_vp)]),
    "mdn_exec_free": (None, [_vp]),
    "mdn_amm_host": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64]),
    "mdn_status_str": (ct.c_char_p, [_i32]),
    "mdn_abi_version": (_i32, []),
    "mdn_amm_variant": (_i32, [_vp, _vp, _i64, ct.c_char_p, _sz]),
    "mdn_stream_probe": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp]),
    "mdn_amm_probe": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "mdn_encode_u8": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "mdn_amm_u8": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "mdn_encode_cm": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "mdn_amm_cm": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "mdn_encode_pq": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "mdn_amm_host_u8": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64]),
    "mdn_amm_cm_host": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64]),
    "mdn_encode_host": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "mdn_scan_host": (_i32, [_vp, _vp, _i64, _vp, _i64]),
    "mdn_encode_host_u8": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "mdn_encode_cm_host": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "mdn_encode_pq_host": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "mdn_amm_pq_host": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64]),
    "mdn_train": (_i32, [_vp, _i64, _i64, _i32, _i32, ct.c_double, _i32, _vp, ct.POINTER(_sz)]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class MdnError(RuntimeError):
    def __init__(self, status: int, where: str, err_off=None):
        msg = f"{where}: {_lib.mdn_status_str(status).decode()} ({status})"
        if err_off is not None:
            msg += f" at byte {err_off}"
        super().__init__(msg)
        self.status = status
        self.err_off = err_off


def _check(st, where, err_off=None):
    if st != 0:
        raise MdnError(st, where, err_off)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _dev_ptr(t, dtype_name, what):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA torch.Tensor")
    if str(t.dtype) != f"torch.{dtype_name}":
        raise TypeError(f"{what} must be {dtype_name}, got {t.dtype}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{what} must be 2-D with unit column stride")
    return t.data_ptr()


# --------------------------------------------------------------- handles --

class Model:
    """Opaque mdn_model handle (trees + prototypes resident on one device)."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = device
        C, D, fp = _i32(), _i32(), ct.c_uint64()
        _check(_lib.mdn_model_info(self._h, ct.byref(C), ct.byref(D), ct.byref(fp)), "mdn_model_info")
        self.C, self.D, self.fingerprint = C.value, D.value, fp.value

    def close(self):
        if self._h and _lib is not None:      # _lib is None during interpreter teardown
            _lib.mdn_model_free(self._h)
            self._h = None

    __del__ = close


class Luts:
    """Opaque mdn_luts handle (quantised tables + alpha, beta on one device)."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = device
        v = [_i32() for _ in range(5)]
        a, b, fp = ct.c_float(), ct.c_float(), ct.c_uint64()
        _check(_lib.mdn_luts_info(self._h, *[ct.byref(x) for x in v], ct.byref(a), ct.byref(b),
                                  ct.byref(fp)), "mdn_luts_info")
        self.C, self.M, self.mode, self.U, self.l = (x.value for x in v)
        self.alpha, self.beta32, self.model_fingerprint = np.float32(a.value), np.float32(b.value), fp.value

    def close(self):
        if self._h and _lib is not None:
            _lib.mdn_luts_free(self._h)
            self._h = None

    __del__ = close


class Exec:
    """Opaque mdn_exec handle: pipelined host-buffer executor (e2e path)."""

    def __init__(self, handle, model, luts):
        self._h, self._model, self._luts = handle, model, luts

    def close(self):
        if self._h and _lib is not None:
            _lib.mdn_exec_free(self._h)
            self._h = None

    __del__ = close


# ------------------------------------------------------------- functions --

def mdn_model_load(buf: bytes, device: int = 0) -> Model:
    h, off = _vp(), _sz(0)
    st = _lib.mdn_model_load(buf, len(buf), device, ct.byref(h), ct.byref(off))
    _check(st, "mdn_model_load", off.value if st == -3 else None)
    return Model(h, device)


def mdn_train(A, C: int, lam: float = 1.0) -> bytes:
    """GPU training: A is the CUDA fp32 training matrix A~ (N x D);
    returns the "model.mdnm v1" bytes (load with mdn_model_load)."""
    pa = _dev_ptr(A, "float32", "A")
    n = _sz(0)
    D = A.shape[1]
    _check(_lib.mdn_train(None, 0, 0, D, C, lam, A.device.index or 0, None, ct.byref(n)), "mdn_train")
    buf = ct.create_string_buffer(n.value)
    _check(_lib.mdn_train(pa, A.shape[0], A.stride(0), D, C, lam, A.device.index or 0, buf,
                          ct.byref(n)), "mdn_train")
    return buf.raw[:n.value]


def mdn_build_luts(model: Model, B, mode: int = MDN_SUM_EXACT, U: int = 16) -> Luts:
    B = np.ascontiguousarray(np.asarray(B, dtype=np.float32))
    h = _vp()
    _check(_lib.mdn_build_luts(model._h, B.ctypes.data, B.shape[1], B.shape[1], mode, U,
                               ct.byref(h)), "mdn_build_luts")
    return Luts(h, model.device)


def mdn_luts_serialize(luts: Luts) -> bytes:
    n = _sz(0)
    _check(_lib.mdn_luts_serialize(luts._h, None, ct.byref(n)), "mdn_luts_serialize")
    buf = ct.create_string_buffer(n.value)
    _check(_lib.mdn_luts_serialize(luts._h, buf, ct.byref(n)), "mdn_luts_serialize")
    return buf.raw[:n.value]


def mdn_luts_load(buf: bytes, device: int = 0) -> Luts:
    h, off = _vp(), _sz(0)
    st = _lib.mdn_luts_load(buf, len(buf), device, ct.byref(h), ct.byref(off))
    _check(st, "mdn_luts_load", off.value if st == -3 else None)
    return Luts(h, device)


def mdn_encode(model: Model, A, codes, stream=None):
    pa = _dev_ptr(A, "float32", "A")
    pc = _dev_ptr(codes, "uint8", "codes")
    if codes.shape != (A.shape[0], (model.C + 1) // 2) or not codes.is_contiguous():
        raise ValueError("codes must be contiguous N x ceil(C/2)")
    _check(_lib.mdn_encode(model._h, pa, A.shape[0], A.stride(0), pc, _stream_ptr(stream)),
           "mdn_encode")
    return codes


def mdn_scan(luts: Luts, codes, sums=None, out=None, stream=None):
    pc = _dev_ptr(codes, "uint8", "codes")
    N = codes.shape[0]
    ps = po = None
    ldo = luts.M
    if sums is not None:
        ps = _dev_ptr(sums, "int32", "sums")
        if sums.shape != (N, luts.M) or not sums.is_contiguous():
            raise ValueError("sums must be contiguous N x M")
    if out is not None:
        po = _dev_ptr(out, "float32", "out")
        if out.shape != (N, luts.M):
            raise ValueError("out must be N x M")
        ldo = out.stride(0)
    _check(_lib.mdn_scan(luts._h, pc, N, ps, po, ldo, _stream_ptr(stream)), "mdn_scan")
    return sums, out


def mdn_amm(model: Model, luts: Luts, A, out, stream=None):
    pa = _dev_ptr(A, "float32", "A")
    po = _dev_ptr(out, "float32", "out")
    if out.shape != (A.shape[0], luts.M):
        raise ValueError("out must be N x M")
    _check(_lib.mdn_amm(model._h, luts._h, pa, A.shape[0], A.stride(0), po, out.stride(0),
                        _stream_ptr(stream)), "mdn_amm")
    return out


def mdn_encode_u8(model: Model, A, codes, stream=None):
    """g for natively 8-bit A (App. B 8-bit split values)."""
    pa = _dev_ptr(A, "uint8", "A")
    pc = _dev_ptr(codes, "uint8", "codes")
    if codes.shape != (A.shape[0], (model.C + 1) // 2) or not codes.is_contiguous():
        raise ValueError("codes must be contiguous N x ceil(C/2)")
    _check(_lib.mdn_encode_u8(model._h, pa, A.shape[0], A.stride(0), pc, _stream_ptr(stream)),
           "mdn_encode_u8")
    return codes


def mdn_amm_u8(model: Model, luts: Luts, A, out, stream=None):
    """Fused g + f + dequant for natively 8-bit A."""
    pa = _dev_ptr(A, "uint8", "A")
    po = _dev_ptr(out, "float32", "out")
    if out.shape != (A.shape[0], luts.M):
        raise ValueError("out must be N x M")
    _check(_lib.mdn_amm_u8(model._h, luts._h, pa, A.shape[0], A.stride(0), po, out.stride(0),
                           _stream_ptr(stream)), "mdn_amm_u8")
    return out


def mdn_encode_pq(model: Model, A, codes, stream=None):
    """g(A) of the PQ comparator (PAPER.md Eq. pqLoss);
    `model` must be a PQ model (flags bit1)."""
    pa = _dev_ptr(A, "float32", "A")
    pc = _dev_ptr(codes, "uint8", "codes")
    if codes.shape != (A.shape[0], (model.C + 1) // 2) or not codes.is_contiguous():
        raise ValueError("codes must be contiguous N x ceil(C/2)")
    _check(_lib.mdn_encode_pq(model._h, pa, A.shape[0], A.stride(0), pc, _stream_ptr(stream)),
           "mdn_encode_pq")
    return codes


def _colmajor(At, what):
    """At: D x N CUDA float32 tensor with unit column stride (A column-major)."""
    pa = _dev_ptr(At, "float32", what)
    return pa, At.shape[1], At.stride(0)


def mdn_encode_cm(model: Model, At, codes, stream=None):
    """g for column-major A: At = A^T, D x N."""
    pa, N, ldt = _colmajor(At, "At")
    pc = _dev_ptr(codes, "uint8", "codes")
    if At.shape[0] != model.D:
        raise ValueError("At must be D x N")
    if codes.shape != (N, (model.C + 1) // 2) or not codes.is_contiguous():
        raise ValueError("codes must be contiguous N x ceil(C/2)")
    _check(_lib.mdn_encode_cm(model._h, pa, N, ldt, pc, _stream_ptr(stream)), "mdn_encode_cm")
    return codes


def mdn_amm_cm(model: Model, luts: Luts, At, out, stream=None):
    """Fused g + f + dequant for column-major A (At = A^T, D x N); out is N x M."""
    pa, N, ldt = _colmajor(At, "At")
    po = _dev_ptr(out, "float32", "out")
    if At.shape[0] != model.D:
        raise ValueError("At must be D x N")
    if out.shape != (N, luts.M):
        raise ValueError("out must be N x M")
    _check(_lib.mdn_amm_cm(model._h, luts._h, pa, N, ldt, po, out.stride(0), _stream_ptr(stream)),
           "mdn_amm_cm")
    return out


def mdn_amm_variant(model: Model, luts: Luts, lda: int) -> str:
    buf = ct.create_string_buffer(64)
    _check(_lib.mdn_amm_variant(model._h, luts._h, lda, buf, 64), "mdn_amm_variant")
    return buf.value.decode()


def mdn_exec_create(model: Model, luts: Luts, chunk_rows: int = 1 << 18, n_slots: int = 3) -> Exec:
    h = _vp()
    _check(_lib.mdn_exec_create(model._h, luts._h, chunk_rows, n_slots, ct.byref(h)),
           "mdn_exec_create")
    return Exec(h, model, luts)


def _host_ptr(x, what):
    if isinstance(x, np.ndarray):
        if x.dtype != np.float32 or x.ndim != 2 or x.strides[1] != 4:
            raise TypeError(f"{what} must be a 2-D float32 array with unit column stride")
        return x.ctypes.data, x.strides[0] // 4, x.shape
    import torch
    if isinstance(x, torch.Tensor) and not x.is_cuda and x.dtype == torch.float32 and x.dim() == 2 \
            and x.stride(1) == 1:
        return x.data_ptr(), x.stride(0), tuple(x.shape)
    raise TypeError(f"{what} must be host float32 (numpy or CPU tensor)")


def mdn_amm_host(ex: Exec, A_host, out_host):
    pa, lda, sa = _host_ptr(A_host, "A_host")
    po, ldo, so = _host_ptr(out_host, "out_host")
    if so[0] != sa[0]:
        raise ValueError("row count mismatch")
    _check(_lib.mdn_amm_host(ex._h, pa, sa[0], lda, po, ldo), "mdn_amm_host")
    return out_host


def mdn_amm_host_u8(ex: Exec, A_host, out_host):
    """Host-buffer pipeline for 8-bit rows: A_host uint8 (numpy or
    CPU tensor, unit column stride), out_host float32."""
    import torch
    if isinstance(A_host, np.ndarray):
        if A_host.dtype != np.uint8 or A_host.ndim != 2 or A_host.strides[1] != 1:
            raise TypeError("A_host must be a 2-D uint8 array with unit column stride")
        pa, lda, sa = A_host.ctypes.data, A_host.strides[0], A_host.shape
    elif isinstance(A_host, torch.Tensor) and not A_host.is_cuda and A_host.dtype == torch.uint8 \
            and A_host.dim() == 2 and A_host.stride(1) == 1:
        pa, lda, sa = A_host.data_ptr(), A_host.stride(0), tuple(A_host.shape)
    else:
        raise TypeError("A_host must be host uint8 (numpy or CPU tensor)")
    po, ldo, so = _host_ptr(out_host, "out_host")
    if so[0] != sa[0]:
        raise ValueError("row count mismatch")
    _check(_lib.mdn_amm_host_u8(ex._h, pa, sa[0], lda, po, ldo), "mdn_amm_host_u8")
    return out_host


def _host_u8(x, what):
    import torch
    if isinstance(x, np.ndarray) and x.dtype == np.uint8 and x.ndim == 2 and x.flags["C_CONTIGUOUS"]:
        return x.ctypes.data, x.shape
    if isinstance(x, torch.Tensor) and not x.is_cuda and x.dtype == torch.uint8 and x.dim() == 2 \
            and x.is_contiguous():
        return x.data_ptr(), tuple(x.shape)
    raise TypeError(f"{what} must be a contiguous 2-D host uint8 array")


def mdn_encode_host(ex: Exec, A_host, codes_host):
    """g through the executor: host fp32 rows -> host packed codes."""
    pa, lda, sa = _host_ptr(A_host, "A_host")
    pc, sc = _host_u8(codes_host, "codes_host")
    if sc != (sa[0], (ex._model.C + 1) // 2):
        raise ValueError("codes_host must be N x ceil(C/2)")
    _check(_lib.mdn_encode_host(ex._h, pa, sa[0], lda, pc), "mdn_encode_host")
    return codes_host


def mdn_encode_host_u8(ex: Exec, A_host, codes_host):
    """g on 8-bit host rows through the executor."""
    import torch
    if isinstance(A_host, np.ndarray) and A_host.dtype == np.uint8 and A_host.ndim == 2 \
            and A_host.strides[1] == 1:
        pa, lda, sa = A_host.ctypes.data, A_host.strides[0], A_host.shape
    elif isinstance(A_host, torch.Tensor) and not A_host.is_cuda and A_host.dtype == torch.uint8 \
            and A_host.dim() == 2 and A_host.stride(1) == 1:
        pa, lda, sa = A_host.data_ptr(), A_host.stride(0), tuple(A_host.shape)
    else:
        raise TypeError("A_host must be host uint8 (numpy or CPU tensor)")
    pc, sc = _host_u8(codes_host, "codes_host")
    if sc != (sa[0], (ex._model.C + 1) // 2):
        raise ValueError("codes_host must be N x ceil(C/2)")
    _check(_lib.mdn_encode_host_u8(ex._h, pa, sa[0], lda, pc), "mdn_encode_host_u8")
    return codes_host


def mdn_scan_host(ex: Exec, codes_host, out_host):
    """f through the executor: host packed codes -> host fp32 out."""
    pc, sc = _host_u8(codes_host, "codes_host")
    po, ldo, so = _host_ptr(out_host, "out_host")
    if sc[1] != (ex._model.C + 1) // 2 or so[0] != sc[0]:
        raise ValueError("codes_host N x ceil(C/2), out_host N x M")
    _check(_lib.mdn_scan_host(ex._h, pc, sc[0], po, ldo), "mdn_scan_host")
    return out_host


def mdn_amm_cm_host(ex: Exec, At_host, out_host):
    """Host-buffer pipeline for column-major A: At_host float32
    D x N (numpy or CPU tensor, unit column stride, row stride >= N); only the
    model's split columns are copied to the device."""
    pa, ldt, sa = _host_ptr(At_host, "At_host")
    po, ldo, so = _host_ptr(out_host, "out_host")
    if sa[0] != ex._model.D:
        raise ValueError("At_host must be D x N")
    if so[0] != sa[1]:
        raise ValueError("row count mismatch")
    _check(_lib.mdn_amm_cm_host(ex._h, pa, sa[1], ldt, po, ldo), "mdn_amm_cm_host")
    return out_host


def mdn_encode_cm_host(ex: Exec, At_host, codes_host):
    """g on column-major host A through the executor (split columns only)."""
    pa, ldt, sa = _host_ptr(At_host, "At_host")
    pc, sc = _host_u8(codes_host, "codes_host")
    if sa[0] != ex._model.D:
        raise ValueError("At_host must be D x N")
    if sc != (sa[1], (ex._model.C + 1) // 2):
        raise ValueError("codes_host must be N x ceil(C/2)")
    _check(_lib.mdn_encode_cm_host(ex._h, pa, sa[1], ldt, pc), "mdn_encode_cm_host")
    return codes_host


def mdn_encode_pq_host(ex: Exec, A_host, codes_host):
    """PQ encode of host rows through a PQ executor."""
    pa, lda, sa = _host_ptr(A_host, "A_host")
    pc, sc = _host_u8(codes_host, "codes_host")
    if sc != (sa[0], (ex._model.C + 1) // 2):
        raise ValueError("codes_host must be N x ceil(C/2)")
    _check(_lib.mdn_encode_pq_host(ex._h, pa, sa[0], lda, pc), "mdn_encode_pq_host")
    return codes_host


def mdn_amm_pq_host(ex: Exec, A_host, out_host):
    """PQ encode + scan + dequant of host rows through a PQ executor."""
    pa, lda, sa = _host_ptr(A_host, "A_host")
    po, ldo, so = _host_ptr(out_host, "out_host")
    if so[0] != sa[0]:
        raise ValueError("row count mismatch")
    _check(_lib.mdn_amm_pq_host(ex._h, pa, sa[0], lda, po, ldo), "mdn_amm_pq_host")
    return out_host


def mdn_stream_probe(A, out, stream=None):
    """Diagnostics: stream A (read) and out (write) with the fused path's byte mix."""
    pa = _dev_ptr(A, "float32", "A")
    po = _dev_ptr(out, "float32", "out")
    _check(_lib.mdn_stream_probe(pa, A.shape[0], A.stride(0), A.shape[1], po, out.stride(0),
                                 out.shape[1], _stream_ptr(stream)), "mdn_stream_probe")
    return out


def mdn_amm_probe(model: Model, luts: Luts, A, out, stream=None):
    """Diagnostics: mdn_amm's own pipeline with encode and scan removed (the
    data-movement ceiling of the fused kernel); out = beta32 everywhere."""
    pa = _dev_ptr(A, "float32", "A")
    po = _dev_ptr(out, "float32", "out")
    if out.shape != (A.shape[0], luts.M):
        raise ValueError("out must be N x M")
    _check(_lib.mdn_amm_probe(model._h, luts._h, pa, A.shape[0], A.stride(0), po, out.stride(0),
                              _stream_ptr(stream)), "mdn_amm_probe")
    return out


def abi_version() -> int:
    return _lib.mdn_abi_version()
