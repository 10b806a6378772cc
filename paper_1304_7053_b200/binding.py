"""Thin Python binding of libtxgemm.so (include/txgemm.h).

Argument marshalling only: every step of the batched GEMM runs in the CUDA
kernels behind the C ABI.  There is no CPU fallback -- if the extension is
missing, every call raises.  PyTorch is used for device memory and streams.

Two levels:
  * the C functions under their own names, e.g. ``tx_gemm_batched_s(transa,
    transb, m, n, k, alpha, A, lda, lda2, B, ldb, ldb2, beta, C, ldc, ldc2,
    batch_count, stream)`` where A/B/C are device addresses (int) or tensors;
  * ``gemm_batched(A, B, C, ...)`` on (batch, rows, cols) tensor views whose
    matrices are column-major (``stride(1) == 1``), e.g.
    ``torch.empty(N, cols, rows).transpose(1, 2)``; ld = stride(2), ld2 = stride(0).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TXGEMM_LIB") or os.path.join(_HERE, "libtxgemm.so")

KINDS = ("s", "d", "c", "z")
PATHS = {0: "none", 1: "bulk", 2: "gather", 3: "ptr", 4: "scale", 5: "direct", 6: "tc", 22: "tc+tail", 17: "bulk+tail",
         33: "bulk", 34: "gather", 35: "ptr", 49: "bulk+tail"}


class TxError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"txgemm status {status}: {msg}")
        self.status = status


class _CF(ctypes.Structure):
    _fields_ = [("re", ctypes.c_float), ("im", ctypes.c_float)]


class _CD(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


_SCALAR = {"s": ctypes.c_float, "d": ctypes.c_double, "c": _CF, "z": _CD}
_lock = threading.Lock()
_lib = None


def build(jobs: int | None = None, extra_nvflags: str = "") -> str:
    """Compile the library in-tree with nvcc for sm_100a (make; see Makefile)."""
    cmd = ["make", "-C", _HERE, f"-j{jobs or os.cpu_count() or 8}"]
    if extra_nvflags:
        cmd.append(f"EXTRA_NVFLAGS={extra_nvflags}")
    subprocess.check_call(cmd, stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib():
    """Load libtxgemm.so.  Raises if it is missing: there is no fallback path."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built (run paper_1304_7053_b200.binding.build() "
                              "or `make -C paper_1304_7053_b200`); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, ci, cll, cc = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_char
        for k in KINDS:
            f = getattr(L, f"tx_gemm_batched_{k}")
            f.argtypes = [cc, cc, ci, ci, ci, vp, vp, ci, cll, vp, ci, cll, vp, vp, ci, cll, ci, vp]
            f.restype = ci
            g = getattr(L, f"tx_gemm_batched_ptr_{k}")
            g.argtypes = [cc, cc, ci, ci, ci, vp, vp, ci, vp, ci, vp, vp, ci, ci, vp]
            g.restype = ci
            h = getattr(L, f"tx_gemm_batched_hostio_{k}")
            h.argtypes = [cc, cc, ci, ci, ci, vp, vp, ci, cll, vp, ci, cll, vp, vp, ci, cll, ci, vp,
                          vp, vp, vp]
            h.restype = ci
        for k in KINDS:
            f = getattr(L, f"tx_gemm_batched_dev_{k}")
            f.argtypes = [cc, cc, ci, ci, ci, vp, vp, ci, cll, vp, ci, cll, vp, vp, ci, cll, ci, vp]
            f.restype = ci
            g = getattr(L, f"tx_gemm_batched_ptr_dev_{k}")
            g.argtypes = [cc, cc, ci, ci, ci, vp, vp, ci, vp, ci, vp, vp, ci, ci, vp]
            g.restype = ci
        L.tx_status_string.argtypes = [ci]
        L.tx_status_string.restype = ctypes.c_char_p
        L.tx_version.restype = ci
        L.tx_last_path.argtypes = [ctypes.POINTER(ci)]
        L.tx_last_path.restype = ci
        L.tx_set_max_ctas.argtypes = [ci]
        L.tx_set_max_ctas.restype = ci
        L.tx_num_instances.restype = ci
        L.tx_set_tuning.argtypes = [ci, ci]
        L.tx_set_tuning.restype = ci
        L.tx_set_jit.argtypes = [ci]
        L.tx_set_jit.restype = ci
        L.tx_set_tc.argtypes = [ci]
        L.tx_set_tc.restype = ci
        L.tx_jit_compiled.restype = ci
        L.tx_prepare.argtypes = [cc, cc, cc, ci, ci, ci, ci, ci]
        L.tx_prepare.restype = ci
        _lib = L
        return L


# ------------------------------------------------------------------ helpers
def _addr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()  # torch tensor


def _scalar(kind, v):
    v = complex(v)
    if kind in ("s", "d"):
        if v.imag != 0:
            raise ValueError("complex alpha/beta for a real kind")
        return _SCALAR[kind](v.real)
    return _SCALAR[kind](v.real, v.imag)


def _op(c):
    return c.encode() if isinstance(c, str) else bytes([c])


def _stream(stream):
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(rc):
    if rc != 0:
        raise TxError(rc, status_string(rc))
    return rc


def status_string(status: int) -> str:
    return lib().tx_status_string(status).decode()


def version() -> int:
    return lib().tx_version()


def last_path():
    """(path name, launches) of this thread's most recent successful call."""
    n = ctypes.c_int(0)
    p = lib().tx_last_path(ctypes.byref(n))
    return PATHS.get(p, str(p)), n.value


def last_path_jit() -> bool:
    """True when the most recent call ran a runtime-specialised (NVRTC) instance."""
    return bool(lib().tx_last_path(None) & 32)


def set_jit(enable: bool) -> int:
    return lib().tx_set_jit(1 if enable else 0)


def set_tc(mode: int) -> int:
    """Tensor-core split-TF32 kernel for packed s / c: -1 automatic, 0 never, 1 wherever
    it applies.  Returns the previous setting."""
    return lib().tx_set_tc(int(mode))


def jit_compiled() -> int:
    return lib().tx_jit_compiled()


def set_max_ctas(v: int) -> int:
    return lib().tx_set_max_ctas(int(v))


def set_tuning(stages: int = 0, stage_kb: int = 0) -> int:
    """Autotuning hook (tx_set_tuning): force pipeline depth / stage size; 0, 0 resets."""
    return lib().tx_set_tuning(int(stages), int(stage_kb))


def num_instances() -> int:
    return lib().tx_num_instances()


LAYOUTS = {"packed": 0, "strided": 1, "ptr": 2}


def prepare(kind, transa, transb, m, n, k, beta_zero=False, layout="packed") -> int:
    """tx_prepare: build the runtime-specialised instances a call of this shape would
    use on the current device, so the first real call does no compilation."""
    return lib().tx_prepare(_op(kind), _op(transa), _op(transb), m, n, k, 1 if beta_zero else 0,
                            LAYOUTS[layout] if isinstance(layout, str) else int(layout))


# ------------------------------------------------------ raw C-ABI mirrors
def tx_gemm_batched(kind, transa, transb, m, n, k, alpha, A, lda, lda2, B, ldb, ldb2, beta, C,
                    ldc, ldc2, batch_count, stream=None, alpha_ptr=True, beta_ptr=True):
    """Strided call; returns the status code (0 or -argpos or cudaError_t)."""
    a, b = _scalar(kind, alpha), _scalar(kind, beta)
    return getattr(lib(), f"tx_gemm_batched_{kind}")(
        _op(transa), _op(transb), m, n, k, ctypes.addressof(a) if alpha_ptr else None, _addr(A),
        lda, lda2, _addr(B), ldb, ldb2, ctypes.addressof(b) if beta_ptr else None, _addr(C), ldc,
        ldc2, batch_count, _stream(stream))


def tx_gemm_batched_ptr(kind, transa, transb, m, n, k, alpha, Aarray, lda, Barray, ldb, beta,
                        Carray, ldc, batch_count, stream=None, alpha_ptr=True, beta_ptr=True):
    """Pointer-array call; X_array are device int64 tensors of addresses (or ints)."""
    a, b = _scalar(kind, alpha), _scalar(kind, beta)
    return getattr(lib(), f"tx_gemm_batched_ptr_{kind}")(
        _op(transa), _op(transb), m, n, k, ctypes.addressof(a) if alpha_ptr else None,
        _addr(Aarray), lda, _addr(Barray), ldb, ctypes.addressof(b) if beta_ptr else None,
        _addr(Carray), ldc, batch_count, _stream(stream))


def tx_gemm_batched_hostio(kind, transa, transb, m, n, k, alpha, hA, lda, lda2, hB, ldb, ldb2,
                           beta, hC, ldc, ldc2, batch_count, stream, dA, dB, dC):
    a, b = _scalar(kind, alpha), _scalar(kind, beta)
    return getattr(lib(), f"tx_gemm_batched_hostio_{kind}")(
        _op(transa), _op(transb), m, n, k, ctypes.addressof(a), _addr(hA), lda, lda2, _addr(hB),
        ldb, ldb2, ctypes.addressof(b), _addr(hC), ldc, ldc2, batch_count, _stream(stream),
        _addr(dA), _addr(dB), _addr(dC))


def tx_gemm_batched_dev(kind, transa, transb, m, n, k, alpha_dev, A, lda, lda2, B, ldb, ldb2,
                        beta_dev, C, ldc, ldc2, batch_count, stream=None):
    """Strided call with DEVICE-resident alpha / beta (device addresses or 1-element tensors)."""
    return getattr(lib(), f"tx_gemm_batched_dev_{kind}")(
        _op(transa), _op(transb), m, n, k, _addr(alpha_dev), _addr(A), lda, lda2, _addr(B), ldb,
        ldb2, _addr(beta_dev), _addr(C), ldc, ldc2, batch_count, _stream(stream))


def tx_gemm_batched_ptr_dev(kind, transa, transb, m, n, k, alpha_dev, Aarray, lda, Barray, ldb,
                            beta_dev, Carray, ldc, batch_count, stream=None):
    return getattr(lib(), f"tx_gemm_batched_ptr_dev_{kind}")(
        _op(transa), _op(transb), m, n, k, _addr(alpha_dev), _addr(Aarray), lda, _addr(Barray),
        ldb, _addr(beta_dev), _addr(Carray), ldc, batch_count, _stream(stream))


def _named(kind, fn):
    def f(*args, **kw):
        return fn(kind, *args, **kw)

    f.__name__ = f"{fn.__name__}_{kind}"
    f.__doc__ = f"{fn.__name__} for kind '{kind}' (see include/txgemm.h)."
    return f


for _k in KINDS:
    globals()[f"tx_gemm_batched_{_k}"] = _named(_k, tx_gemm_batched)
    globals()[f"tx_gemm_batched_ptr_{_k}"] = _named(_k, tx_gemm_batched_ptr)
    globals()[f"tx_gemm_batched_hostio_{_k}"] = _named(_k, tx_gemm_batched_hostio)
    globals()[f"tx_gemm_batched_dev_{_k}"] = _named(_k, tx_gemm_batched_dev)
    globals()[f"tx_gemm_batched_ptr_dev_{_k}"] = _named(_k, tx_gemm_batched_ptr_dev)


# ------------------------------------------------------------ tensor API
def kind_of(dtype) -> str:
    import torch

    return {torch.float32: "s", torch.float64: "d", torch.complex64: "c",
            torch.complex128: "z"}[dtype]


def _ld(X, rows, cols):
    """(ld, ld2) of a (batch, rows, cols) column-major view."""
    if X.dim() != 3 or X.shape[1] != rows or X.shape[2] != cols:
        raise ValueError(f"expected shape (batch, {rows}, {cols}), got {tuple(X.shape)}")
    if rows > 1 and X.stride(1) != 1:
        raise ValueError("matrices must be column-major: stride(1) == 1")
    ld = X.stride(2) if cols > 1 else max(rows, 1)
    ld2 = X.stride(0) if X.shape[0] > 1 else ld * cols
    return ld, ld2


def gemm_batched(A, B, C, transa="N", transb="N", alpha=1.0, beta=0.0, stream=None):
    """C <- alpha*op(A) op(B) + beta*C on (batch, rows, cols) column-major views
    (PAPER.md:251-255).  A is (batch, m, k) for 'N' else (batch, k, m); B likewise."""
    import torch

    kind = kind_of(C.dtype)
    if A.dtype != C.dtype or B.dtype != C.dtype:
        raise ValueError("A, B and C must share a dtype")
    _same_device(A=A, B=B, C=C)
    batch, m, n = C.shape
    k = A.shape[2] if transa in "nN" else A.shape[1]
    ra, ca = (m, k) if transa in "nN" else (k, m)
    rb, cb = (k, n) if transb in "nN" else (n, k)
    if A.shape[0] != batch and A.shape[0] != 1 or B.shape[0] != batch and B.shape[0] != 1:
        raise ValueError("batch mismatch")
    lda, lda2 = _ld(A, ra, ca)
    ldb, ldb2 = _ld(B, rb, cb)
    ldc, ldc2 = _ld(C, m, n)
    if A.shape[0] == 1:
        lda2 = 0
    if B.shape[0] == 1:
        ldb2 = 0
    with torch.cuda.device(C.device):
        return _check(tx_gemm_batched(kind, transa, transb, m, n, k, alpha, A, lda, lda2, B, ldb,
                                      ldb2, beta, C, ldc, ldc2, batch, stream))


def _same_device(**tensors):
    """All tensors are CUDA tensors on one device (the library works on the current
    device; a tensor elsewhere would be a wild address there)."""
    dev = None
    for name, X in tensors.items():
        if not X.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
        if dev is None:
            dev = X.device
        elif X.device != dev:
            raise ValueError(f"{name} is on {X.device}, expected {dev}")
    return dev


def gemm_batched_ptr(Aarray, Barray, Carray, m, n, k, transa="N", transb="N", alpha=1.0,
                     beta=0.0, lda=None, ldb=None, ldc=None, dtype=None, stream=None):
    """Pointer-array batch (the paper's TGEMM_multi_nounif):
    C^p <- alpha*op(A^p) op(B^p) + beta*C^p with X^p at the device address Xarray[p].

    Xarray are int64 CUDA tensors of device addresses (e.g. from pointer_array()),
    all on one device; ``dtype`` is the matrices' torch dtype; ld* default to the
    stored rows (packed matrices).  The pointed-to matrices must live on that device
    and be aligned to the element size; C^p must not overlap each other or A, B
    (include/txgemm.h)."""
    import torch

    if dtype is None:
        raise ValueError("dtype of the matrices is required")
    kind = kind_of(dtype)
    dev = _same_device(Aarray=Aarray, Barray=Barray, Carray=Carray)
    for name, X in (("Aarray", Aarray), ("Barray", Barray), ("Carray", Carray)):
        if X.dtype != torch.int64 or X.dim() != 1:
            raise ValueError(f"{name} must be a 1-D int64 tensor of device addresses")
        if not X.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    batch = Carray.shape[0]
    if Aarray.shape[0] < batch or Barray.shape[0] < batch:
        raise ValueError("pointer arrays shorter than Carray")
    ra = m if transa in "nN" else k
    rb = k if transb in "nN" else n
    lda = max(1, ra) if lda is None else lda
    ldb = max(1, rb) if ldb is None else ldb
    ldc = max(1, m) if ldc is None else ldc
    with torch.cuda.device(dev):
        return _check(tx_gemm_batched_ptr(kind, transa, transb, m, n, k, alpha, Aarray, lda,
                                          Barray, ldb, beta, Carray, ldc, batch, stream))


def pointer_array(X, offsets=None):
    """Device int64 tensor of the addresses of matrices of a (batch, rows, cols) view."""
    import torch

    es = X.element_size()
    if offsets is None:
        offsets = torch.arange(X.shape[0], dtype=torch.int64) * X.stride(0)
    return (torch.as_tensor(offsets, dtype=torch.int64) * es + X.data_ptr()).to(X.device)
