"""Thin ctypes binding of the C ABI in include/tn.h (argument marshalling only).

Every step of a contraction runs in ``libtn.so``'s CUDA kernels; this module
converts numpy / torch arguments into pointers and status codes into
exceptions.  There is no fallback: if the library is missing, importing a
function that needs it raises ``TNLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtn.so")

EXTENDED, MIXED = 0, 1
_STATUS = {0: "TN_OK", 1: "TN_ERR_USAGE", 2: "TN_ERR_DATA", 3: "TN_ERR_RESOURCE",
           4: "TN_ERR_CUDA", 5: "TN_ERR_INTERNAL"}

# every symbol include/tn.h declares (checked by tests/test_abi.py)
SYMBOLS = ["tn_create", "tn_load_network", "tn_upload_tensors", "tn_set_path", "tn_set_slices",
           "tn_contract", "tn_reset_accumulator", "tn_sum_slices", "tn_sum_slices_host",
           "tn_get_info", "tn_plan_json", "tn_set_profiling", "tn_get_kernel_stats",
           "tn_reset_kernel_stats", "tn_get_step_stats", "tn_cgemm", "tn_last_error", "tn_version",
           "tn_last_overflow", "tn_destroy"]


class TNLibraryError(RuntimeError):
    pass


class TNError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Info(C.Structure):
    _fields_ = [("n_slices", C.c_int64), ("n_out", C.c_int64), ("n_steps", C.c_int32),
                ("n_tc_steps", C.c_int32), ("flops_per_slice", C.c_double),
                ("tc_flops_per_slice", C.c_double), ("bytes_per_slice", C.c_double),
                ("peak_elements", C.c_double), ("device_bytes", C.c_int64),
                ("arena_bytes", C.c_int64), ("scratch_bytes", C.c_int64),
                ("graph_replays", C.c_int64)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    """tn_allocator (include/tn.h)."""
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


def _torch_alloc(nbytes, device, stream, user):
    """tn_allocator.alloc -> torch's CUDA caching allocator on the context stream."""
    try:
        import torch
        return torch.cuda.caching_allocator_alloc(int(nbytes), device=int(device), stream=int(stream or 0))
    except Exception:  # noqa: BLE001  (out of memory -> NULL -> TN_ERR_RESOURCE)
        return None


def _torch_free(ptr, nbytes, device, stream, user):
    try:
        import torch
        torch.cuda.caching_allocator_delete(int(ptr))
    except Exception:  # noqa: BLE001  (interpreter shutdown)
        pass


# one process-wide pair of callbacks (ctypes keeps them alive while referenced here)
_TORCH_ALLOCATOR = Allocator(ALLOC_FN(_torch_alloc), FREE_FN(_torch_free), None)


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


_lib = None


def lib():
    """Load libtn.so, (re)building it first when it is missing or older than its
    sources and nvcc exists; a present library is used as is when nvcc is absent."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build
    alt = os.environ.get("TN_LIB_PATH")      # tooling only: A/B of two builds (tools/gpu_ab.sh)
    if alt:
        _lib = _bind(C.CDLL(alt))
        return _lib
    if _build.needs_build():
        have_nvcc = os.path.exists(_build.NVCC)
        if have_nvcc:
            try:
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise TNLibraryError(f"libtn.so could not be built: {e}") from e
        elif not os.path.exists(LIB_PATH):
            raise TNLibraryError(f"libtn.so missing and nvcc not found at {_build.NVCC}")
    _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def _bind(L):
    """Declare the C-ABI signatures (include/tn.h) on a loaded libtn."""
    P, I32, I64, D, VP = C.POINTER, C.c_int32, C.c_int64, C.c_double, C.c_void_p
    sig = {
        "tn_create": [P(VP), C.c_int, P(Allocator), VP],
        "tn_load_network": [VP, I32, VP, VP, VP, VP, I32, VP, I64, VP],
        "tn_upload_tensors": [VP, VP],
        "tn_set_path": [VP, I32, VP],
        "tn_set_slices": [VP, I32, VP, P(I64)],
        "tn_contract": [VP, I64, I64, C.c_int, I32],
        "tn_reset_accumulator": [VP],
        "tn_sum_slices": [VP, VP, I64],
        "tn_sum_slices_host": [VP, VP, I64],
        "tn_get_info": [VP, P(Info)],
        "tn_plan_json": [VP, C.c_char_p, C.c_size_t, P(C.c_size_t)],
        "tn_set_profiling": [VP, C.c_int],
        "tn_get_kernel_stats": [VP, C.c_int, P(KernelStats)],
        "tn_reset_kernel_stats": [VP],
        "tn_get_step_stats": [VP, C.c_int, I64, VP],
        "tn_cgemm": [VP, VP, VP, VP, I64, I64, I64, I64, I64, I64, VP, VP, C.c_int, C.c_int, C.c_int],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.tn_last_overflow.argtypes = [VP]
    L.tn_last_overflow.restype = C.c_int
    L.tn_last_error.restype = C.c_char_p
    L.tn_version.restype = C.c_char_p
    L.tn_destroy.argtypes = [VP]
    L.tn_destroy.restype = None
    return L


def _check(st):
    if st != 0:
        raise TNError(st, lib().tn_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _tptr(t):
    """Device pointer of a torch tensor (or an int / None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return C.c_void_p(t)
    return C.c_void_p(t.data_ptr())


class Contraction:
    """One context = one device + stream (``tn_create``)."""

    def __init__(self, device: int = 0, stream=None, allocator: str = "torch"):
        """device = -1 builds a host-only planner (bookkeeping, no execution).
        ``stream``: a torch.cuda.Stream (kept as ``self.stream``; every call of this
        context is enqueued on it), a raw cudaStream_t int, or None (legacy stream).
        ``allocator``: "torch" = every device allocation of the context comes from
        torch's caching allocator (tn_allocator callbacks); "cuda" = cudaMalloc."""
        L = lib()
        h = C.c_void_p()
        s = None
        if stream is not None:
            s = C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
        if allocator not in ("torch", "cuda"):
            raise ValueError("allocator must be 'torch' or 'cuda'")
        a = C.byref(_TORCH_ALLOCATOR) if allocator == "torch" and device >= 0 else None
        _check(L.tn_create(C.byref(h), int(device), a, s))
        self.allocator = allocator
        self._h = h
        self.device = device
        self.stream = stream if stream is not None and not isinstance(stream, int) else None
        self.n_slices = None
        self.n_out = None

    @property
    def torch_device(self):
        import torch
        return torch.device("cuda", self.device) if self.device >= 0 else torch.device("cpu")

    def close(self):
        if getattr(self, "_h", None):
            lib().tn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # --------------------------------------------------------------- setup
    def load_network(self, ranks, labels, dims, data, open_labels, samples=None):
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        data = np.ascontiguousarray(np.asarray(data, dtype=np.complex128)).view(np.float64)
        opens = np.ascontiguousarray(open_labels, dtype=np.int64)
        if samples is None:
            sp, ns = None, 0
        else:
            samples = np.ascontiguousarray(samples, dtype=np.uint8)
            sp, ns = _ptr(samples), samples.shape[0]
        _check(lib().tn_load_network(self._h, len(ranks), _ptr(ranks), _ptr(labels), _ptr(dims),
                                     _ptr(data), len(opens), _ptr(opens), ns, sp))
        self._keep = (ranks, labels, dims, data, opens, samples)

    def upload_tensors(self, data):
        data = np.ascontiguousarray(np.asarray(data, dtype=np.complex128)).view(np.float64)
        _check(lib().tn_upload_tensors(self._h, _ptr(data)))

    def set_path(self, pairs):
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        _check(lib().tn_set_path(self._h, p.shape[0], _ptr(p)))

    def set_slices(self, sliced_labels=()):
        s = np.ascontiguousarray(np.asarray(list(sliced_labels), dtype=np.int64))
        n = C.c_int64()
        _check(lib().tn_set_slices(self._h, len(s), _ptr(s) if len(s) else None, C.byref(n)))
        self.n_slices = n.value
        self.n_out = self.info()["n_out"]
        return n.value

    # --------------------------------------------------------------- execution
    def contract(self, begin=0, end=None, precision="extended", mixed_topk=10):
        end = self.n_slices if end is None else end
        prec = MIXED if precision == "mixed" else EXTENDED
        _check(lib().tn_contract(self._h, int(begin), int(end), prec, int(mixed_topk)))

    def reset_accumulator(self):
        _check(lib().tn_reset_accumulator(self._h))

    def sum_slices(self, out):
        """Write amplitudes into a complex128 CUDA torch tensor of length n_out."""
        _check(lib().tn_sum_slices(self._h, _tptr(out), int(self.n_out)))

    def overflow(self) -> bool:
        """tn_last_overflow: a fused epilogue saturated an fp16 plane (synchronises)."""
        v = lib().tn_last_overflow(self._h)
        if v < 0:
            raise TNError(1, "tn_last_overflow: bad or host-only context")
        return bool(v)

    def sum_slices_host(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.zeros(self.n_out, dtype=np.complex128)
        _check(lib().tn_sum_slices_host(self._h, _ptr(out.view(np.float64)), int(self.n_out)))
        return out

    # --------------------------------------------------------------- reports
    def info(self) -> dict:
        i = Info()
        _check(lib().tn_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in Info._fields_}

    def plan_json(self) -> dict:
        n = C.c_size_t()
        _check(lib().tn_plan_json(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().tn_plan_json(self._h, buf, n.value + 1, C.byref(n)))
        return json.loads(buf.value.decode())

    def set_profiling(self, on: bool = True):
        _check(lib().tn_set_profiling(self._h, int(bool(on))))

    def kernel_stats(self) -> dict:
        names = ["gemm_tcgen05", "prep", "einsum_simt", "slice_select"]
        out = {}
        for f, nm in enumerate(names):
            k = KernelStats()
            _check(lib().tn_get_kernel_stats(self._h, f, C.byref(k)))
            out[nm] = {"launches": k.launches, "ms": k.ms, "flops": k.flops, "bytes": k.bytes}
        return out

    def step_stats(self, family: int = -1) -> np.ndarray:
        """Device ms per path step accumulated while profiling (tn_get_step_stats);
        family 0 GEMM, 1 prep, 2 SIMT, -1 all."""
        n = self.info()["n_steps"]
        ms = np.zeros(n, np.float64)
        _check(lib().tn_get_step_stats(self._h, family, n, _ptr(ms)))
        return ms

    def reset_kernel_stats(self):
        _check(lib().tn_reset_kernel_stats(self._h))

    # --------------------------------------------------------------- convenience
    def setup(self, net, samples, path, sliced):
        """Load a ``tnworkloads`` network (``.flat()``), path and slices."""
        ranks, labels, dims, data, opens = net.flat()
        self.load_network(ranks, labels, dims, data, opens, samples)
        self.set_path(path)
        return self.set_slices(sliced)

    FORMATS = {"fp16": 0, "bf16": 1, "tf32": 2}

    def cgemm(self, A, B, Cout, J, m, n, k, ga=1, gb=1, ia=None, ib=None, passes=3,
              force_simt=False, fmt="fp16"):
        """Stand-alone complex GEMM on torch complex64 CUDA tensors (unit tests, the
        precision study); fmt = operand format of the tensor-core path (tn_cgemm)."""
        _check(lib().tn_cgemm(self._h, _tptr(A), _tptr(B), _tptr(Cout), int(J), int(m), int(n),
                              int(k), int(ga), int(gb), _tptr(ia), _tptr(ib), int(passes),
                              int(bool(force_simt)), self.FORMATS[fmt]))
