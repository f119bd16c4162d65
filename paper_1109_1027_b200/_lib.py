"""ctypes declarations of the C-ABI in include/nlse2shoc.h (argument marshalling only).

Loading fails loudly if libnlse2shoc.so is missing: there is no CPU or Python fallback for
any step of the path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("NLSE_LIB") or os.path.join(_HERE, "libnlse2shoc.so")

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ENONFINITE, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
BC = {"dirichlet": 0, "lapzero": 1, "msd": 2}
DTYPE = {"c64": 0, "c128": 1}
VKIND = {"none": 0, "harmonic": 1, "array": 2}


class Potential(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("xmin", ctypes.c_double * 3),
        ("w", ctypes.c_double * 3),
        ("c", ctypes.c_double * 3),
        ("data", ctypes.c_void_p),
    ]


class NLSE2SHOCError(RuntimeError):
    def __init__(self, status, where, detail):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a).  There is no fallback implementation."
            )
        L = ctypes.CDLL(SO_PATH)
        H = ctypes.c_void_p
        i64p = ctypes.POINTER(ctypes.c_int64)
        dbl3 = ctypes.c_double * 3
        i643 = ctypes.c_int64 * 3
        sig = {
            "nlse2shoc_create": [ctypes.POINTER(H), ctypes.c_int, i643, dbl3, ctypes.c_double, ctypes.c_double,
                                 ctypes.POINTER(Potential), ctypes.c_int, ctypes.c_int],
            "nlse2shoc_get_unique_id": [ctypes.c_void_p],
            "nlse2shoc_create_sharded": [ctypes.POINTER(H), ctypes.c_int, i643, dbl3, ctypes.c_double, ctypes.c_double,
                                         ctypes.POINTER(Potential), ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int, ctypes.c_int],
            "nlse2shoc_create_loopback": [ctypes.POINTER(H), ctypes.c_int, i643, dbl3, ctypes.c_double,
                                          ctypes.c_double, ctypes.POINTER(Potential), ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int],
            "nlse2shoc_local_extent": [H, i64p, i64p],
            "nlse2shoc_split": [ctypes.c_int64, ctypes.c_int, ctypes.c_int, i64p, i64p],
            "nlse2shoc_set_variant": [H, ctypes.c_int],
            "nlse2shoc_set_scheme": [H, ctypes.c_int],
            "nlse2shoc_set_option": [H, ctypes.c_int, ctypes.c_int64],
            "nlse2shoc_ipc_handle": [H, ctypes.c_void_p],
            "nlse2shoc_connect_peers": [H, ctypes.c_void_p, ctypes.c_void_p],
            "nlse2shoc_laplacian": [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
            "nlse2shoc_rk4": [H, ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p],
            "nlse2shoc_stability_bound": [H, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p],
            "nlse2shoc_check_finite": [H, ctypes.c_void_p, ctypes.c_void_p],
            "nlse2shoc_set_workspace": [H, ctypes.c_void_p, ctypes.c_size_t],
            "nlse2shoc_padded_layout": [H, i643, i643],
            "nlse2shoc_rk4_padded": [H, ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p],
        }
        for name, args in sig.items():
            if os.environ.get("NLSE_LIB") and not hasattr(L, name):
                continue  # an older library under test (A/B timing): its missing calls stay unbound
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.nlse2shoc_workspace_bytes.argtypes = [H]
        L.nlse2shoc_workspace_bytes.restype = ctypes.c_size_t
        if hasattr(L, "nlse2shoc_stage_workspace_bytes"):
            L.nlse2shoc_stage_workspace_bytes.argtypes = [H]
            L.nlse2shoc_stage_workspace_bytes.restype = ctypes.c_size_t
        if hasattr(L, "nlse2shoc_exchange_timeouts"):
            L.nlse2shoc_exchange_timeouts.argtypes = [H]
            L.nlse2shoc_exchange_timeouts.restype = ctypes.c_int64
        L.nlse2shoc_last_launch_count.argtypes = [H]
        L.nlse2shoc_last_launch_count.restype = ctypes.c_int64
        L.nlse2shoc_strerror.argtypes = [ctypes.c_int]
        L.nlse2shoc_strerror.restype = ctypes.c_char_p
        L.nlse2shoc_last_error.argtypes = []
        L.nlse2shoc_last_error.restype = ctypes.c_char_p
        L.nlse2shoc_version.argtypes = []
        L.nlse2shoc_version.restype = ctypes.c_char_p
        if hasattr(L, "nlse2shoc_checked_violations"):
            L.nlse2shoc_checked_violations.argtypes = []
            L.nlse2shoc_checked_violations.restype = ctypes.c_int64
        L.nlse2shoc_destroy.argtypes = [H]
        L.nlse2shoc_destroy.restype = None
        has_alloc = hasattr(L, "nlse2shoc_set_allocator")
        if has_alloc:
            L.nlse2shoc_set_allocator.argtypes = [ALLOC_FN, FREE_FN, ctypes.c_void_p]
            L.nlse2shoc_set_allocator.restype = ctypes.c_int
        _lib = L
        if has_alloc and os.environ.get("NLSE_CUDA_MALLOC") != "1":
            use_torch_allocator()
    return _lib


# All device memory the library owns comes from torch's caching allocator (north star:
# PyTorch for device memory).  NLSE_CUDA_MALLOC=1 keeps the library's own cudaMalloc.
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


def _torch_alloc(nbytes, device, ctx):
    try:
        import torch

        return int(torch.cuda.caching_allocator_alloc(int(nbytes), device=int(device)))
    except Exception:  # out of memory (or torch unusable): the library reports ENOMEM
        return None


def _torch_free(ptr, device, ctx):
    try:
        import torch

        torch.cuda.caching_allocator_delete(int(ptr))
    except Exception:  # interpreter shutdown
        pass


_ALLOC_CB = ALLOC_FN(_torch_alloc)
_FREE_CB = FREE_FN(_torch_free)


def use_torch_allocator(enable: bool = True):
    """Route the library's device allocations through torch (process-wide, for handles
    created afterwards); enable=False restores cudaMalloc."""
    L = lib()
    if enable:
        check(L.nlse2shoc_set_allocator(_ALLOC_CB, _FREE_CB, None), "set_allocator")
    else:
        check(L.nlse2shoc_set_allocator(ALLOC_FN(), FREE_FN(), None), "set_allocator")


def check(status, where):
    if status != OK:
        L = lib()
        raise NLSE2SHOCError(status, where, (L.nlse2shoc_strerror(status).decode() + ": "
                                             + L.nlse2shoc_last_error().decode()))
    return status


# Header symbols, for the "library exports everything include/*.h declares" test.
EXPORTS = [
    "nlse2shoc_create", "nlse2shoc_get_unique_id", "nlse2shoc_create_sharded", "nlse2shoc_create_loopback",
    "nlse2shoc_local_extent",
    "nlse2shoc_split", "nlse2shoc_workspace_bytes", "nlse2shoc_set_variant", "nlse2shoc_set_scheme", "nlse2shoc_set_option",
    "nlse2shoc_ipc_handle", "nlse2shoc_connect_peers",
    "nlse2shoc_exchange_timeouts", "nlse2shoc_laplacian",
    "nlse2shoc_rk4", "nlse2shoc_stability_bound", "nlse2shoc_check_finite", "nlse2shoc_last_launch_count",
    "nlse2shoc_strerror", "nlse2shoc_last_error", "nlse2shoc_version", "nlse2shoc_destroy",
    "nlse2shoc_set_allocator", "nlse2shoc_checked_violations",
    "nlse2shoc_stage_workspace_bytes", "nlse2shoc_set_workspace", "nlse2shoc_padded_layout", "nlse2shoc_rk4_padded",
]
