"""paper_1109_1027_b200 — B200-native RK4 + 2SHOC NLSE step (arxiv 1109.1027).

Thin Python binding over the C-ABI of ``libnlse2shoc.so`` (include/nlse2shoc.h).  The
functions below carry the C names and only marshal arguments (torch tensors -> device
pointers, the current CUDA stream -> cudaStream_t); every step of the path runs in the
library's sm_100a kernels.  PyTorch provides device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes

from ._lib import BC, DTYPE, VKIND, NLSE2SHOCError, Potential, check, lib

__all__ = [
    "Solver", "NLSE2SHOCError", "nlse2shoc_create", "nlse2shoc_create_sharded", "nlse2shoc_get_unique_id",
    "nlse2shoc_laplacian", "nlse2shoc_rk4", "nlse2shoc_stability_bound", "nlse2shoc_check_finite",
    "nlse2shoc_split", "nlse2shoc_version", "solver_from_work", "nlse2shoc_create_loopback", "nlse2shoc_set_option",
    "nlse2shoc_ipc_handle", "nlse2shoc_connect_peers", "peer_handles", "gather_peer_handles",
]


def _stream(stream):
    import torch

    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _potential(V, dims):
    p = Potential()
    keep = None
    if V is None or V.get("kind", "none") == "none":
        p.kind = VKIND["none"]
        return p, keep
    p.kind = VKIND[V["kind"]]
    for d in range(3):
        p.xmin[d] = float(V.get("xmin", [0.0] * 3)[d]) if d < len(V.get("xmin", [])) else 0.0
        p.w[d] = float(V.get("w", [0.0] * 3)[d]) if d < len(V.get("w", [])) else 0.0
        p.c[d] = float(V.get("c", [0.0] * 3)[d]) if d < len(V.get("c", [])) else 0.0
    if V["kind"] == "array":
        keep = V["data"]  # torch tensor on the device; kept alive by the Solver
        p.data = keep.data_ptr()
    return p, keep


def nlse2shoc_version() -> str:
    return lib().nlse2shoc_version().decode()


def nlse2shoc_split(n_slow: int, nranks: int, rank: int):
    z0, nz = ctypes.c_int64(), ctypes.c_int64()
    check(lib().nlse2shoc_split(int(n_slow), int(nranks), int(rank), ctypes.byref(z0), ctypes.byref(nz)), "split")
    return z0.value, nz.value


def nlse2shoc_get_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    check(lib().nlse2shoc_get_unique_id(buf), "get_unique_id")
    return bytes(buf)


def _args(dims, N, h):
    n = [int(v) for v in list(N)[:dims]] + [1] * (3 - dims)
    hh = [float(v) for v in list(h)[:dims]] + [1.0] * (3 - dims)
    return (ctypes.c_int64 * 3)(*n), (ctypes.c_double * 3)(*hh)


def nlse2shoc_create(dims, N, h, a, s, V=None, bc="dirichlet", dtype="c64"):
    H = ctypes.c_void_p()
    n, hh = _args(dims, N, h)
    pv, keep = _potential(V, dims)
    check(lib().nlse2shoc_create(ctypes.byref(H), int(dims), n, hh, float(a), float(s), ctypes.byref(pv), BC[bc],
                                 DTYPE[dtype]), "create")
    return H, keep


def nlse2shoc_create_sharded(dims, N, h, a, s, V, bc, dtype, uid: bytes, rank: int, nranks: int):
    H = ctypes.c_void_p()
    n, hh = _args(dims, N, h)
    pv, keep = _potential(V, dims)
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    check(lib().nlse2shoc_create_sharded(ctypes.byref(H), int(dims), n, hh, float(a), float(s), ctypes.byref(pv),
                                         BC[bc], DTYPE[dtype], buf, int(rank), int(nranks)), "create_sharded")
    return H, keep


def nlse2shoc_create_loopback(dims, N, h, a, s, V, bc, dtype, nslabs: int):
    H = ctypes.c_void_p()
    n, hh = _args(dims, N, h)
    pv, keep = _potential(V, dims)
    check(lib().nlse2shoc_create_loopback(ctypes.byref(H), int(dims), n, hh, float(a), float(s), ctypes.byref(pv),
                                          BC[bc], DTYPE[dtype], int(nslabs)), "create_loopback")
    return H, keep


def nlse2shoc_laplacian(H, psi, L, stream=None):
    check(lib().nlse2shoc_laplacian(H, _ptr(psi), _ptr(L), _stream(stream)), "laplacian")
    return L


def nlse2shoc_rk4(H, psi, dt, nsteps, stream=None):
    check(lib().nlse2shoc_rk4(H, _ptr(psi), float(dt), int(nsteps), _stream(stream)), "rk4")
    return psi


def nlse2shoc_stability_bound(H, psi, stream=None) -> float:
    k = ctypes.c_double()
    check(lib().nlse2shoc_stability_bound(H, _ptr(psi), ctypes.byref(k), _stream(stream)), "stability_bound")
    return k.value


def nlse2shoc_check_finite(H, psi, stream=None):
    check(lib().nlse2shoc_check_finite(H, _ptr(psi), _stream(stream)), "check_finite")


OPTIONS = {"cuda_graph": 0, "overlap": 1, "resident_1d": 2, "reverse_order": 3, "lean_steps": 4, "zchunks": 5,
           "tile_schedule": 6, "fused_exchange": 7, "tail_chunks": 8, "check_every": 9}


def nlse2shoc_set_option(H, option, value: int):
    check(lib().nlse2shoc_set_option(H, OPTIONS.get(option, option), int(value)), "set_option")


def nlse2shoc_ipc_handle(H) -> bytes:
    buf = (ctypes.c_ubyte * 64)()
    check(lib().nlse2shoc_ipc_handle(H, buf), "ipc_handle")
    return bytes(buf)


def nlse2shoc_connect_peers(H, lower: bytes | None, upper: bytes | None):
    lo = (ctypes.c_ubyte * 64).from_buffer_copy(lower) if lower is not None else None
    hi = (ctypes.c_ubyte * 64).from_buffer_copy(upper) if upper is not None else None
    check(lib().nlse2shoc_connect_peers(H, lo, hi), "connect_peers")


def peer_handles(handles, rank: int, nranks: int):
    """The (lower, upper) neighbours' entries of an all-gathered list (None at the ends)."""
    if len(handles) != nranks:
        raise ValueError(f"expected {nranks} handles, got {len(handles)}")
    return (handles[rank - 1] if rank > 0 else None), (handles[rank + 1] if rank < nranks - 1 else None)


def gather_peer_handles(mine: bytes, group=None):
    """All-gather every rank's 64-byte IPC handle over torch.distributed (any backend) and
    return this rank's (lower, upper) neighbours' handles."""
    import torch.distributed as dist

    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    out = [None] * ws
    dist.all_gather_object(out, mine, group=group)
    return peer_handles(out, rank, ws)


def _check_V_array(V, dims, N, dtype, shard):
    """V kind 'array' reaches the library as a raw pointer that the kernels read as R (float32
    for c64, float64 for c128) over the whole grid (single-GPU / loopback handles) or the
    local z-slab (NCCL shards): check what the pointer cannot carry."""
    import torch

    t = V.get("data") if V else None
    if t is None or not isinstance(t, torch.Tensor):
        raise ValueError("V['data'] must be a torch tensor for V kind 'array'")
    want = torch.float32 if dtype == "c64" else torch.float64
    if not t.is_cuda or t.device.index != torch.cuda.current_device():
        raise ValueError(f"V['data'] must be a CUDA tensor on device {torch.cuda.current_device()}")
    if t.dtype != want:
        raise ValueError(f"V['data'] has dtype {t.dtype}, the handle computes in {want}")
    if not t.is_contiguous():
        raise ValueError("V['data'] must be contiguous ([z][y][x], x fastest)")
    n = [int(v) for v in list(N)[:dims]]
    total = 1
    for v in n:
        total *= v
    if shard is not None and "loopback" not in shard:
        _, nz = nlse2shoc_split(n[-1], shard["nranks"], shard["rank"])
        total = total // n[-1] * nz
    if t.numel() != total:
        raise ValueError(f"V['data'] has {t.numel()} values, expected {total}")


class Solver:
    """Owns one nlse2shoc handle.  Psi tensors are contiguous torch complex64/complex128
    CUDA tensors of shape (Nz, Ny, Nx) / (Ny, Nx) / (Nx,) (sharded: the local slab)."""

    def __init__(self, dims, N, h, a, s, V=None, bc="dirichlet", dtype="c64", shard=None):
        self.dims, self.dtype, self.bc = int(dims), dtype, bc
        self.N = [int(v) for v in list(N)[:dims]]
        if V is not None and V.get("kind") == "array":
            _check_V_array(V, self.dims, N, dtype, shard)
        if shard is None:
            self._h, self._keep = nlse2shoc_create(dims, N, h, a, s, V, bc, dtype)
        elif "loopback" in shard:
            self._h, self._keep = nlse2shoc_create_loopback(dims, N, h, a, s, V, bc, dtype, shard["loopback"])
        else:
            self._h, self._keep = nlse2shoc_create_sharded(dims, N, h, a, s, V, bc, dtype, shard["uid"],
                                                           shard["rank"], shard["nranks"])
        z0, nz = ctypes.c_int64(), ctypes.c_int64()
        check(lib().nlse2shoc_local_extent(self._h, ctypes.byref(z0), ctypes.byref(nz)), "local_extent")
        self.z0, self.nz = z0.value, nz.value

    @property
    def local_shape(self):
        if self.dims == 1:
            return (self.N[0],)
        if self.dims == 2:
            return (self.nz, self.N[0])
        return (self.nz, self.N[1], self.N[0])

    def set_variant(self, variant: int):
        check(lib().nlse2shoc_set_variant(self._h, int(variant)), "set_variant")

    def set_option(self, option, value: int):
        """Execution-path option (include/nlse2shoc.h nlse2shoc_option): 'cuda_graph',
        'overlap', 'resident_1d', 'reverse_order', 'lean_steps', 'zchunks', 'tile_schedule',
        'fused_exchange', 'tail_chunks', 'check_every'."""
        nlse2shoc_set_option(self._h, option, value)

    def connect_peers(self, group=None):
        """Sharded (NCCL) handles: exchange halo-arena IPC handles with the neighbour ranks
        (torch.distributed all-gather) and switch rk4 to the fused exchange.  Collective."""
        lo, hi = gather_peer_handles(nlse2shoc_ipc_handle(self._h), group)
        nlse2shoc_connect_peers(self._h, lo, hi)

    def set_scheme(self, scheme):
        """0/"2shoc" (default) or 1/"cd" (the paper's RK4+CD comparison scheme)."""
        code = {"2shoc": 0, "cd": 1}.get(scheme, scheme)
        check(lib().nlse2shoc_set_scheme(self._h, int(code)), "set_scheme")

    def _check(self, t, name="psi"):
        """The C ABI takes raw pointers: check what it cannot (device, dtype, layout, shape)."""
        import torch

        want = torch.complex64 if self.dtype == "c64" else torch.complex128
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype != want:
            raise ValueError(f"{name} has dtype {t.dtype}, the handle computes in {want}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous ([z][y][x], x fastest)")
        if tuple(t.shape) != tuple(self.local_shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(self.local_shape)}")
        return t

    def laplacian(self, psi, out=None, stream=None):
        import torch

        self._check(psi)
        if out is None:
            out = torch.empty_like(psi)
        return nlse2shoc_laplacian(self._h, psi, self._check(out, "out"), stream)

    def rk4(self, psi, dt, nsteps, stream=None):
        return nlse2shoc_rk4(self._h, self._check(psi), dt, nsteps, stream)

    @property
    def padded_layout(self):
        """(pitch, offset): elements per x-row / per plane / per local field the kernels use in
        place, and the (zero) ghost offsets (nlse2shoc_padded_layout)."""
        pitch, off = (ctypes.c_int64 * 3)(), (ctypes.c_int64 * 3)()
        check(lib().nlse2shoc_padded_layout(self._h, pitch, off), "padded_layout")
        return list(pitch), list(off)

    def rk4_padded(self, psi, dt, nsteps, stream=None):
        """rk4 on a Psi already in padded_layout (rows of pitch[0] elements): a CUDA tensor
        whose last dimension is pitch[0] (the pad column is ignored and left untouched)."""
        import torch

        pitch, _ = self.padded_layout
        want = torch.complex64 if self.dtype == "c64" else torch.complex128
        shape = tuple(self.local_shape[:-1]) + (pitch[0],)
        if (not isinstance(psi, torch.Tensor) or not psi.is_cuda or psi.dtype != want or not psi.is_contiguous()
                or tuple(psi.shape) != shape):
            raise ValueError(f"psi must be a contiguous CUDA {want} tensor of shape {shape}")
        st = _stream(stream)
        check(lib().nlse2shoc_rk4_padded(self._h, psi.data_ptr(), float(dt), int(nsteps), st), "rk4_padded")
        return psi

    @property
    def stage_workspace_bytes(self) -> int:
        return int(lib().nlse2shoc_stage_workspace_bytes(self._h))

    def set_workspace(self, buf):
        """Place the three stage fields in the caller's CUDA tensor (any dtype, at least
        stage_workspace_bytes, 256-byte aligned); the Solver keeps a reference to it."""
        import torch

        if not isinstance(buf, torch.Tensor) or not buf.is_cuda or not buf.is_contiguous():
            raise ValueError("workspace must be a contiguous CUDA tensor")
        check(lib().nlse2shoc_set_workspace(self._h, buf.data_ptr(), buf.numel() * buf.element_size()), "set_workspace")
        self._workspace = buf

    def stability_bound(self, psi, stream=None) -> float:
        return nlse2shoc_stability_bound(self._h, self._check(psi), stream)

    def check_finite(self, psi, stream=None):
        nlse2shoc_check_finite(self._h, self._check(psi), stream)

    @property
    def exchange_timeouts(self) -> int:
        """Fused-exchange waits that gave up (0 in a correct run); syncs the device."""
        return int(lib().nlse2shoc_exchange_timeouts(self._h))

    @property
    def workspace_bytes(self) -> int:
        return int(lib().nlse2shoc_workspace_bytes(self._h))

    @property
    def last_launch_count(self) -> int:
        return int(lib().nlse2shoc_last_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib().nlse2shoc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solver_from_work(work: dict, dtype: str, V_array=None, shard=None) -> Solver:
    """Solver for a workload dict (icgen.configs layout: grid, a, s, V, bc).  ``V_array`` is
    the device tensor for V kind 'array'."""
    g = work["grid"]
    dims = g["dims"]
    V = dict(work["V"])
    if V["kind"] in ("harmonic", "array"):
        V["xmin"] = list(g["xmin"])
    if V["kind"] == "array":
        V["data"] = V_array
    return Solver(dims, g["n"][:dims], g["h"][:dims], work["a"], work["s"], V, work["bc"], dtype, shard=shard)
