"""paper_2510_23346_b200 -- B200-native BD-LoRA tensor-parallel multi-adapter LoRA layer.

Thin Python binding over libbdlora.so (include/bdlora.h): the functions below have the C-ABI's
names and only marshal arguments (torch tensors -> device pointers, the current CUDA stream).
Every step of the layer runs in the library's sm_100a kernels; PyTorch provides device memory,
streams and torch.distributed (for the NCCL unique-id bootstrap) only.  There is no CPU or eager
fallback: if libbdlora.so is missing, importing the library raises.

Paper: "Block-diagonal LoRA", arXiv 2510.23346 -- y = XW + s X A[a(t)] B[a(t)] per token, with
BD-LoRA sharding (B block-diagonal in column layers, A block-diagonal in row layers).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

from . import _lib
from ._lib import BdloraError, PoolDesc, call

COLUMN, ROW = 0, 1
SHARD_BD, SHARD_SLORA, SHARD_NFS = 0, 1, 2

__all__ = [
    "COLUMN", "ROW", "SHARD_BD", "SHARD_SLORA", "SHARD_NFS", "nfs_column_forward", "nfs_row_partial",
    "nfs_row_forward", "bdlora_column_forward_gather", "BdloraError", "Pool", "Comm",
    "bdlora_abi_version", "bdlora_device_check", "bdlora_kernel_launches", "bdlora_comm_unique_id", "bdlora_comm_init",
    "bdlora_comm_destroy", "bdlora_comm_stats", "bdlora_create_pool", "bdlora_destroy_pool",
    "bdlora_load_adapter", "bdlora_unload_adapter", "bdlora_pool_bytes", "bdlora_pool_geometry",
    "bdlora_workspace_bytes", "bdlora_build_segments", "bdlora_column_forward", "bdlora_row_partial",
    "bdlora_row_forward", "slora_column_forward", "slora_row_forward", "bdlora_lora_shrink",
    "bdlora_base_expand", "bdlora_v_elems", "make_workspace", "bdlora_workspace_init", "bdlora_last_launch_info",
    "Peer", "bdlora_peer_create", "bdlora_peer_create_local", "bdlora_peer_error", "bdlora_row_partial_push",
    "bdlora_peer_reduce", "bdlora_row_forward_fused", "bdlora_set_decode_lora", "bdlora_load_adapter_blocks",
]


def _torch():
    import torch

    return torch


def _stream(stream) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _need(t, name, dtype=None, device=None, shape=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} must live on {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


class Pool:
    """Owning handle of a bdlora_pool (one per device, projection and sharding mode)."""

    def __init__(self, handle: int, desc: PoolDesc, device: int):
        self.handle = handle
        self.desc = desc
        self.device = device
        k, m = ctypes.c_int32(), ctypes.c_int32()
        call("bdlora_pool_geometry", handle, ctypes.byref(k), ctypes.byref(m))
        self.k_loc, self.m_loc = k.value, m.value

    @property
    def tdevice(self):
        return _torch().device("cuda", self.device)

    def close(self):
        if self.handle:
            call("bdlora_destroy_pool", self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            if self.handle and _lib._lib is not None:
                _lib._lib.bdlora_destroy_pool(self.handle)
                self.handle = None
        except Exception:
            pass


class Comm:
    def __init__(self, handle: int, nranks: int, rank: int, device: int):
        self.handle, self.nranks, self.rank, self.device = handle, nranks, rank, device

    def close(self):
        if self.handle:
            call("bdlora_comm_destroy", self.handle)
            self.handle = None


class Peer:
    """Owning handle of a bdlora_peer (fused row all-reduce peer group, include/bdlora.h)."""

    def __init__(self, handle: int, rank: int, nranks: int, device: int):
        self.handle, self.rank, self.nranks, self.device = handle, rank, nranks, device

    def close(self):
        if self.handle:
            call("bdlora_peer_destroy", self.handle)
            self.handle = None


def _comm_ptr(comm: Optional[Comm]):
    return None if comm is None else comm.handle


# ------------------------------------------------------------------------------------------ library
def bdlora_abi_version() -> int:
    return _lib.load().bdlora_abi_version()


def bdlora_device_check(device: int = 0) -> None:
    call("bdlora_device_check", device)


def bdlora_kernel_launches() -> int:
    n = ctypes.c_int64()
    call("bdlora_kernel_launches", ctypes.byref(n))
    return n.value


# ------------------------------------------------------------------------------------------ comm
def bdlora_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    call("bdlora_comm_unique_id", buf)
    return bytes(buf)


def bdlora_comm_init(uid: bytes, nranks: int, rank: int, device: int) -> Comm:
    if len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    call("bdlora_comm_init", buf, nranks, rank, device, ctypes.byref(h))
    return Comm(h.value, nranks, rank, device)


def broadcast_unique_id(group=None, device=None) -> bytes:
    """Rank 0 of the process group draws an NCCL unique id (bdlora_comm_unique_id) and broadcasts
    the 128 bytes over torch.distributed (any backend: gloo on CPU, nccl on `device`)."""
    torch = _torch()
    import torch.distributed as dist

    rank = dist.get_rank(group)
    uid = bdlora_comm_unique_id() if rank == 0 else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
    if dist.get_backend(group) == "nccl":
        t = t.to(torch.device("cuda", device))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def comm_from_process_group(device: int, group=None) -> Optional[Comm]:
    """NCCL bootstrap over torch.distributed: rank 0 draws the unique id, broadcast, init."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return None
    uid = broadcast_unique_id(group, device)
    return bdlora_comm_init(uid, world, dist.get_rank(group), device)


def bdlora_comm_destroy(comm: Comm) -> None:
    comm.close()


def bdlora_comm_stats(comm: Comm) -> dict:
    arr = (ctypes.c_int64 * 6)()
    call("bdlora_comm_stats", comm.handle, arr)
    keys = ["base_allreduce_calls", "lora_allgather_calls", "lora_allreduce_calls",
            "base_allreduce_bytes", "lora_allgather_bytes", "lora_allreduce_bytes"]
    return dict(zip(keys, list(arr)))


# ------------------------------------------------------------------------------------------ pool
def bdlora_create_pool(parallel: int, sharding: int, tp_size: int, tp_rank: int, d_in: int,
                       d_out: Sequence[int], capacity: int, max_rank: int, arena_bytes: int = 0,
                       device: int = 0) -> Pool:
    d = PoolDesc()
    d.parallel, d.sharding, d.tp_size, d.tp_rank = parallel, sharding, tp_size, tp_rank
    d.d_in = d_in
    d.n_slices = len(d_out)
    for j in range(3):
        d.d_out[j] = int(d_out[j]) if j < len(d_out) else 0
    d.capacity, d.max_rank, d.arena_bytes = capacity, max_rank, arena_bytes
    h = ctypes.c_void_p()
    call("bdlora_create_pool", ctypes.byref(d), device, ctypes.byref(h))
    return Pool(h.value, d, device)


def bdlora_destroy_pool(pool: Pool) -> None:
    pool.close()


def _factor_ptrs(pool: Pool, A: Sequence, B: Sequence):
    torch = _torch()
    J = pool.desc.n_slices
    if len(A) != J or len(B) != J:
        raise ValueError(f"need {J} A and {J} B factors")
    on_dev = None
    for t in list(A) + list(B):
        _need(t, "factor", dtype=torch.bfloat16)
        if not t.is_contiguous():
            raise ValueError("factors must be contiguous (row-major)")
        if on_dev is None:
            on_dev = t.is_cuda
        elif on_dev != t.is_cuda:
            raise ValueError("factors must be all host or all device tensors")
    pa = (ctypes.c_void_p * J)(*[a.data_ptr() for a in A])
    pb = (ctypes.c_void_p * J)(*[b.data_ptr() for b in B])
    return pa, pb, 1 if on_dev else 0


def bdlora_load_adapter(pool: Pool, slot: int, rank: int, scale: float, A: Sequence, B: Sequence,
                        stream=None) -> None:
    """A, B: per-slice bf16 torch tensors in the load format of include/bdlora.h (all on the pool's
    device, or all on the CPU)."""
    pa, pb, on_dev = _factor_ptrs(pool, A, B)
    call("bdlora_load_adapter", pool.handle, slot, rank, ctypes.c_float(scale), pa, pb, on_dev, _stream(stream))


def bdlora_load_adapter_blocks(pool: Pool, slot: int, rank: int, scale: float, A: Sequence, B: Sequence,
                               n_blocks: int, stream=None) -> None:
    """Downward-compatible BD serving: factors trained with n_blocks = N_h diagonal blocks,
    served on this pool's tp_size = N_l devices (include/bdlora.h)."""
    pa, pb, on_dev = _factor_ptrs(pool, A, B)
    call("bdlora_load_adapter_blocks", pool.handle, slot, rank, ctypes.c_float(scale), pa, pb, int(n_blocks), on_dev,
         _stream(stream))


def bdlora_unload_adapter(pool: Pool, slot: int) -> None:
    call("bdlora_unload_adapter", pool.handle, slot)


def bdlora_pool_bytes(pool: Pool):
    r, a = ctypes.c_int64(), ctypes.c_int64()
    call("bdlora_pool_bytes", pool.handle, ctypes.byref(r), ctypes.byref(a))
    return r.value, a.value


def bdlora_pool_geometry(pool: Pool):
    return pool.k_loc, pool.m_loc


def bdlora_workspace_bytes(pool: Pool, T: int) -> int:
    n = ctypes.c_size_t()
    call("bdlora_workspace_bytes", pool.handle, T, ctypes.byref(n))
    return n.value


def bdlora_v_elems(pool: Pool, T: int) -> int:
    n = ctypes.c_int64()
    call("bdlora_v_elems", pool.handle, T, ctypes.byref(n))
    return n.value


def bdlora_workspace_init(pool: Pool, ws, stream=None) -> None:
    """Zero the workspace's counter region (required once before first use; include/bdlora.h)."""
    torch = _torch()
    _need(ws, "workspace", dtype=torch.uint8, device=pool.tdevice)
    call("bdlora_workspace_init", pool.handle, _ptr(ws), ws.numel(), _stream(stream))


def make_workspace(pool: Pool, T: int, stream=None):
    """Device workspace for T tokens, counter region initialised (bdlora_workspace_init); the library
    leaves the counters zero after every call."""
    torch = _torch()
    ws = torch.empty(bdlora_workspace_bytes(pool, T), dtype=torch.uint8, device=pool.tdevice)
    bdlora_workspace_init(pool, ws, stream)
    return ws


def bdlora_last_launch_info() -> dict:
    """The calling thread's last tensor-core kernel launch (include/bdlora.h): instantiation, BN, grid, ..."""
    arr = (ctypes.c_int32 * 8)()
    call("bdlora_last_launch_info", arr)
    keys = ["kind", "bn", "grid", "cluster", "stages", "m_tiles", "n_tiles", "k_blocks"]
    return dict(zip(keys, list(arr)))


# ------------------------------------------------------------------------------------------ routing
def bdlora_build_segments(ids, stream=None):
    """Returns (seg_start, seg_len, seg_id, n_seg) device int32 tensors (n_seg is a 1-element tensor)."""
    torch = _torch()
    _need(ids, "ids", dtype=torch.int32)
    T = ids.numel()
    dev = ids.device
    ss = torch.empty(max(T, 1), dtype=torch.int32, device=dev)
    sl = torch.empty_like(ss)
    si = torch.empty_like(ss)
    n = torch.empty(1, dtype=torch.int32, device=dev)
    call("bdlora_build_segments", _ptr(ids), T, _ptr(ss), _ptr(sl), _ptr(si), _ptr(n), _stream(stream))
    return ss, sl, si, n


# ------------------------------------------------------------------------------------------ forwards
def _check_fwd(pool: Pool, X, W, ids, Y, ws, x_cols: int, y_cols: int):
    torch = _torch()
    dev = pool.tdevice
    _need(X, "X", dtype=torch.bfloat16, device=dev)
    T = X.shape[0]
    _need(X, "X", shape=(T, x_cols))
    _need(W, "W", dtype=torch.bfloat16, device=dev, shape=(y_cols if pool.desc.parallel == COLUMN else pool.m_loc,
                                                           pool.k_loc))
    _need(ids, "ids", dtype=torch.int32, device=dev, shape=(T,))
    _need(Y, "Y", dtype=torch.bfloat16, device=dev, shape=(T, y_cols))
    _need(ws, "workspace", dtype=torch.uint8, device=dev)
    return T


def bdlora_column_forward(pool: Pool, X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("bdlora_column_forward", pool.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws), ws.numel(),
         _stream(stream))


def bdlora_row_partial(pool: Pool, X, W, ids, P, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, P, ws, pool.k_loc, pool.m_loc)
    call("bdlora_row_partial", pool.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(P), _ptr(ws), ws.numel(),
         _stream(stream))


def bdlora_row_forward(pool: Pool, comm: Optional[Comm], X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("bdlora_row_forward", pool.handle, _comm_ptr(comm), _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws),
         ws.numel(), _stream(stream))


def bdlora_column_forward_gather(pool: Pool, comm: Optional[Comm], X, W, ids, Y, ws, stream=None) -> None:
    """Alg. 2: column forward + all-gather; Y [T, N * M_loc] = device blocks in rank order."""
    torch = _torch()
    dev = pool.tdevice
    _need(X, "X", dtype=torch.bfloat16, device=dev)
    T = X.shape[0]
    _need(X, "X", shape=(T, pool.k_loc))
    _need(W, "W", dtype=torch.bfloat16, device=dev, shape=(pool.m_loc, pool.k_loc))
    _need(ids, "ids", dtype=torch.int32, device=dev, shape=(T,))
    _need(Y, "Y", dtype=torch.bfloat16, device=dev, shape=(T, pool.m_loc * pool.desc.tp_size))
    _need(ws, "workspace", dtype=torch.uint8, device=dev)
    call("bdlora_column_forward_gather", pool.handle, _comm_ptr(comm), _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y),
         _ptr(ws), ws.numel(), _stream(stream))


def slora_column_forward(pool: Pool, comm: Optional[Comm], X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("slora_column_forward", pool.handle, _comm_ptr(comm), _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws),
         ws.numel(), _stream(stream))


def slora_row_forward(pool: Pool, comm: Optional[Comm], X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("slora_row_forward", pool.handle, _comm_ptr(comm), _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws),
         ws.numel(), _stream(stream))


def nfs_column_forward(pool: Pool, X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("nfs_column_forward", pool.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws), ws.numel(),
         _stream(stream))


def nfs_row_partial(pool: Pool, X, W, ids, P, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, P, ws, pool.k_loc, pool.m_loc)
    call("nfs_row_partial", pool.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(P), _ptr(ws), ws.numel(),
         _stream(stream))


def nfs_row_forward(pool: Pool, comm: Optional[Comm], X, W, ids, Y, ws, stream=None) -> None:
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("nfs_row_forward", pool.handle, _comm_ptr(comm), _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws),
         ws.numel(), _stream(stream))


def bdlora_peer_create(comm: Comm, max_elems: int) -> Peer:
    """Collective: this rank's peer group of the fused row all-reduce (CUDA IPC handles exchanged via NCCL)."""
    h = ctypes.c_void_p()
    call("bdlora_peer_create", comm.handle, int(max_elems), ctypes.byref(h))
    return Peer(h.value, comm.rank, comm.nranks, comm.device)


def bdlora_peer_create_local(nranks: int, max_elems: int, device: int = 0) -> List[Peer]:
    """nranks emulated peer groups on one device (tests): element r is rank r's group."""
    arr = (ctypes.c_void_p * nranks)()
    call("bdlora_peer_create_local", int(nranks), int(device), int(max_elems), arr)
    return [Peer(arr[r], r, nranks, device) for r in range(nranks)]


def bdlora_peer_error(peer: Peer) -> int:
    e = ctypes.c_int32()
    call("bdlora_peer_error", peer.handle, ctypes.byref(e))
    return e.value


def bdlora_row_partial_push(pool: Pool, peer: Peer, X, W, ids, ws, stream=None) -> None:
    torch = _torch()
    dev = pool.tdevice
    _need(X, "X", dtype=torch.bfloat16, device=dev)
    T = X.shape[0]
    _need(X, "X", shape=(T, pool.k_loc))
    _need(W, "W", dtype=torch.bfloat16, device=dev, shape=(pool.m_loc, pool.k_loc))
    _need(ids, "ids", dtype=torch.int32, device=dev, shape=(T,))
    _need(ws, "workspace", dtype=torch.uint8, device=dev)
    call("bdlora_row_partial_push", pool.handle, peer.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(ws), ws.numel(),
         _stream(stream))


def bdlora_peer_reduce(peer: Peer, Y, stream=None) -> None:
    torch = _torch()
    _need(Y, "Y", dtype=torch.bfloat16)
    call("bdlora_peer_reduce", peer.handle, _ptr(Y), Y.shape[0], Y.shape[1], _stream(stream))


def bdlora_row_forward_fused(pool: Pool, peer: Peer, X, W, ids, Y, ws, stream=None) -> None:
    """Row layer with the base all-reduce fused into the GEMM over peer memory (include/bdlora.h)."""
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    call("bdlora_row_forward_fused", pool.handle, peer.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(Y), _ptr(ws),
         ws.numel(), _stream(stream))


def bdlora_lora_shrink(pool: Pool, X, ids, v, ws, stream=None) -> None:
    torch = _torch()
    dev = pool.tdevice
    _need(X, "X", dtype=torch.bfloat16, device=dev)
    T = X.shape[0]
    _need(ids, "ids", dtype=torch.int32, device=dev, shape=(T,))
    _need(v, "v", dtype=torch.float32, device=dev)
    if v.numel() < bdlora_v_elems(pool, T):
        raise ValueError("v too small")
    call("bdlora_lora_shrink", pool.handle, _ptr(X), T, _ptr(ids), _ptr(v), _ptr(ws), ws.numel(), _stream(stream))


def bdlora_base_expand(pool: Pool, X, W, ids, v, Y, ws, stream=None) -> None:
    torch = _torch()
    T = _check_fwd(pool, X, W, ids, Y, ws, pool.k_loc, pool.m_loc)
    _need(v, "v", dtype=torch.float32, device=pool.tdevice)
    call("bdlora_base_expand", pool.handle, _ptr(X), T, _ptr(W), _ptr(ids), _ptr(v), _ptr(Y), _ptr(ws), ws.numel(),
         _stream(stream))


def bdlora_debug_trace(buf) -> None:
    """Profiling hook: per-CTA timestamps of subsequent GEMM launches into `buf` (device int64), or None."""
    call("bdlora_debug_trace", None if buf is None else buf.data_ptr())


def bdlora_set_decode_lora(mode: int) -> None:
    """Decode LoRA schedule of the fused forward: 0 global shrink, 1 auto (default), 2 K-local (bdlora.h)."""
    call("bdlora_set_decode_lora", int(mode))


def bdlora_set_pdl(enable: bool) -> None:
    """Programmatic-dependent-launch chaining of the library's kernels (default on; see bdlora.h)."""
    call("bdlora_set_pdl", 1 if enable else 0)
