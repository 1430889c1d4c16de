"""ctypes loader for libbdlora.so (include/bdlora.h).  Argument marshalling only.

Fails loudly if the shared library is missing: there is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libbdlora.so")

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_vp = ctypes.c_void_p
c_size = ctypes.c_size_t
c_u8p = ctypes.POINTER(ctypes.c_uint8)


class PoolDesc(ctypes.Structure):
    _fields_ = [
        ("parallel", c_i32), ("sharding", c_i32), ("tp_size", c_i32), ("tp_rank", c_i32),
        ("d_in", c_i32), ("n_slices", c_i32), ("d_out", c_i32 * 3), ("capacity", c_i32),
        ("max_rank", c_i32), ("arena_bytes", c_i64),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "bdlora_abi_version": (c_int, []),
    "bdlora_last_error": (ctypes.c_char_p, []),
    "bdlora_device_check": (c_int, [c_int]),
    "bdlora_kernel_launches": (c_int, [ctypes.POINTER(c_i64)]),
    "bdlora_debug_trace": (c_int, [c_vp]),
    "bdlora_set_pdl": (c_int, [c_int]),
    "bdlora_set_decode_lora": (c_int, [c_int]),
    "bdlora_comm_unique_id": (c_int, [c_u8p]),
    "bdlora_comm_init": (c_int, [c_u8p, c_int, c_int, c_int, ctypes.POINTER(c_vp)]),
    "bdlora_comm_destroy": (c_int, [c_vp]),
    "bdlora_comm_stats": (c_int, [c_vp, ctypes.POINTER(c_i64)]),
    "bdlora_create_pool": (c_int, [ctypes.POINTER(PoolDesc), c_int, ctypes.POINTER(c_vp)]),
    "bdlora_destroy_pool": (c_int, [c_vp]),
    "bdlora_load_adapter": (c_int, [c_vp, c_i32, c_i32, c_f32, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i32, c_vp]),
    "bdlora_unload_adapter": (c_int, [c_vp, c_i32]),
    "bdlora_load_adapter_blocks": (c_int, [c_vp, c_i32, c_i32, c_f32, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i32,
                                           c_i32, c_vp]),
    "bdlora_pool_bytes": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "bdlora_pool_geometry": (c_int, [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "bdlora_workspace_bytes": (c_int, [c_vp, c_i64, ctypes.POINTER(c_size)]),
    "bdlora_workspace_init": (c_int, [c_vp, c_vp, c_size, c_vp]),
    "bdlora_peer_create": (c_int, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "bdlora_peer_create_local": (c_int, [c_int, c_int, c_i64, ctypes.POINTER(c_vp)]),
    "bdlora_peer_destroy": (c_int, [c_vp]),
    "bdlora_peer_error": (c_int, [c_vp, ctypes.POINTER(c_i32)]),
    "bdlora_row_partial_push": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_peer_reduce": (c_int, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "bdlora_row_forward_fused": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_last_launch_info": (c_int, [ctypes.POINTER(c_i32)]),
    "bdlora_build_segments": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bdlora_column_forward": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_row_partial": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_row_forward": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_column_forward_gather": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "slora_column_forward": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "slora_row_forward": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "nfs_column_forward": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "nfs_row_partial": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "nfs_row_forward": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_lora_shrink": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_base_expand": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "bdlora_v_elems": (c_int, [c_vp, c_i64, ctypes.POINTER(c_i64)]),
}


def header_symbols(path: str | None = None):
    """Function names declared in include/bdlora.h (used by the ABI export test)."""
    import re

    path = path or os.path.join(os.path.dirname(_PKG), "include", "bdlora.h")
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+((?:bdlora|slora|nfs)_\w+)\s*\(", src, flags=re.M)))


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libbdlora.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    # BDLORA_AB_OLD_LIB=1 (same-box A/B tooling only, scripts/ab_dec.sh): an older build may lack newer entry
    # points; they are then left unbound instead of failing the load
    tolerant = os.environ.get("BDLORA_AB_OLD_LIB") == "1"
    for name, (res, args) in SIGNATURES.items():
        if tolerant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class BdloraError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} failed with status {code} ({STATUS.get(code, '?')}): {msg}")
        self.code = code


STATUS = {0: "OK", 1: "E_ARG", 2: "E_DIVISIBILITY", 3: "E_CAPACITY", 4: "E_NOT_LOADED", 5: "E_MODE",
          6: "E_CUDA", 7: "E_NCCL", 8: "E_ARCH"}


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise BdloraError(rc, name, lib.bdlora_last_error().decode(errors="replace"))
    return rc
