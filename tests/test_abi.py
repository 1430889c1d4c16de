"""C-ABI library checks that need no GPU: libbdlora.so loads, exports every symbol include/bdlora.h
declares, and host-side validation returns the documented status codes before touching a device."""
import ctypes
import os
import subprocess

import pytest

from paper_2510_23346_b200 import _lib
import paper_2510_23346_b200 as bd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    names = _lib.header_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/bdlora.h but not exported"
    # and the binding declares a signature for each
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_nm_dynamic_exports(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in _lib.header_symbols():
        assert f" T {n}" in out


def test_sass_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_last_error(lib):
    assert bd.bdlora_abi_version() == 1
    assert isinstance(lib.bdlora_last_error(), bytes)


def _desc(**kw):
    d = _lib.PoolDesc()
    base = dict(parallel=0, sharding=0, tp_size=2, tp_rank=0, d_in=256, n_slices=1, capacity=4, max_rank=8,
                arena_bytes=0)
    base.update(kw)
    for k, v in base.items():
        if k != "d_out":
            setattr(d, k, v)
    dout = kw.get("d_out", [512, 0, 0])
    for j in range(3):
        d.d_out[j] = dout[j]
    return d


@pytest.mark.parametrize("kw,code", [
    (dict(parallel=7), 1),
    (dict(tp_size=0), 1),
    (dict(tp_rank=2), 1),
    (dict(n_slices=4), 1),
    (dict(parallel=1, n_slices=2, d_out=[256, 256, 0]), 1),
    (dict(tp_size=4, d_out=[514, 0, 0]), 2),  # column d_out not divisible by N
    (dict(max_rank=7), 2),               # N does not divide max_rank
    (dict(parallel=1, tp_size=4, d_in=510), 2),  # row d_in not divisible by N
    (dict(capacity=0), 3),
    (dict(max_rank=5000), 3),
])
def test_create_pool_validation(lib, kw, code):
    h = ctypes.c_void_p()
    d = _desc(**kw)
    rc = lib.bdlora_create_pool(ctypes.byref(d), 0, ctypes.byref(h))
    assert rc == code, lib.bdlora_last_error()
    assert lib.bdlora_last_error() != b""


def test_null_arguments(lib):
    assert lib.bdlora_create_pool(None, 0, None) == 1
    assert lib.bdlora_workspace_bytes(None, 4, None) == 1
    assert lib.bdlora_column_forward(None, None, 1, None, None, None, None, 0, None) == 1
    assert lib.bdlora_comm_stats(None, None) == 1
    assert lib.bdlora_destroy_pool(None) == 0
    assert lib.bdlora_comm_destroy(None) == 0


def test_peer_host_validation(lib):
    """Fused row all-reduce peer groups: argument errors are caught on the host before any device work."""
    import ctypes as ct

    arr = (ct.c_void_p * 4)()
    assert lib.bdlora_peer_create_local(0, 0, 1024, arr) == 1
    assert lib.bdlora_peer_create_local(2, 0, 0, arr) == 1
    assert lib.bdlora_peer_create_local(2, 0, 1024, None) == 1
    assert lib.bdlora_peer_create(None, 1024, arr) == 1
    assert lib.bdlora_peer_destroy(None) == 0
    assert lib.bdlora_peer_reduce(None, None, 1, 1, None) == 1
    assert lib.bdlora_row_forward_fused(None, None, None, 1, None, None, None, None, 0, None) == 1
    assert lib.bdlora_peer_error(None, None) == 1
    assert lib.bdlora_workspace_init(None, None, 0, None) == 1
    info = (ct.c_int32 * 8)()
    assert lib.bdlora_last_launch_info(info) == 0 and info[0] == -1


def test_device_check_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc = lib.bdlora_device_check(0)
    assert rc in (1, 6), lib.bdlora_last_error()


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load()
