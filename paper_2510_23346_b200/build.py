"""Build libbdlora.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbdlora.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    """NCCL 2.28 shipped with the torch wheel (the one torch.distributed itself loads)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec is not None and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    cands.append(os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                              "site-packages", "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers (nvidia/nccl) not found next to torch")


def sources():
    """Translation units, built in parallel into objects under build/ and linked into one .so."""
    return [os.path.join(CSRC, "runtime.cu"), os.path.join(CSRC, "decode.cu"), os.path.join(CSRC, "peer.cu")]


# private headers of each translation unit (a change rebuilds only the units that include them)
_TU_DEPS = {
    "runtime.cu": ["runtime.cu", "common.cuh", "ptx.cuh", "kernels_core.cuh", "kernels_umma.cuh", "kernels_route.cuh",
                   "decode.h", "peer.h", "../../include/bdlora.h"],
    "decode.cu": ["decode.cu", "decode.h", "kernels_decode.cuh", "common.cuh", "ptx.cuh", "peer.h"],
    "peer.cu": ["peer.cu", "peer.h"],
}


def deps():
    out = []
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            if f.endswith((".cu", ".cuh", ".h", ".hpp")):
                out.append(os.path.join(d, f))
    return out


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in deps())


def _obj(src: str) -> str:
    return os.path.join(ROOT, "build", os.path.basename(src) + ".o")


def _obj_stale(src: str) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return any(os.path.getmtime(os.path.normpath(os.path.join(CSRC, d))) > t
               for d in _TU_DEPS.get(os.path.basename(src), [os.path.basename(src)]))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nc = nccl_dir()
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    common = [
        NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nc, "include"),
        "-DBDLORA_BUILD",
    ]
    procs = []
    for src in sources():
        if force or _obj_stale(src):
            cmd = common + ["-c", src, "-o", _obj(src) + ".tmp"]
            procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, cmd, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out)
        if verbose:
            sys.stderr.write(out)
        os.replace(_obj(src) + ".tmp", _obj(src))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            *[_obj(s) for s in sources()],
            "-L", os.path.join(nc, "lib"), "-l:libnccl.so.2",
            "-Xlinker", f"-rpath={os.path.join(nc, 'lib')}", "-o", LIB + ".tmp"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(link) + "\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
