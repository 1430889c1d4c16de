"""Test harness shared by the GPU parity tests: builds seeded cases (synth), slices the BASE weight
for a device the way Megatron does (the library slices adapters itself in load_adapter), runs the
C-ABI through the Python binding and compares with the fp64 oracle.  Holds no LoRA arithmetic."""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

import synth


def torch_bf16(bits: np.ndarray, device=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)
    return t.to(device) if device is not None else t


def base_shard_T(W: synth.Bf16, proj: synth.Projection, n: int, i: int) -> np.ndarray:
    """W_i^T bits as [M_loc, K_loc] (include/bdlora.h layout) from the paper-orientation W [d_in, sum d_out]."""
    b = W.bits
    if proj.parallel == "column":
        parts = []
        c0 = 0
        for dj in proj.d_out:
            w = dj // n
            parts.append(b[:, c0 + i * w:c0 + (i + 1) * w])
            c0 += dj
        return np.ascontiguousarray(np.concatenate(parts, axis=1).T)
    k = proj.d_in // n
    return np.ascontiguousarray(b[i * k:(i + 1) * k, :].T)


def x_shard(X: synth.Bf16, proj: synth.Projection, n: int, i: int) -> np.ndarray:
    if proj.parallel == "column":
        return X.bits
    k = proj.d_in // n
    return np.ascontiguousarray(X.bits[:, i * k:(i + 1) * k])


@dataclasses.dataclass
class Case:
    proj: synth.Projection
    sharding: str
    n: int
    X: synth.Bf16
    W: synth.Bf16
    ids: np.ndarray
    adapters: Dict[int, synth.AdapterInput]
    capacity: int
    max_rank: int

    def oracle_adapters(self) -> Dict[int, dict]:
        return {a: {"rank": ad.rank, "scale": ad.scale, "A": [x.f64 for x in ad.A], "B": [x.f64 for x in ad.B]}
                for a, ad in self.adapters.items()}


def make_case(seed: int, proj: synth.Projection, sharding: str, n: int, T: int, ranks: Sequence[int],
              ids: Optional[np.ndarray] = None, capacity: Optional[int] = None, zero: Dict[int, str] = None,
              integer: bool = False, w_zero: bool = False, alpha: float = 16.0) -> Case:
    rng = synth.rng_for(seed, 7)
    capacity = capacity or len(ranks)
    zero = zero or {}
    ads = {}
    for a, r in enumerate(ranks):
        if integer:
            s = 2.0 ** (a % 3 - 1)
            ads[a] = synth.make_int_adapter(rng, proj, sharding, r, n, s, signature=a)
        else:
            s = synth.rs_scale(alpha, r, n, sharding)
            ads[a] = synth.make_adapter(rng, proj, sharding, r, n, s, zero=zero.get(a, ""))
    if integer:
        X = synth.int_tensor(rng, (T, proj.d_in), 0.5)
        W = synth.int_tensor(rng, (proj.d_in, sum(proj.d_out)), 0.05)
    else:
        X = synth.make_x(rng, T, proj.d_in)
        W = synth.make_base(rng, proj, zero=w_zero)
    if ids is None:
        ids = synth.ids_runs(rng, T, len(ranks), p_none=0.1)
    return Case(proj, sharding, n, X, W, np.asarray(ids, np.int32), ads, capacity, max(ranks))


def make_pool(case: Case, i: int, device: int = 0, arena_bytes: int = 0):
    import paper_2510_23346_b200 as bd

    par = bd.COLUMN if case.proj.parallel == "column" else bd.ROW
    sh = {"bd": bd.SHARD_BD, "slora": bd.SHARD_SLORA, "nfs": bd.SHARD_NFS}[case.sharding]
    pool = bd.bdlora_create_pool(par, sh, case.n, i, case.proj.d_in, case.proj.d_out, case.capacity,
                                 case.max_rank, arena_bytes=arena_bytes, device=device)
    for a, ad in case.adapters.items():
        bd.bdlora_load_adapter(pool, a, ad.rank, ad.scale, [torch_bf16(x.bits) for x in ad.A],
                               [torch_bf16(x.bits) for x in ad.B])
    return pool


def device_inputs(case: Case, i: int, device):
    import torch

    X = torch_bf16(x_shard(case.X, case.proj, case.n, i), device)
    W = torch_bf16(base_shard_T(case.W, case.proj, case.n, i), device)
    ids = torch.from_numpy(case.ids).to(device)
    return X, W, ids
