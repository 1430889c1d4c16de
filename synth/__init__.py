"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module is deliberately method-free: it draws random numbers, rounds them to
bf16 (round-to-nearest-even) and describes the paper's layer shapes.  It holds
none of the LoRA / sharding arithmetic -- that lives independently in `oracle/`
(fp64, numpy) and in `paper_2510_23346_b200/` (CUDA).  Neither of those imports
the other; both may import this module.

Input recipe:
  X ~ N(0,1), W ~ N(0, 1/d_in), A ~ N(0, 1/d_in),
  B ~ N(0, 1/(s_a^2 * r_a / N)) so that the LoRA delta has O(1) variance like XW,
  all stored as bf16 (RNE from fp32).  Generators are numpy PCG64(seed).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# bf16 helpers (storage format only)
# ----------------------------------------------------------------------------


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 with round-to-nearest-even; return uint16 bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    rounded = (u + 0x7FFF + lsb) >> 16
    # NaN stays NaN (not produced by our generators, kept for completeness)
    nan = np.isnan(x)
    out = rounded.astype(np.uint16)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(bits).astype(np.float64)


@dataclasses.dataclass
class Bf16:
    """A bf16 tensor: canonical bit pattern plus its exact fp64 value."""

    bits: np.ndarray  # uint16

    @property
    def f64(self) -> np.ndarray:
        return bf16_bits_to_f64(self.bits)

    @property
    def shape(self):
        return self.bits.shape


def rng_for(seed: int, *stream: int) -> np.random.Generator:
    """Independent PCG64 stream per (seed, tag...)."""
    ss = np.random.SeedSequence([int(seed)] + [int(s) for s in stream])
    return np.random.Generator(np.random.PCG64(ss))


def bf16_normal(rng: np.random.Generator, shape, std: float) -> Bf16:
    x = rng.standard_normal(size=shape, dtype=np.float32) * np.float32(std)
    return Bf16(f32_to_bf16_bits(x))


def bf16_from_f64(x: np.ndarray) -> Bf16:
    return Bf16(f32_to_bf16_bits(np.asarray(x, dtype=np.float32)))


# ----------------------------------------------------------------------------
# Layer shapes of the paper's workloads (BASELINE.json configs)
# ----------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Projection:
    name: str
    parallel: str  # "column" | "row"
    d_in: int  # FULL input dim
    d_out: Tuple[int, ...]  # FULL output dim per slice (q|k|v, gate|up, or single)


def llama_projections(d_h: int, d_i: int, d_kv: int, d_q: Optional[int] = None) -> List[Projection]:
    d_q = d_h if d_q is None else d_q
    return [
        Projection("qkv", "column", d_h, (d_q, d_kv, d_kv)),
        Projection("o", "row", d_q, (d_h,)),
        Projection("gate_up", "column", d_h, (d_i, d_i)),
        Projection("down", "row", d_i, (d_h,)),
    ]


ARCHS: Dict[str, dict] = {
    # d_kv forced by the paper's parameter counts (SURVEY §8(c) reading #16)
    "llama-3.2-1b": dict(d_h=2048, d_i=8192, d_kv=512, n_layers=16),
    "llama-3.1-8b": dict(d_h=4096, d_i=14336, d_kv=1024, n_layers=32),
    "llama-3.1-70b": dict(d_h=8192, d_i=28672, d_kv=1024, n_layers=80),
    # configs[0]: tiny column+row pair (d=256, d_ff=512)
    "tiny": dict(d_h=256, d_i=512, d_kv=256, n_layers=1),
}


def arch_projections(arch: str) -> List[Projection]:
    a = ARCHS[arch]
    return llama_projections(a["d_h"], a["d_i"], a["d_kv"])


def tiny_pair() -> List[Projection]:
    """configs[0]: column 256->512 (J=1) then row 512->256."""
    return [Projection("col", "column", 256, (512,)), Projection("row", "row", 512, (256,))]


# ----------------------------------------------------------------------------
# Adapter-id streams
# ----------------------------------------------------------------------------


def ids_runs(rng: np.random.Generator, T: int, n_adapters: int, p_none: float = 0.0,
             mean_run: float = 2.0) -> np.ndarray:
    """Runs of mixed length of equal ids (exercise segments), optional -1 tokens."""
    out = np.empty(T, dtype=np.int32)
    t = 0
    while t < T:
        run = 1 + int(rng.geometric(1.0 / mean_run)) - 1
        run = max(1, min(run, T - t))
        a = -1 if rng.random() < p_none else int(rng.integers(0, n_adapters))
        out[t:t + run] = a
        t += run
    return out


def ids_uniform(rng: np.random.Generator, T: int, n_adapters: int) -> np.ndarray:
    return rng.integers(0, n_adapters, size=T).astype(np.int32)


def ids_zipf(rng: np.random.Generator, T: int, n_adapters: int, a: float = 1.0) -> np.ndarray:
    ranks = np.arange(1, n_adapters + 1, dtype=np.float64)
    p = ranks ** (-a)
    p /= p.sum()
    return rng.choice(n_adapters, size=T, p=p).astype(np.int32)


def ids_distinct(rng: np.random.Generator, T: int, n_adapters: int) -> np.ndarray:
    assert T <= n_adapters
    return rng.permutation(n_adapters)[:T].astype(np.int32)


def ids_segments(T: int, n_requests: int, first_adapter: int = 0) -> np.ndarray:
    """Prefill batch: n_requests contiguous requests of T/n_requests tokens each."""
    per = T // n_requests
    out = np.empty(T, dtype=np.int32)
    for q in range(n_requests):
        hi = T if q == n_requests - 1 else (q + 1) * per
        out[q * per:hi] = first_adapter + q
    return out


# ----------------------------------------------------------------------------
# Factor generators in the LOAD format of the C-ABI (include/bdlora.h):
#   column+BD : A[j] d_in x r ; B[j] compact (r/N) x d_out[j] (blocks side by side)
#   row+BD    : A compact d_in x (r/N) (blocks stacked) ; B r x d_out
#   *+SLORA / NFS / plain : dense A[j] d_in x r ; B[j] r x d_out[j]
# ----------------------------------------------------------------------------


def rs_scale(alpha: float, r: int, n: int, sharding: str) -> float:
    """Scale s_a used by the benches: rsLoRA alpha/sqrt(r) or BD alpha*sqrt(N)/sqrt(r).

    This is a bench/generator convention only (the library receives s as an input)."""
    if sharding == "bd":
        return alpha * math.sqrt(n) / math.sqrt(r)
    return alpha / math.sqrt(r)


@dataclasses.dataclass
class AdapterInput:
    rank: int
    scale: float
    A: List[Bf16]  # per slice (row layers: 1)
    B: List[Bf16]


def make_adapter(rng: np.random.Generator, proj: Projection, sharding: str, rank: int, n: int,
                 scale: float, zero: str = "") -> AdapterInput:
    """One adapter's factors in load format for `sharding` in {"bd", "slora", "nfs"} (S-LoRA and NFS-LoRA
    take dense factors, include/bdlora.h).

    zero: "" | "A" | "B"  -> force that factor to exact zeros (P5)."""
    J = len(proj.d_out)
    rl = rank // n if sharding == "bd" else rank
    b_std = 1.0 / math.sqrt(max(scale, 1e-30) ** 2 * max(rank / n, 1.0))
    a_std = 1.0 / math.sqrt(proj.d_in)
    As: List[Bf16] = []
    Bs: List[Bf16] = []
    for j in range(J):
        if sharding == "bd" and proj.parallel == "row":
            a_shape = (proj.d_in, rank // n)
        else:
            a_shape = (proj.d_in, rank)
        if sharding == "bd" and proj.parallel == "column":
            b_shape = (rank // n, proj.d_out[j])
        else:
            b_shape = (rank, proj.d_out[j])
        A = bf16_normal(rng, a_shape, a_std)
        B = bf16_normal(rng, b_shape, b_std)
        if zero == "A":
            A = Bf16(np.zeros(a_shape, np.uint16))
        if zero == "B":
            B = Bf16(np.zeros(b_shape, np.uint16))
        As.append(A)
        Bs.append(B)
    del rl
    return AdapterInput(rank=rank, scale=float(np.float32(scale)), A=As, B=Bs)


def make_base(rng: np.random.Generator, proj: Projection, zero: bool = False) -> Bf16:
    """Base weight in the PAPER orientation W in R^{d_in x sum_j d_out_j}."""
    shape = (proj.d_in, int(sum(proj.d_out)))
    if zero:
        return Bf16(np.zeros(shape, np.uint16))
    return bf16_normal(rng, shape, 1.0 / math.sqrt(proj.d_in))


def make_x(rng: np.random.Generator, T: int, d: int) -> Bf16:
    return bf16_normal(rng, (T, d), 1.0)


# ----------------------------------------------------------------------------
# Exact-integer mode (P10): entries in {-1,0,1}, sparse W, s a power of two
# ----------------------------------------------------------------------------


def int_tensor(rng: np.random.Generator, shape, p_nonzero: float) -> Bf16:
    v = rng.integers(-1, 2, size=shape).astype(np.float32)
    mask = rng.random(size=shape) < p_nonzero
    return bf16_from_f64(np.where(mask, v, 0.0))


def make_int_adapter(rng: np.random.Generator, proj: Projection, sharding: str, rank: int, n: int,
                     scale: float, signature: int) -> AdapterInput:
    """Integer adapter: A, B in {-1,0,1}; B carries a distinct per-adapter signature
    (B[0, signature % d_out_j] = 1 for the first slice) so routing errors show up."""
    base = make_adapter(rng, proj, sharding, rank, n, scale)
    As, Bs = [], []
    for j, (A, B) in enumerate(zip(base.A, base.B)):
        As.append(int_tensor(rng, A.shape, 0.05))
        b = int_tensor(rng, B.shape, 0.05).f64
        b[0, (signature * 7 + j) % b.shape[1]] = 1.0
        Bs.append(bf16_from_f64(b))
    return AdapterInput(rank=rank, scale=scale, A=As, B=Bs)
