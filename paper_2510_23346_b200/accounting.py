"""Algorithmic bytes and FLOPs of one projection on one device for one step of T tokens
(DESIGN.md "Roofline").  Host-side bookkeeping for bench.py -- no layer math.

Counted: the base weight shard, the activations in and out, and for every DISTINCT adapter touched
this step the device-local compact factor shards (block-diagonal zeros are never stored or read,
P:389), plus the int32 ids.  Not counted: the fp32 intermediate v (on-chip / L2 sized),
dense dW (never formed) and S-LoRA's replicated intermediates."""
from __future__ import annotations

from typing import Dict, Iterable, Sequence


def factor_elems(parallel: str, sharding: str, d_in: int, d_out: Sequence[int], n: int, r: int) -> int:
    """Elements of one adapter's factors resident on one device."""
    if parallel == "column":
        tot = 0
        for dj in d_out:
            if sharding == "bd":      # A [r/N, d_in], B [r/N, d_out_j/N]
                tot += d_in * r // n + (r // n) * (dj // n)
            elif sharding == "slora":  # A [r/N, d_in], B [r, d_out_j/N]
                tot += d_in * r // n + r * (dj // n)
            else:                      # nfs: A replicated [r, d_in], B [r, d_out_j/N]
                tot += d_in * r + r * (dj // n)
        return tot
    d = d_out[0]
    if sharding == "bd":               # A [r/N, d_in/N], B [r/N, d_out]
        return (d_in // n) * (r // n) + (r // n) * d
    if sharding == "slora":            # A [r, d_in/N], B [r, d_out/N]
        return (d_in // n) * r + r * (d // n)
    return (d_in // n) * r + r * d     # nfs: B replicated


def proj_bytes(parallel: str, sharding: str, d_in: int, d_out: Sequence[int], n: int, T: int,
               ranks_touched: Iterable[int]) -> int:
    """Algorithmic HBM bytes of one device's projection call (bf16 = 2 B, ids int32)."""
    m_loc = sum(d_out) // n if parallel == "column" else d_out[0]
    k_loc = d_in if parallel == "column" else d_in // n
    e = k_loc * m_loc + T * k_loc + T * m_loc
    for r in ranks_touched:
        e += factor_elems(parallel, sharding, d_in, d_out, n, r)
    return 2 * e + 4 * T


def proj_flops(parallel: str, sharding: str, d_in: int, d_out: Sequence[int], n: int,
               token_ranks: Iterable[int]) -> int:
    """2 * MACs: base GEMM plus per-token LoRA factors (2 * S * params per factor).
    token_ranks: rank of each token's adapter (0 for id -1)."""
    m_loc = sum(d_out) // n if parallel == "column" else d_out[0]
    k_loc = d_in if parallel == "column" else d_in // n
    token_ranks = list(token_ranks)
    f = 2 * len(token_ranks) * k_loc * m_loc
    for r in token_ranks:
        if r:
            f += 2 * factor_elems(parallel, sharding, d_in, d_out, n, r)
    return f


def layer_bytes(projs, sharding: str, n: int, T: int, ranks_touched: Sequence[int]) -> Dict[str, int]:
    return {p.name: proj_bytes(p.parallel, sharding, p.d_in, p.d_out, n, T, ranks_touched) for p in projs}
