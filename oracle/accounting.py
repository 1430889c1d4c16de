"""Closed-form accounting of BD-LoRA vs LoRA / S-LoRA (TEST INFRASTRUCTURE ONLY -- see oracle/lora.py).

Everything here is a formula the paper states, written out:
  * trainable-parameter counts per projection (App. A Table "costs"; the per-projection
    rule reproduces every "# Trainable Parameters" value in the result tables, e.g. P:1273-1283),
  * the parameter-matched BD rank r' = r (d_H + d_I) / (d_H + d_I/N),
  * LoRA FLOPs = 2 * S * (# parameters) per factor,
  * S-LoRA's extra communication per attention module 5(N-1) r S / N vs the base's
    2(N-1) d_H S / N,
  * rsLoRA and BD-rsLoRA scaling factors alpha/sqrt(r), alpha*sqrt(N)/sqrt(r),
  * the collective-count table of Fig. 2 / Fig. 3.

Pinned by tests/test_oracle_pins.py against the integers the paper prints.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, Tuple

# Llama shapes (d_kv forced by the printed counts, SURVEY §8(c) reading #16)
ARCH = {
    "llama-3.2-1b": dict(d_h=2048, d_i=8192, d_q=2048, d_kv=512, n_layers=16),
    "llama-3.1-8b": dict(d_h=4096, d_i=14336, d_q=4096, d_kv=1024, n_layers=32),
    "llama-3.1-70b": dict(d_h=8192, d_i=28672, d_q=8192, d_kv=1024, n_layers=80),
}


def params_dense(d_in: int, d_out: int, r: int) -> int:
    """Plain LoRA on d_in -> d_out: A d_in x r plus B r x d_out."""
    return (d_in + d_out) * r


def params_bd_column(d_in: int, d_out: int, r: int, n: int) -> int:
    """BD column projection: A_1 dense d_in x r, B_1 block-diagonal with N blocks of
    (r/N) x (d_out/N) -> d_out * r / N non-zeros (rows A_1 / B_1)."""
    if r % n:
        raise ValueError("BD-LoRA needs N | r (P:462)")
    return d_in * r + d_out * r // n


def params_bd_row(d_in: int, d_out: int, r: int, n: int) -> int:
    """BD row projection: A_2 block-diagonal (d_in * r / N non-zeros), B_2 dense r x d_out."""
    if r % n:
        raise ValueError("BD-LoRA needs N | r (P:462)")
    return d_in * r // n + d_out * r


def count_params(arch: str, method: str, r: int, n: int = 1, targets: Tuple[str, ...] = ("attn", "mlp")) -> int:
    """Whole-model trainable parameters: q,k,v,gate,up column; o,down row."""
    a = ARCH[arch]
    d_h, d_i, d_q, d_kv, L = a["d_h"], a["d_i"], a["d_q"], a["d_kv"], a["n_layers"]
    col = [] if "attn" not in targets else [(d_h, d_q), (d_h, d_kv), (d_h, d_kv)]
    row = [] if "attn" not in targets else [(d_q, d_h)]
    if "mlp" in targets:
        col += [(d_h, d_i), (d_h, d_i)]
        row += [(d_i, d_h)]
    total = 0
    for d_in, d_out in col:
        total += params_dense(d_in, d_out, r) if method == "dense" else params_bd_column(d_in, d_out, r, n)
    for d_in, d_out in row:
        total += params_dense(d_in, d_out, r) if method == "dense" else params_bd_row(d_in, d_out, r, n)
    return total * L


def match_rank(d_h: int, d_i: int, n: int, r: int) -> Fraction:
    """r' = r (d_H + d_I) / (d_H + d_I / N), exact rational."""
    return Fraction(r * (d_h + d_i)) / (Fraction(d_h) + Fraction(d_i, n))


def mlp_params_per_device(d_h: int, d_i: int, n: int, r, method: str):
    """Sum row of Table "costs": S-LoRA 2 (d_H + d_I) r/N, BD 2 (d_H + d_I/N) r'/N."""
    r = Fraction(r)
    if method == "slora":
        return 2 * (d_h + d_i) * r / n
    return 2 * (Fraction(d_h) + Fraction(d_i, n)) * r / n


def mlp_lora_flops_per_device(S: int, d_h: int, d_i: int, n: int, r, method: str):
    """# operations column: 2 * S * (# parameters), per factor and summed."""
    return 2 * S * mlp_params_per_device(d_h, d_i, n, r, method)


def slora_attn_comm_elems(n: int, r: int, S: int) -> Fraction:
    """Extra elements communicated per attention module by S-LoRA: 5 (N-1) r S / N."""
    return Fraction(5 * (n - 1) * r * S, n)


def base_attn_comm_elems(n: int, d_h: int, S: int) -> Fraction:
    """Base model's 2 (N-1) d_H S / N."""
    return Fraction(2 * (n - 1) * d_h * S, n)


def scale_standard(alpha: float, r: int) -> float:
    return alpha / r


def scale_rslora(alpha: float, r: int) -> float:
    """gamma_r = alpha / sqrt(r)."""
    return alpha / r ** 0.5


def scale_bd_rslora(alpha: float, r: int, n: int) -> float:
    """BD-LoRA trains independent rank r/N adapters: alpha * sqrt(N) / sqrt(r)."""
    if r % n:
        raise ValueError("N | r required")
    return alpha * n ** 0.5 / r ** 0.5


def lora_collectives(method: str, module: str, merged: bool = True) -> Dict[str, int]:
    """LoRA-specific collectives per module on top of the base's single all-reduce.

    S-LoRA: basic MLP 1 AG + 1 AR; GLU 2 AG + 1 AR; attention 3 AG + 1 AR
    (P:336-341), merged to 1 AG in practice (P:340-341 footnote).  BD-LoRA and NFS-LoRA: none
    (Fig. 3 caption P:438-443)."""
    if method in ("bd", "nfs", "base"):
        return {"all_gather": 0, "all_reduce": 0}
    ag = {"mlp": 1, "glu": 2, "attn": 3}[module]
    return {"all_gather": 1 if merged else ag, "all_reduce": 1}
