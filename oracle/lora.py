"""fp64 CPU oracle of the tensor-parallel multi-adapter LoRA layer (BD-LoRA, arXiv 2510.23346).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` legs may import anything under `oracle/`.  The
product path (`paper_2510_23346_b200/`, `libbdlora.so`) never imports, links or
calls it, and this module imports nothing from the product path.

What it computes is the PLAIN definition of the layer, unsharded, with the dense
adapter update materialised:

    y_t = x_t W + s_{a(t)} x_t (A_{a(t)} B_{a(t)})

with the block-diagonal factors of BD-LoRA expanded to dense matrices
and the per-device outputs read off as column blocks (column-parallel, P:298-304,
P:400-401) or the replicated sum (row-parallel).  Sharding is
an exact algebraic regrouping ("lines 6-16 allow for full parallelization"),
so the sharded GPU result must equal this definition up to fp summation order and
the bf16 rounding points.  No blocking, fusion or reordering is done here.

Notation follows the paper: W in R^{d_in x d_out}, A in R^{d_in x r},
B in R^{r x d_out}; N = number of devices; block i sits on device i.

Pins: tests/test_oracle_pins.py (brute force on tiny integer inputs, closed forms,
special cases, the paper's printed parameter counts).  Functions whose floating
point outputs at realistic shapes have no printed paper value are pinned only
through those properties -- "parity unpinned" for realistic-shape fp values, see
DESIGN.md §Oracle.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# Block-diagonal expansion (compact storage P:1082)
# ----------------------------------------------------------------------------


def bd_expand_side_by_side(compact: np.ndarray, n: int) -> np.ndarray:
    """B1 stored compact as (r/N) x d_out with the N blocks "next to each other".

    Returns the dense r x d_out block-diagonal matrix: block i = compact[:, i*d_out/N:(i+1)*d_out/N]
    placed at rows i*r/N.., columns i*d_out/N.. (SURVEY §8(c) reading #3)."""
    rb, d_out = compact.shape
    assert d_out % n == 0
    cb = d_out // n
    dense = np.zeros((rb * n, d_out), dtype=np.float64)
    for i in range(n):
        dense[i * rb:(i + 1) * rb, i * cb:(i + 1) * cb] = compact[:, i * cb:(i + 1) * cb]
    return dense


def bd_expand_stacked(compact: np.ndarray, n: int) -> np.ndarray:
    """A2 stored compact as d_in x (r/N) with the N blocks "on top of each other".

    Returns the dense d_in x r block-diagonal matrix: block i = compact[i*d_in/N:(i+1)*d_in/N, :]
    placed at rows i*d_in/N.., columns i*r/N.. (SURVEY §8(c) reading #3)."""
    d_in, rb = compact.shape
    assert d_in % n == 0
    bb = d_in // n
    dense = np.zeros((d_in, rb * n), dtype=np.float64)
    for i in range(n):
        dense[i * bb:(i + 1) * bb, i * rb:(i + 1) * rb] = compact[i * bb:(i + 1) * bb, :]
    return dense


def dense_factors(parallel: str, sharding: str, A: Sequence[np.ndarray], B: Sequence[np.ndarray],
                  n: int) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Dense fp64 (A_j, B_j) per slice j from the load format.

    column+bd : A_j dense d_in x r,  B_j = bd_expand_side_by_side(compact)
    row+bd    : A = bd_expand_stacked(compact), B dense r x d_out
    slora/nfs : dense as given
    """
    out = []
    for a, b in zip(A, B):
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        if sharding == "bd" and parallel == "column":
            out.append((a, bd_expand_side_by_side(b, n)))
        elif sharding == "bd" and parallel == "row":
            out.append((bd_expand_stacked(a, n), b))
        elif sharding in ("slora", "nfs", "plain"):
            out.append((a, b))
        else:
            raise ValueError(f"unknown parallel/sharding {parallel}/{sharding}")
    return out


# ----------------------------------------------------------------------------
# The plain layer ("replace the computation of XW ... by XW+XAB", P:266 gamma_r)
# ----------------------------------------------------------------------------


def lora_layer(X: np.ndarray, W: np.ndarray, adapters: Dict[int, Tuple[float, np.ndarray, np.ndarray]],
               ids: np.ndarray, materialise: bool = True) -> np.ndarray:
    """y_t = x_t W + s_a x_t dW_a with dW_a = A_a B_a materialised.

    adapters: slot -> (s, A dense d_in x r, B dense r x d_out).  ids[t] == -1 -> no LoRA term
    (SURVEY §8(c) reading #8).  materialise=False computes the factored (x A) B instead --
    the dual oracle used only as a cross-check."""
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    y = X @ W
    ids = np.asarray(ids)
    for a in sorted(set(int(v) for v in ids.tolist()) - {-1}):
        s, A, B = adapters[a]
        rows = np.nonzero(ids == a)[0]
        if materialise:
            dW = A @ B  # d_in x d_out, one adapter at a time
            y[rows] += s * (X[rows] @ dW)
            del dW
        else:
            y[rows] += s * ((X[rows] @ A) @ B)
    return y


def lora_layer_sampled(X: np.ndarray, W: np.ndarray,
                       adapters: Dict[int, Tuple[float, np.ndarray, np.ndarray]],
                       ids: np.ndarray, samples: Sequence[Tuple[int, int]]) -> np.ndarray:
    """Selected outputs y[t, c] of `lora_layer`, computed one by one for full-size shapes.

    y[t, c] = x_t . W[:, c] + s_a x_t . (A_a B_a[:, c])  -- column c of dW_a materialised."""
    X = np.asarray(X, dtype=np.float64)
    out = np.empty(len(samples), dtype=np.float64)
    for k, (t, c) in enumerate(samples):
        v = float(X[t] @ np.asarray(W[:, c], dtype=np.float64))
        a = int(ids[t])
        if a >= 0:
            s, A, B = adapters[a]
            dW_c = A @ np.asarray(B[:, c], dtype=np.float64)
            v += s * float(X[t] @ dW_c)
        out[k] = v
    return out


# ----------------------------------------------------------------------------
# Column-parallel and row-parallel layers (Alg. 1)
# ----------------------------------------------------------------------------


def _slice_adapters(adapter_inputs: Dict[int, dict], parallel: str, sharding: str, n: int, j: int):
    out = {}
    for slot, ad in adapter_inputs.items():
        fac = dense_factors(parallel, sharding, ad["A"], ad["B"], n)
        A, B = fac[j]
        out[slot] = (float(ad["scale"]), A, B)
    return out


def column_layer(X: np.ndarray, W: np.ndarray, d_out: Sequence[int], adapter_inputs: Dict[int, dict],
                 ids: np.ndarray, sharding: str, n: int) -> List[np.ndarray]:
    """Full (unsharded) output of a column-parallel projection, per slice j.

    W: d_in x sum_j d_out_j with the slices side by side (q|k|v or gate|up, reading #4: each
    slice has its own A_j, B_j).  adapter_inputs: slot -> {"scale", "A": [per slice], "B": [...]}."""
    outs = []
    c0 = 0
    for j, dj in enumerate(d_out):
        Wj = np.asarray(W[:, c0:c0 + dj], dtype=np.float64)
        outs.append(lora_layer(X, Wj, _slice_adapters(adapter_inputs, "column", sharding, n, j), ids))
        c0 += dj
    return outs


def column_device_output(slice_outputs: Sequence[np.ndarray], n: int, i: int) -> np.ndarray:
    """Device i's expected output = concat_j y_j[:, i*d_out_j/N:(i+1)*d_out_j/N] ("column-sharded";
    block i on device i)."""
    parts = []
    for y in slice_outputs:
        w = y.shape[1] // n
        parts.append(y[:, i * w:(i + 1) * w])
    return np.concatenate(parts, axis=1)


def row_layer(X_full: np.ndarray, W: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray,
              sharding: str, n: int) -> np.ndarray:
    """Replicated output of a row-parallel projection y = AllReduce_i(P_i) = X_full W + s X_full A B
    (Alg. 1 line 15)."""
    return lora_layer(X_full, W, _slice_adapters(adapter_inputs, "row", sharding, n, 0), ids)


def row_partial_bd(X_full: np.ndarray, W: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray,
                   n: int, i: int) -> np.ndarray:
    """Per-device partial of a BD-LoRA row layer, Alg. 1 lines 9-12:

        P_i = X^i W^i + s (X^i A_2^(i)) B_2^(i)

    X^i = X_full[:, i*d_in/N:(i+1)*d_in/N]; W^i = W[i*d_in/N:(i+1)*d_in/N, :] (row shard);
    A_2^(i) = the i-th stacked compact block (d_in/N x r/N, reading #6);
    B_2^(i) = B_2[i*r/N:(i+1)*r/N, :] (row shard).  Sum over i is pinned to `row_layer` (P2)."""
    X_full = np.asarray(X_full, dtype=np.float64)
    d_in = X_full.shape[1]
    bi = d_in // n
    Xi = X_full[:, i * bi:(i + 1) * bi]
    Wi = np.asarray(W[i * bi:(i + 1) * bi, :], dtype=np.float64)
    P = Xi @ Wi
    for a in sorted(set(int(v) for v in np.asarray(ids).tolist()) - {-1}):
        ad = adapter_inputs[a]
        r = int(ad["rank"])
        rb = r // n
        A_c = np.asarray(ad["A"][0], dtype=np.float64)  # d_in x r/N compact, stacked
        B = np.asarray(ad["B"][0], dtype=np.float64)    # r x d_out
        Ai = A_c[i * bi:(i + 1) * bi, :]
        Bi = B[i * rb:(i + 1) * rb, :]
        rows = np.nonzero(np.asarray(ids) == a)[0]
        P[rows] += float(ad["scale"]) * (Xi[rows] @ Ai @ Bi)
    return P


def row_partial_bd_blocks(X_full: np.ndarray, W: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray,
                          n_blocks: int, n_dev: int, i: int) -> np.ndarray:
    """Downward-compatible BD-LoRA row partial: an adapter trained with N_h = n_blocks diagonal
    blocks served on N_l = n_dev devices.  Device i holds the row shard i of X, W (d_in/N_l rows) and
    runs the N_h-layout devices i*m .. (i+1)*m - 1 (m = N_h/N_l):

        P_i = X^i W^i + s X^i (A_2[rows i, :] B_2),   A_2 = bd_expand_stacked(compact, N_h)

    i.e. the dense block-diagonal A_2 of the TRAINING layout restricted to this device's rows.  Pinned
    to the sum of the N_h-layout partials `row_partial_bd(..., N_h, d)` over d in the group and, summed
    over i, to `row_layer(..., "bd", N_h)` (tests/test_oracle_pins.py)."""
    X_full = np.asarray(X_full, dtype=np.float64)
    d_in = X_full.shape[1]
    bi = d_in // n_dev
    Xi = X_full[:, i * bi:(i + 1) * bi]
    P = Xi @ np.asarray(W[i * bi:(i + 1) * bi, :], dtype=np.float64)
    for a in sorted(set(int(v) for v in np.asarray(ids).tolist()) - {-1}):
        ad = adapter_inputs[a]
        A = bd_expand_stacked(np.asarray(ad["A"][0], dtype=np.float64), n_blocks)
        B = np.asarray(ad["B"][0], dtype=np.float64)
        rows = np.nonzero(np.asarray(ids) == a)[0]
        P[rows] += float(ad["scale"]) * (Xi[rows] @ (A[i * bi:(i + 1) * bi, :] @ B))
    return P


def row_partial_nfs(X_full: np.ndarray, W: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray,
                    n: int, i: int) -> np.ndarray:
    """Per-device partial of an NFS-LoRA row layer ("adapters A_1 and B_2 are not sharded
    across devices, but replicated so that each device maintains a full copy"; A_2 keeps the standard
    row sharding of the base weight):

        P_i = X^i W^i + s (X^i A_2[i*d_in/N:(i+1)*d_in/N, :]) B_2          (full rank r, full B_2)

    The base all-reduce sums the partials (same collective count as BD-LoRA).  Sum over i is
    pinned to `row_layer(..., "nfs", n)` (tests/test_oracle_pins.py)."""
    X_full = np.asarray(X_full, dtype=np.float64)
    d_in = X_full.shape[1]
    bi = d_in // n
    Xi = X_full[:, i * bi:(i + 1) * bi]
    P = Xi @ np.asarray(W[i * bi:(i + 1) * bi, :], dtype=np.float64)
    for a in sorted(set(int(v) for v in np.asarray(ids).tolist()) - {-1}):
        ad = adapter_inputs[a]
        A = np.asarray(ad["A"][0], dtype=np.float64)  # d_in x r, dense
        B = np.asarray(ad["B"][0], dtype=np.float64)  # r x d_out, replicated
        rows = np.nonzero(np.asarray(ids) == a)[0]
        P[rows] += float(ad["scale"]) * (Xi[rows] @ A[i * bi:(i + 1) * bi, :] @ B)
    return P


def column_shard_nfs(X: np.ndarray, W: np.ndarray, d_out: Sequence[int], adapter_inputs: Dict[int, dict],
                     ids: np.ndarray, n: int, i: int) -> np.ndarray:
    """Device i of an NFS-LoRA column layer computed shard-locally: A_1 replicated (the full
    v = X A_1, N-fold redundant), B_1 column-sharded like W_1:

        Y^i_j = X W_j^(i) + s (X A_j) B_j[:, i*d_out_j/N:(i+1)*d_out_j/N]

    Pinned to `column_layer(..., "nfs", n)` (tests/test_oracle_pins.py)."""
    X = np.asarray(X, dtype=np.float64)
    parts = []
    c0 = 0
    for j, dj in enumerate(d_out):
        w = dj // n
        Y = X @ np.asarray(W[:, c0 + i * w:c0 + (i + 1) * w], dtype=np.float64)
        for a in sorted(set(int(v) for v in np.asarray(ids).tolist()) - {-1}):
            ad = adapter_inputs[a]
            A = np.asarray(ad["A"][j], dtype=np.float64)
            B = np.asarray(ad["B"][j], dtype=np.float64)[:, i * w:(i + 1) * w]
            rows = np.nonzero(np.asarray(ids) == a)[0]
            Y[rows] += float(ad["scale"]) * ((X[rows] @ A) @ B)
        parts.append(Y)
        c0 += dj
    return np.concatenate(parts, axis=1)


def column_shard_bd(X: np.ndarray, W: np.ndarray, d_out: Sequence[int], adapter_inputs: Dict[int, dict],
                    ids: np.ndarray, n: int, i: int) -> np.ndarray:
    """Device i of a BD-LoRA column layer computed shard-locally, Alg. 2 lines 3-6:

        Y^i_j = X W_j^(i) + s (X A_j^(i)) B_j^(i)

    W_j^(i) = column block i of slice j; A_j^(i) = columns i*r/N.. of A_j (column shard);
    B_j^(i) = compact[:, i*d_out_j/N..] (diagonal block i).  Pinned to `column_layer` (P2)."""
    X = np.asarray(X, dtype=np.float64)
    parts = []
    c0 = 0
    for j, dj in enumerate(d_out):
        w = dj // n
        Wij = np.asarray(W[:, c0 + i * w:c0 + (i + 1) * w], dtype=np.float64)
        Y = X @ Wij
        for a in sorted(set(int(v) for v in np.asarray(ids).tolist()) - {-1}):
            ad = adapter_inputs[a]
            rb = int(ad["rank"]) // n
            A = np.asarray(ad["A"][j], dtype=np.float64)[:, i * rb:(i + 1) * rb]
            B = np.asarray(ad["B"][j], dtype=np.float64)[:, i * w:(i + 1) * w]
            rows = np.nonzero(np.asarray(ids) == a)[0]
            Y[rows] += float(ad["scale"]) * ((X[rows] @ A) @ B)
        parts.append(Y)
        c0 += dj
    return np.concatenate(parts, axis=1)


# ----------------------------------------------------------------------------
# S-LoRA intermediates: what the extra collectives carry
# ----------------------------------------------------------------------------


def slora_column_gathered_v(X: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray, j: int
                            ) -> Dict[int, np.ndarray]:
    """After matmul_3 + all-gather: v_t = s_a x_t A_j (full rank r).  token -> vector."""
    X = np.asarray(X, dtype=np.float64)
    out = {}
    for t, a in enumerate(np.asarray(ids).tolist()):
        if a < 0:
            continue
        ad = adapter_inputs[a]
        out[t] = float(ad["scale"]) * (X[t] @ np.asarray(ad["A"][j], dtype=np.float64))
    return out


def slora_row_reduced_v(X_full: np.ndarray, adapter_inputs: Dict[int, dict], ids: np.ndarray
                        ) -> Dict[int, np.ndarray]:
    """After matmul_5 + all-reduce: v_t = s_a x_t A_2 (full input, full rank)."""
    return slora_column_gathered_v(X_full, adapter_inputs, ids, 0)


# ----------------------------------------------------------------------------
# Routing metadata: segments (SURVEY §8(a) a2, §8(c) reading #10)
# ----------------------------------------------------------------------------


def segments(ids: Sequence[int]) -> List[Tuple[int, int, int]]:
    """Maximal runs of equal consecutive ids in token order: (start, length, id).

    No permutation; two runs of the same id stay separate; -1 runs are segments too."""
    out: List[Tuple[int, int, int]] = []
    ids = [int(v) for v in ids]
    t = 0
    while t < len(ids):
        u = t
        while u + 1 < len(ids) and ids[u + 1] == ids[t]:
            u += 1
        out.append((t, u - t + 1, ids[t]))
        t = u + 1
    return out


# ----------------------------------------------------------------------------
# Comparison rule (BASELINE north_star tolerance)
# ----------------------------------------------------------------------------


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> nearest bf16 value (RNE), returned as fp64.  Used for the exact-integer mode (P10),
    where both sides take one RNE rounding of an exact value (SURVEY §8(c) reading #7)."""
    x32 = np.asarray(x, dtype=np.float64).astype(np.float32)
    # fp64 -> fp32 is exact for the integer-mode values (|v| < 2^24); then RNE to bf16
    u = x32.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = (((u + 0x7FFF + lsb) >> 16) << 16).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def within_tolerance(y_gpu: np.ndarray, y_ref: np.ndarray, max_rel: float = 2e-2, l1_rel: float = 5e-3
                     ) -> Tuple[bool, float, float]:
    """max|y - y_ref| <= 2e-2 * max|y_ref| and sum|y - y_ref| / sum|y_ref| <= 5e-3."""
    y = np.asarray(y_gpu, dtype=np.float64)
    r = np.asarray(y_ref, dtype=np.float64)
    if r.size == 0:
        return True, 0.0, 0.0
    err = np.abs(y - r)
    scale = float(np.max(np.abs(r)))
    l1 = float(np.sum(np.abs(r)))
    m = float(err.max()) / scale if scale > 0 else float(err.max())
    l = float(err.sum()) / l1 if l1 > 0 else float(err.sum())
    return (m <= max_rel and l <= l1_rel), m, l
