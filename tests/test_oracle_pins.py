"""Pins of the fp64 oracle against what the paper and the mathematics fix (CPU only).

Each test says which SURVEY §8(c) pin (P1..P11) it realises and which passage fixes it.
The brute-force references below are pure-Python loops over the PER-SHARD formulation of
Alg. 1 / Alg. 2 ("independent LoRA adapters of rank r/N" P:457-478) -- a
different formulation from the oracle's dense block-diagonal expansion, so a dropped term,
a wrong block offset, a transposed operand or a missing scale fails here.
"""
import decimal
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import accounting as acc
from oracle import lora as ol
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- helpers

def _int_mat(rng, shape, lo=-2, hi=3):
    return rng.integers(lo, hi, size=shape).astype(np.float64)


def _bf_column_device(X, W, d_out, adapters, ids, n, i):
    """Pure-Python Alg. 2 lines 3-6 on device i: Y^i = X W^(i) + s (X A^(i)) B^(i), per slice j."""
    T, d_in = len(X), len(X[0])
    out_cols = []
    c0 = 0
    for j, dj in enumerate(d_out):
        w = dj // n
        for cc in range(i * w, (i + 1) * w):
            col = []
            for t in range(T):
                v = 0.0
                for d in range(d_in):
                    v += X[t][d] * W[d][c0 + cc]
                a = ids[t]
                if a >= 0:
                    ad = adapters[a]
                    rb = ad["rank"] // n
                    A = ad["A"][j]          # d_in x r   (column shard i: columns i*rb..)
                    Bc = ad["B"][j]         # (r/N) x d_out_j compact, block i: columns i*w..
                    for k in range(rb):
                        z = 0.0
                        for d in range(d_in):
                            z += X[t][d] * A[d][i * rb + k]
                        v += ad["scale"] * z * Bc[k][cc]
                col.append(v)
            out_cols.append(col)
        c0 += dj
    return np.array(out_cols).T


def _bf_row_partial(X, W, adapters, ids, n, i):
    """Pure-Python Alg. 1 lines 9-12 on device i: P_i = X^i W^i + s (X^i A_2^(i)) B_2^(i)."""
    T, d_in = len(X), len(X[0])
    d_out = len(W[0])
    bi = d_in // n
    P = [[0.0] * d_out for _ in range(T)]
    for t in range(T):
        for c in range(d_out):
            v = 0.0
            for d in range(i * bi, (i + 1) * bi):
                v += X[t][d] * W[d][c]
            a = ids[t]
            if a >= 0:
                ad = adapters[a]
                rb = ad["rank"] // n
                Ac = ad["A"][0]   # d_in x r/N, blocks stacked: block i = rows i*bi..
                B = ad["B"][0]    # r x d_out, row shard i = rows i*rb..
                for k in range(rb):
                    z = 0.0
                    for d in range(i * bi, (i + 1) * bi):
                        z += X[t][d] * Ac[d][k]
                    v += ad["scale"] * z * B[i * rb + k][c]
            P[t][c] = v
    return np.array(P)


def _tiny_bd(rng, parallel, n, d_in=8, d_out=(8, 4), r=4, n_ad=3, scales=(2.0, 0.5, -1.0)):
    J = len(d_out) if parallel == "column" else 1
    d_out = d_out if parallel == "column" else (d_out[0],)
    ads = {}
    for a in range(n_ad):
        As, Bs = [], []
        for j in range(J):
            if parallel == "column":
                As.append(_int_mat(rng, (d_in, r)))
                Bs.append(_int_mat(rng, (r // n, d_out[j])))
            else:
                As.append(_int_mat(rng, (d_in, r // n)))
                Bs.append(_int_mat(rng, (r, d_out[j])))
        ads[a] = {"rank": r, "scale": scales[a % len(scales)], "A": As, "B": Bs}
    return d_out, ads


# ----------------------------------------------------------------------------- P1

def test_bd_expand_spec_examples():
    # SPEC S:197-199 examples: n=1 -> the single block; n=2 blocks [[1]],[[2]] -> [[1,0],[0,2]]
    c = np.array([[1.0, 2.0]])  # (r/N=1) x d_out=2, two 1x1 blocks side by side
    assert np.array_equal(ol.bd_expand_side_by_side(c, 2), np.array([[1.0, 0.0], [0.0, 2.0]]))
    c2 = np.array([[1.0], [2.0]])  # d_in=2 x r/N=1, stacked
    assert np.array_equal(ol.bd_expand_stacked(c2, 2), np.array([[1.0, 0.0], [0.0, 2.0]]))
    m = np.arange(6.0).reshape(2, 3)
    assert np.array_equal(ol.bd_expand_side_by_side(m, 1), m)
    assert np.array_equal(ol.bd_expand_stacked(m, 1), m)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_block_diag_identity_bruteforce(n):
    """P1: [X^1|..|X^N] blockdiag(W^1..W^N) = [X^1W^1|..|X^NW^N]; zeros never touched."""
    rng = np.random.default_rng(n)
    bi, bo, T = 3, 5, 4
    X = _int_mat(rng, (T, bi * n))
    compact = _int_mat(rng, (bi * n, bo)) + 0.5   # non-zero entries, stacked blocks W^i
    dense = ol.bd_expand_stacked(compact, n)      # stacked compact d_in x (r/N) -> dense d_in x r
    assert dense.shape == (bi * n, bo * n)
    assert np.count_nonzero(dense) == compact.size
    lhs = X @ dense
    for i in range(n):
        for t in range(T):
            for c in range(bo):
                v = sum(X[t][i * bi + d] * compact[i * bi + d][c] for d in range(bi))
                assert lhs[t][i * bo + c] == v
    # side-by-side orientation (B_1): Z [T, r] times blockdiag of (r/N) x (d_out/N) blocks
    rb, cb = 2, 3
    Z = _int_mat(rng, (T, rb * n))
    cmp2 = _int_mat(rng, (rb, cb * n)) + 0.5
    d2 = ol.bd_expand_side_by_side(cmp2, n)
    assert d2.shape == (rb * n, cb * n) and np.count_nonzero(d2) == cmp2.size
    lhs2 = Z @ d2
    for i in range(n):
        for t in range(T):
            for c in range(cb):
                v = sum(Z[t][i * rb + k] * cmp2[k][i * cb + c] for k in range(rb))
                assert lhs2[t][i * cb + c] == v


# ----------------------------------------------------------------------------- P2 / P10 brute force

@pytest.mark.parametrize("n", [1, 2, 4])
def test_column_layer_matches_per_shard_bruteforce(n):
    """P2 + P10: oracle column layer (dense expanded factors, unsharded) read off per device equals the
    pure-Python per-shard Alg. 2 on integer inputs, exactly."""
    rng = np.random.default_rng(10 + n)
    d_out, ads = _tiny_bd(rng, "column", n)
    T, d_in = 7, 8
    X = _int_mat(rng, (T, d_in))
    W = _int_mat(rng, (d_in, sum(d_out)))
    ids = np.array([0, 0, 2, -1, 1, 2, 0], dtype=np.int32)
    full = ol.column_layer(X, W, d_out, ads, ids, "bd", n)
    for i in range(n):
        got = ol.column_device_output(full, n, i)
        ref = _bf_column_device(X.tolist(), W.tolist(), d_out, ads, ids.tolist(), n, i)
        assert got.shape == ref.shape
        assert np.array_equal(got, ref)
        assert np.array_equal(ol.column_shard_bd(X, W, d_out, ads, ids, n, i), ref)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_row_layer_matches_sum_of_bruteforce_partials(n):
    """P2 + P10: sum_i P_i (Alg. 1 line 15 all-reduce) equals the oracle's unsharded row layer, and the
    oracle's per-rank partial equals the pure-Python one, exactly on integers."""
    rng = np.random.default_rng(20 + n)
    d_out, ads = _tiny_bd(rng, "row", n, d_in=8, d_out=(6,))
    T, d_in = 6, 8
    X = _int_mat(rng, (T, d_in))
    W = _int_mat(rng, (d_in, d_out[0]))
    ids = np.array([1, -1, 1, 0, 2, 2], dtype=np.int32)
    y = ol.row_layer(X, W, ads, ids, "bd", n)
    acc_ = np.zeros_like(y)
    for i in range(n):
        ref = _bf_row_partial(X.tolist(), W.tolist(), ads, ids.tolist(), n, i)
        got = ol.row_partial_bd(X, W, ads, ids, n, i)
        assert np.array_equal(got, ref)
        acc_ += ref
    assert np.array_equal(acc_, y)


def test_column_layer_random_float_shard_equivalence():
    """P2 on random fp values (sharded regrouping is exact up to summation order)."""
    rng = np.random.default_rng(3)
    n = 4
    d_in, d_out, r = 32, (64, 16, 16), 8
    ads = {}
    for a in range(3):
        ads[a] = {"rank": r, "scale": 1.7, "A": [rng.standard_normal((d_in, r)) for _ in d_out],
                  "B": [rng.standard_normal((r // n, dj)) for dj in d_out]}
    X = rng.standard_normal((9, d_in))
    W = rng.standard_normal((d_in, sum(d_out)))
    ids = np.array([0, 1, 2, -1, 0, 0, 2, 1, 1])
    full = ol.column_layer(X, W, d_out, ads, ids, "bd", n)
    for i in range(n):
        a = ol.column_device_output(full, n, i)
        b = ol.column_shard_bd(X, W, d_out, ads, ids, n, i)
        assert np.allclose(a, b, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------- NFS-LoRA

def _bf_nfs_column_device(X, W, d_out, adapters, ids, n, i):
    """Pure-Python NFS column device i: full A_1 (replicated), B_1 column block i."""
    T, d_in = len(X), len(X[0])
    cols, c0 = [], 0
    for j, dj in enumerate(d_out):
        w = dj // n
        for cc in range(i * w, (i + 1) * w):
            col = []
            for t in range(T):
                v = sum(X[t][d] * W[d][c0 + cc] for d in range(d_in))
                a = ids[t]
                if a >= 0:
                    ad = adapters[a]
                    for k in range(ad["rank"]):
                        z = sum(X[t][d] * ad["A"][j][d][k] for d in range(d_in))
                        v += ad["scale"] * z * ad["B"][j][k][cc]
                col.append(v)
            cols.append(col)
        c0 += dj
    return np.array(cols).T


def _bf_nfs_row_partial(X, W, adapters, ids, n, i):
    """Pure-Python NFS row partial on device i: A_2 row shard i (full rank), B_2 replicated."""
    T, d_in, d_out = len(X), len(X[0]), len(W[0])
    bi = d_in // n
    P = [[0.0] * d_out for _ in range(T)]
    for t in range(T):
        for c in range(d_out):
            v = sum(X[t][d] * W[d][c] for d in range(i * bi, (i + 1) * bi))
            a = ids[t]
            if a >= 0:
                ad = adapters[a]
                for k in range(ad["rank"]):
                    z = sum(X[t][d] * ad["A"][0][d][k] for d in range(i * bi, (i + 1) * bi))
                    v += ad["scale"] * z * ad["B"][0][k][c]
            P[t][c] = v
    return np.array(P)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_nfs_column_and_row_bruteforce(n):
    """NFS-LoRA: replicated A_1 / B_2 make every device's LoRA term local (no LoRA
    collective); the oracle's unsharded layer read off per device, its shard-local form, and the
    pure-Python per-shard loops agree exactly on integers, and the row partials sum to the layer."""
    rng = np.random.default_rng(40 + n)
    d_in, d_out, r, T = 8, (8, 4), 3, 6   # NFS needs no N | r
    ads = {a: {"rank": r, "scale": (2.0, -0.5)[a], "A": [_int_mat(rng, (d_in, r)) for _ in d_out],
               "B": [_int_mat(rng, (r, dj)) for dj in d_out]} for a in range(2)}
    X = _int_mat(rng, (T, d_in))
    W = _int_mat(rng, (d_in, sum(d_out)))
    ids = np.array([1, -1, 0, 0, 1, 1], dtype=np.int32)
    full = ol.column_layer(X, W, d_out, ads, ids, "nfs", n)
    for i in range(n):
        ref = _bf_nfs_column_device(X.tolist(), W.tolist(), d_out, ads, ids.tolist(), n, i)
        assert np.array_equal(ol.column_device_output(full, n, i), ref)
        assert np.array_equal(ol.column_shard_nfs(X, W, d_out, ads, ids, n, i), ref)
    rads = {a: {"rank": r, "scale": ad["scale"], "A": [ad["A"][0]], "B": [ad["B"][0][:, :6]]} for a, ad in ads.items()}
    Wr = _int_mat(rng, (d_in, 6))
    y = ol.row_layer(X, Wr, rads, ids, "nfs", n)
    acc_ = np.zeros_like(y)
    for i in range(n):
        ref = _bf_nfs_row_partial(X.tolist(), Wr.tolist(), rads, ids.tolist(), n, i)
        assert np.array_equal(ol.row_partial_nfs(X, Wr, rads, ids, n, i), ref)
        acc_ += ref
    assert np.array_equal(acc_, y)


# ----------------------------------------------------------------------------- downward-compatible BD

@pytest.mark.parametrize("nh,nl", [(4, 2), (4, 1), (8, 2)])
def test_downward_compatible_bd_bruteforce(nh, nl):
    """An adapter trained for N_h devices served on N_l | N_h devices: device i of N_l runs the N_h-layout
    devices i*m..(i+1)*m-1 ("stacking the computations of different devices").  Column: its
    output block is the concatenation (per slice) of those devices' pure-Python Alg. 2 outputs; row: its
    partial is the sum of their Alg. 1 partials; both exactly on integers."""
    rng = np.random.default_rng(60 + nh + nl)
    m = nh // nl
    d_out, ads = _tiny_bd(rng, "column", nh, d_in=8, d_out=(8, 16), r=8)
    T, d_in = 5, 8
    X = _int_mat(rng, (T, d_in))
    W = _int_mat(rng, (d_in, sum(d_out)))
    ids = np.array([0, 2, -1, 1, 0], dtype=np.int32)
    full = ol.column_layer(X, W, d_out, ads, ids, "bd", nh)
    for i in range(nl):
        got = ol.column_device_output(full, nl, i)
        parts, c0 = [], 0
        for j, dj in enumerate(d_out):   # slice j of device i = the slice-j blocks of its m N_h-devices
            for d in range(i * m, (i + 1) * m):
                dev = _bf_column_device(X.tolist(), W.tolist(), d_out, ads, ids.tolist(), nh, d)
                off = sum(dk // nh for dk in d_out[:j])
                parts.append(dev[:, off:off + dj // nh])
        assert np.array_equal(got, np.concatenate(parts, axis=1))
    d_out_r, rads = _tiny_bd(rng, "row", nh, d_in=16, d_out=(6,), r=8)
    Xr = _int_mat(rng, (T, 16))
    Wr = _int_mat(rng, (16, 6))
    y = ol.row_layer(Xr, Wr, rads, ids, "bd", nh)
    acc_ = np.zeros_like(y)
    for i in range(nl):
        ref = sum(_bf_row_partial(Xr.tolist(), Wr.tolist(), rads, ids.tolist(), nh, d) for d in range(i * m, (i + 1) * m))
        got = ol.row_partial_bd_blocks(Xr, Wr, rads, ids, nh, nl, i)
        assert np.array_equal(got, ref)
        acc_ += got
    assert np.array_equal(acc_, y)


# ----------------------------------------------------------------------------- P3 / P4 / P5

def test_n1_bd_is_plain_lora():
    """P3 (rank r/N per shard): with N = 1 the BD expansion is the identity and BD = plain LoRA."""
    rng = np.random.default_rng(4)
    d_in, d_out, r = 16, (24,), 4
    A = rng.standard_normal((d_in, r))
    B = rng.standard_normal((r, d_out[0]))
    ads = {0: {"rank": r, "scale": 3.0, "A": [A], "B": [B]}}
    X = rng.standard_normal((5, d_in))
    W = rng.standard_normal((d_in, d_out[0]))
    ids = np.zeros(5, np.int32)
    bd = ol.column_layer(X, W, d_out, ads, ids, "bd", 1)[0]
    plain = X @ W + 3.0 * (X @ A @ B)
    assert np.allclose(bd, plain, rtol=1e-12, atol=1e-12)
    row = ol.row_layer(X, W, ads, ids, "bd", 1)
    assert np.allclose(row, plain, rtol=1e-12, atol=1e-12)


def test_slora_dense_is_plain_lora():
    """P4: S-LoRA shards dense factors; unsharded it is plain LoRA for any N."""
    rng = np.random.default_rng(5)
    d_in, d_out, r = 16, (8, 8), 8
    ads = {a: {"rank": r, "scale": 0.25 * (a + 1), "A": [rng.standard_normal((d_in, r)) for _ in d_out],
               "B": [rng.standard_normal((r, dj)) for dj in d_out]} for a in range(2)}
    X = rng.standard_normal((4, d_in))
    W = rng.standard_normal((d_in, 16))
    ids = np.array([1, 0, -1, 1])
    outs = ol.column_layer(X, W, d_out, ads, ids, "slora", 4)
    for j in range(2):
        ref = X @ W[:, 8 * j:8 * j + 8]
        for t, a in enumerate(ids):
            if a >= 0:
                ref[t] += ads[a]["scale"] * X[t] @ ads[a]["A"][j] @ ads[a]["B"][j]
        assert np.allclose(outs[j], ref, rtol=1e-12, atol=1e-12)


def _bf_slora_col_shard_v(X, A, s, ids_t, n, i):
    """Pure-Python matmul_3 on device i: v^i = s x_t A[:, i*r/N:(i+1)*r/N] -- its rank chunk."""
    d_in, r = len(A), len(A[0])
    rb = r // n
    return [s * sum(X[ids_t][d] * A[d][i * rb + k] for d in range(d_in)) for k in range(rb)]


def _bf_slora_row_shard_v(X, A, s, t, n, i):
    """Pure-Python matmul_5 on device i: v^i = s x_t[rows i] A[rows i, :] -- a full-rank partial."""
    d_in, r = len(A), len(A[0])
    bi = d_in // n
    return [s * sum(X[t][d] * A[d][k] for d in range(i * bi, (i + 1) * bi)) for k in range(r)]


@pytest.mark.parametrize("n", [1, 2, 4])
def test_slora_column_gathered_v_bruteforce(n):
    """The S-LoRA column payload after the all-gather: the concatenation, in rank order,
    of every device's matmul_3 rank chunk equals the oracle's s x_t A_j (full rank), exactly on integers."""
    rng = np.random.default_rng(40 + n)
    d_in, d_out, r = 8, (8, 4), 8
    ads = {a: {"rank": r, "scale": (2.0, -0.5, 1.0)[a], "A": [_int_mat(rng, (d_in, r)) for _ in d_out],
               "B": [_int_mat(rng, (r, dj)) for dj in d_out]} for a in range(3)}
    X = _int_mat(rng, (5, d_in))
    ids = np.array([2, 0, -1, 2, 1])
    Xl = X.tolist()
    for j in range(len(d_out)):
        got = ol.slora_column_gathered_v(X, ads, ids, j)
        assert sorted(got) == [0, 1, 3, 4]  # no entry for id -1
        for t, vec in got.items():
            a = int(ids[t])
            ref = []
            for i in range(n):
                ref += _bf_slora_col_shard_v(Xl, ads[a]["A"][j].tolist(), ads[a]["scale"], t, n, i)
            assert vec.tolist() == ref, (n, j, t)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_slora_row_reduced_v_bruteforce(n):
    """The S-LoRA row payload after the all-reduce: the sum over devices of the matmul_5
    partials (row block i of x_t and of A) equals the oracle's s x_t A (full input, full rank), exactly."""
    rng = np.random.default_rng(50 + n)
    d_in, r = 8, 4
    ads = {a: {"rank": r, "scale": (0.25, 3.0)[a], "A": [_int_mat(rng, (d_in, r))], "B": [_int_mat(rng, (r, 6))]}
           for a in range(2)}
    X = _int_mat(rng, (4, d_in))
    ids = np.array([1, -1, 0, 1])
    got = ol.slora_row_reduced_v(X, ads, ids)
    assert sorted(got) == [0, 2, 3]
    for t, vec in got.items():
        a = int(ids[t])
        ref = [0.0] * r
        for i in range(n):
            part = _bf_slora_row_shard_v(X.tolist(), ads[a]["A"][0].tolist(), ads[a]["scale"], t, n, i)
            ref = [x + y for x, y in zip(ref, part)]
        assert vec.tolist() == ref, (n, t)
    # and the expand that follows reproduces the S-LoRA row layer (R12: v replicated, B column-sharded)
    W = _int_mat(rng, (d_in, 6))
    y = ol.row_layer(X, W, ads, ids, "slora", n)
    for t in range(4):
        ref = X[t] @ W
        if ids[t] >= 0:
            ref = ref + got[t] @ ads[int(ids[t])]["B"][0]
        assert np.array_equal(y[t], ref)


@pytest.mark.parametrize("which", ["A", "B"])
def test_zero_adapter_is_base(which):
    """P5: a zero adapter leaves y = XW exactly (bitwise)."""
    rng = np.random.default_rng(6)
    proj = synth.Projection("p", "column", 64, (32, 32))
    ad = synth.make_adapter(rng, proj, "bd", 8, 2, 2.0, zero=which)
    ads = {0: {"rank": 8, "scale": 2.0, "A": [a.f64 for a in ad.A], "B": [b.f64 for b in ad.B]}}
    X = synth.make_x(rng, 6, 64).f64
    W = synth.make_base(rng, proj).f64
    ids = np.zeros(6, np.int32)
    outs = ol.column_layer(X, W, proj.d_out, ads, ids, "bd", 2)
    assert np.array_equal(np.concatenate(outs, axis=1), X @ W)


def test_dual_oracle_materialised_vs_factored():
    """materialised x (A B) vs factored (x A) B agree to 1e-9 relative."""
    rng = np.random.default_rng(7)
    d_in, d_out, r = 128, 96, 16
    ads = {a: (1.3, rng.standard_normal((d_in, r)), rng.standard_normal((r, d_out))) for a in range(3)}
    X = rng.standard_normal((10, d_in))
    W = rng.standard_normal((d_in, d_out))
    ids = rng.integers(-1, 3, size=10)
    m = ol.lora_layer(X, W, ads, ids, materialise=True)
    f = ol.lora_layer(X, W, ads, ids, materialise=False)
    assert np.max(np.abs(m - f)) <= 1e-9 * np.max(np.abs(f))


def test_sampled_matches_full():
    rng = np.random.default_rng(8)
    d_in, d_out, r = 64, 48, 8
    ads = {a: (0.7, rng.standard_normal((d_in, r)), rng.standard_normal((r, d_out))) for a in range(2)}
    X = rng.standard_normal((6, d_in))
    W = rng.standard_normal((d_in, d_out))
    ids = np.array([0, 1, -1, 1, 0, 0])
    full = ol.lora_layer(X, W, ads, ids)
    samples = [(0, 0), (2, 47), (5, 13), (3, 30)]
    got = ol.lora_layer_sampled(X, W, ads, ids, samples)
    for k, (t, c) in enumerate(samples):
        assert abs(got[k] - full[t, c]) <= 1e-12 * max(1.0, abs(full[t, c]))


# ----------------------------------------------------------------------------- P6 / P7 / P8 / P9

def _printed(count: int) -> str:
    q = decimal.Decimal(count) / decimal.Decimal(1_000_000)
    return str(q.quantize(decimal.Decimal("0.1"), rounding=decimal.ROUND_HALF_UP)) + "M"


def test_param_counts_match_paper_tables():
    """P6: every '# Trainable Parameters' value checked (tests/golden/param_counts.json, lines cited)."""
    with open(os.path.join(GOLDEN, "param_counts.json")) as f:
        g = json.load(f)
    for arch, method, n, r, printed, line in g["entries"]:
        got = acc.count_params(arch, method, r, n)
        assert _printed(got) == printed, (arch, method, n, r, line, got)


def test_param_counts_exact_spec_values():
    # SPEC S:423-425 exact integers (derived from the paper's per-projection rule)
    assert acc.count_params("llama-3.1-8b", "dense", 16) == 41_943_040
    assert acc.count_params("llama-3.1-8b", "bd", 32, 8) == 36_175_872
    assert acc.count_params("llama-3.1-70b", "dense", 16) == 207_093_760
    assert acc.count_params("llama-3.1-70b", "bd", 32, 8) == 180_224_000


def _ratio2(x: Fraction) -> str:
    q = decimal.Decimal(x.numerator) / decimal.Decimal(x.denominator)
    return str(q.quantize(decimal.Decimal("0.01"), rounding=decimal.ROUND_HALF_UP))


def test_parameter_ratios_printed_in_captions():
    """'0.86x / 1.73x' (8B), '0.87x / 1.74x' (70B), '0.51 / 1.03x' (8B TP4)."""
    c = acc.count_params
    assert _ratio2(Fraction(c("llama-3.1-8b", "bd", 32, 8), c("llama-3.1-8b", "dense", 16))) == "0.86"
    assert _ratio2(Fraction(c("llama-3.1-8b", "bd", 64, 8), c("llama-3.1-8b", "dense", 16))) == "1.73"
    assert _ratio2(Fraction(c("llama-3.1-70b", "bd", 32, 8), c("llama-3.1-70b", "dense", 16))) == "0.87"
    assert _ratio2(Fraction(c("llama-3.1-70b", "bd", 64, 8), c("llama-3.1-70b", "dense", 16))) == "1.74"
    assert _ratio2(Fraction(c("llama-3.1-8b", "bd", 32, 4), c("llama-3.1-8b", "dense", 32))) == "0.51"
    assert _ratio2(Fraction(c("llama-3.1-8b", "bd", 64, 4), c("llama-3.1-8b", "dense", 32))) == "1.03"


def test_bd_requires_divisibility():
    with pytest.raises(ValueError):
        acc.params_bd_column(16, 16, 6, 4)


def test_scales():
    """P7: rsLoRA alpha=16, r=256 -> 1.0; BD alpha=16, r=64, N=4 -> 4.0."""
    assert acc.scale_rslora(16, 256) == 1.0
    assert acc.scale_bd_rslora(16, 64, 4) == 4.0
    assert acc.scale_standard(16, 16) == 1.0
    # BD scale equals rsLoRA evaluated at rank r/N (independent rank-r/N adapters)
    for r, n in [(32, 8), (64, 2), (512, 8)]:
        assert math.isclose(acc.scale_bd_rslora(16, r, n), acc.scale_rslora(16, r // n), rel_tol=1e-15)


def test_slora_comm_volume():
    """P8: 5(N-1)rS/N = 71,680 at N=8, r=16, S=1024; ratio to base 5r/(2 d_H) > 15% at r=256."""
    assert acc.slora_attn_comm_elems(8, 16, 1024) == 71_680
    ratio = acc.slora_attn_comm_elems(8, 256, 1024) / acc.base_attn_comm_elems(8, 4096, 1024)
    assert ratio == Fraction(5 * 256, 2 * 4096) and float(ratio) > 0.15
    assert acc.slora_attn_comm_elems(1, 16, 1024) == 0


def test_match_rank_and_flop_identity():
    """P9: r' = r (d_H+d_I)/(d_H+d_I/N); S-LoRA and BD FLOPs equal at r'."""
    rp = acc.match_rank(4096, 14336, 8, 16)
    assert rp == Fraction(1152, 23) == Fraction(294912, 5888)
    assert acc.match_rank(512, 512, 1, 16) == 16
    assert (acc.mlp_lora_flops_per_device(1024, 4096, 14336, 8, 16, "slora")
            == acc.mlp_lora_flops_per_device(1024, 4096, 14336, 8, rp, "bd"))
    assert 1 < rp < 16 * (1 + Fraction(14336, 4096))  # bound stated at P:977-979


def test_collective_table():
    """Fig. 2 / Fig. 3: S-LoRA 1 AG + 1 AR per module (merged), BD and NFS zero."""
    assert acc.lora_collectives("bd", "attn") == {"all_gather": 0, "all_reduce": 0}
    assert acc.lora_collectives("nfs", "glu") == {"all_gather": 0, "all_reduce": 0}
    assert acc.lora_collectives("slora", "attn", merged=False) == {"all_gather": 3, "all_reduce": 1}
    assert acc.lora_collectives("slora", "glu", merged=False) == {"all_gather": 2, "all_reduce": 1}
    assert acc.lora_collectives("slora", "mlp") == {"all_gather": 1, "all_reduce": 1}


# ----------------------------------------------------------------------------- P11

def test_segments_golden():
    with open(os.path.join(GOLDEN, "segments.json")) as f:
        g = json.load(f)
    for case in g["cases"]:
        assert [list(s) for s in ol.segments(case["ids"])] == case["segments"]


def test_segments_bruteforce_random():
    rng = np.random.default_rng(11)
    for _ in range(50):
        ids = rng.integers(-1, 4, size=int(rng.integers(0, 40))).tolist()
        segs = ol.segments(ids)
        # reassembles the stream, runs are maximal, lengths positive
        flat = [sid for (s, l, sid) in segs for _ in range(l)]
        assert flat == ids
        for k in range(1, len(segs)):
            assert segs[k][2] != segs[k - 1][2]
            assert segs[k][0] == segs[k - 1][0] + segs[k - 1][1]


# ----------------------------------------------------------------------------- comparison rule

def test_within_tolerance_rejects_plausible_mistakes():
    rng = np.random.default_rng(12)
    ref = rng.standard_normal((16, 64))
    ok, _, _ = ol.within_tolerance(ref * (1 + 1e-3), ref)
    assert ok
    assert not ol.within_tolerance(-ref, ref)[0]                 # sign error
    bad = ref.copy(); bad[:, :8] = 0.0
    assert not ol.within_tolerance(bad, ref)[0]                  # dropped block
    assert not ol.within_tolerance(ref[::-1], ref)[0]            # permuted tokens


def test_bf16_round_matches_synth():
    rng = np.random.default_rng(13)
    x = rng.integers(-600, 600, size=1000).astype(np.float64)
    a = ol.bf16_round(x)
    b = synth.bf16_bits_to_f64(synth.f32_to_bf16_bits(x.astype(np.float32)))
    assert np.array_equal(a, b)
    assert ol.bf16_round(np.array([257.0]))[0] == 256.0   # tie -> even
    assert ol.bf16_round(np.array([259.0]))[0] == 260.0


def test_synth_bf16_rne():
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1.0); 1 + 3*2^-9 rounds up
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5], dtype=np.float32)
    b = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(x))
    assert b[0] == 1.0 and b[1] == np.float32(1.0 + 2 ** -7) and b[2] == -2.5
