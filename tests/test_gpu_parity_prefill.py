"""GPU parity of the compute-bound token tiles (BN = 64 / 128 / 256) at configs[2] shapes -- Llama-3.1-8B
prefill S = 1024, ranks 8 and 256, one request (1 segment) and 8 requests x 128 tokens (8 segments) --
element by element against the fp64 oracle, on ONE emulated rank i of an N-way TP group.

Only device i's base-weight shard is generated.  The oracle is the plain definition of device i's
problem: the column layer Y_i = X W_i + s (X A_j[:, chunk i]) B_j^(i) is the N = 1 layer of its shard with
the rank-r/N adapter (A_j[:, chunk i], B_j^(i)) (Alg. 2 lines 3-6; pinned to the unsharded
layer by P2 in tests/test_oracle_pins.py), the row partial P_i = X_i W_i + s (X_i A_2^(i)) B_2^(i) likewise
(Alg. 1 lines 9-12).  Which token-tile width the library took is read back through
bdlora_last_launch_info and asserted, so every instantiation (<64,0>, <128,0>, <256,0>) is covered."""
import numpy as np
import pytest

import synth
from oracle import lora as ol
from tests import _harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch

    import paper_2510_23346_b200 as bd

    bd.bdlora_device_check(0)
    return torch.device("cuda", 0)


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _ids(kind, T, n_ad):
    if kind == "one":
        return np.zeros(T, np.int32)
    return synth.ids_segments(T, n_ad)


def _column_case(seed, proj, n, i, T, r, ids_kind, integer=False):
    """Full adapters (load format), device i's base columns only, X; plus device i's shard problem."""
    rng = synth.rng_for(seed, 21)
    n_ad = 1 if ids_kind == "one" else 8
    ads = {}
    for a in range(n_ad):
        if integer:
            ads[a] = synth.make_int_adapter(rng, proj, "bd", r, n, 2.0 ** (a % 3 - 1), signature=a)
        else:
            ads[a] = synth.make_adapter(rng, proj, "bd", r, n, synth.rs_scale(16.0, r, n, "bd"))
    if integer:
        X = synth.int_tensor(rng, (T, proj.d_in), 0.5)
        w_loc = [synth.int_tensor(rng, (proj.d_in, dj // n), 0.05) for dj in proj.d_out]
    else:
        X = synth.make_x(rng, T, proj.d_in)
        w_loc = [synth.bf16_normal(rng, (proj.d_in, dj // n), 1 / np.sqrt(proj.d_in)) for dj in proj.d_out]
    ids = _ids(ids_kind, T, n_ad)
    # device i's shard problem at N = 1: rank r/N adapter (A_j[:, chunk i], diagonal block i of B_j)
    rb = r // n
    shard_ads = {}
    for a, ad in ads.items():
        As = [x.f64[:, i * rb:(i + 1) * rb] for x in ad.A]
        Bs = [x.f64[:, i * (dj // n):(i + 1) * (dj // n)] for x, dj in zip(ad.B, proj.d_out)]
        shard_ads[a] = {"rank": rb, "scale": ad.scale, "A": As, "B": Bs}
    W_loc = np.concatenate([w.f64 for w in w_loc], axis=1)
    ref = np.concatenate(ol.column_layer(X.f64, W_loc, [dj // n for dj in proj.d_out], shard_ads, ids, "bd", 1), axis=1)
    return ads, X, w_loc, ids, ref


def _run_column(dev, proj, n, i, r, ads, X, w_loc, ids):
    import torch

    import paper_2510_23346_b200 as bd

    pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, n, i, proj.d_in, proj.d_out, len(ads), r, device=0)
    for a, ad in ads.items():
        bd.bdlora_load_adapter(pool, a, ad.rank, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                               [H.torch_bf16(x.bits) for x in ad.B])
    Wt = H.torch_bf16(np.ascontiguousarray(np.concatenate([w.bits for w in w_loc], axis=1).T), dev)
    T = X.shape[0]
    Y = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    bd.bdlora_column_forward(pool, H.torch_bf16(X.bits, dev), Wt, torch.from_numpy(ids).to(dev), Y,
                             bd.make_workspace(pool, T))
    info = bd.bdlora_last_launch_info()
    torch.cuda.synchronize()
    pool.close()
    return _np(Y), info


def _assert_tol(y, ref, what):
    ok, m, l1 = ol.within_tolerance(y, ref)
    assert ok, f"{what}: max-rel {m:.3e} (<=2e-2), l1-rel {l1:.3e} (<=5e-3)"


QKV, O, GATE_UP, DOWN = synth.arch_projections("llama-3.1-8b")


@pytest.mark.parametrize("r", [8, 256])
@pytest.mark.parametrize("ids_kind", ["one", "8seg"])
@pytest.mark.parametrize("name,proj,n,bn", [("gate_up_tp8", GATE_UP, 8, 256), ("qkv_tp4", QKV, 4, 128),
                                            ("qkv_tp8", QKV, 8, 64)])
def test_prefill_column_tiles(dev, name, proj, n, bn, r, ids_kind):
    """configs[2] column projections at S = 1024: the chosen token tile (asserted) against the oracle."""
    i = n - 1
    ads, X, w_loc, ids, ref = _column_case(3000 + n + r, proj, n, i, 1024, r, ids_kind)
    y, info = _run_column(dev, proj, n, i, r, ads, X, w_loc, ids)
    assert info["kind"] == 0 and info["bn"] == bn, info
    _assert_tol(y, ref, f"{name} r={r} {ids_kind}")


@pytest.mark.parametrize("r", [8, 256])
@pytest.mark.parametrize("ids_kind", ["one", "8seg"])
@pytest.mark.parametrize("name,proj,n", [("o_tp8", O, 8), ("down_tp8", DOWN, 8)])
def test_prefill_row_tiles(dev, name, proj, n, r, ids_kind):
    """configs[2] row projections at S = 1024 (BN = 256): device i's partial against the oracle's."""
    import torch

    import paper_2510_23346_b200 as bd

    i = 2
    T = 1024
    rng = synth.rng_for(3100 + r, 22)
    n_ad = 1 if ids_kind == "one" else 8
    ads = {a: synth.make_adapter(rng, proj, "bd", r, n, synth.rs_scale(16.0, r, n, "bd")) for a in range(n_ad)}
    kl = proj.d_in // n
    Xi = synth.make_x(rng, T, kl)
    Wi = synth.bf16_normal(rng, (kl, proj.d_out[0]), 1 / np.sqrt(proj.d_in))
    ids = _ids(ids_kind, T, n_ad)
    rb = r // n
    shard = {a: {"rank": rb, "scale": ad.scale, "A": [ad.A[0].f64[i * kl:(i + 1) * kl, :]],
                 "B": [ad.B[0].f64[i * rb:(i + 1) * rb, :]]} for a, ad in ads.items()}
    ref = ol.row_layer(Xi.f64, Wi.f64, shard, ids, "bd", 1)
    pool = bd.bdlora_create_pool(bd.ROW, bd.SHARD_BD, n, i, proj.d_in, proj.d_out, n_ad, r, device=0)
    for a, ad in ads.items():
        bd.bdlora_load_adapter(pool, a, ad.rank, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                               [H.torch_bf16(x.bits) for x in ad.B])
    P = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    bd.bdlora_row_partial(pool, H.torch_bf16(Xi.bits, dev), H.torch_bf16(np.ascontiguousarray(Wi.bits.T), dev),
                          torch.from_numpy(ids).to(dev), P, bd.make_workspace(pool, T))
    info = bd.bdlora_last_launch_info()
    torch.cuda.synchronize()
    pool.close()
    assert info["kind"] == 0 and info["bn"] == 256, info
    _assert_tol(_np(P), ref, f"{name} r={r} {ids_kind}")


def test_prefill_tp1_qkv_full(dev):
    """TP = 1 QKV at S = 1024 (BN = 128: 48 row tiles x 8 token tiles = 384 whole tiles), r = 64, 8 segments."""
    ads, X, w_loc, ids, ref = _column_case(3200, QKV, 1, 0, 1024, 64, "8seg")
    y, info = _run_column(dev, QKV, 1, 0, 64, ads, X, w_loc, ids)
    assert info["bn"] == 128, info
    _assert_tol(y, ref, "qkv tp1")


@pytest.mark.parametrize("T,bn", [(1024, 256), (520, 128)])
def test_prefill_integer_bit_exact(dev, T, bn):
    """P10 on the wide token tiles: M_loc = 3584 (28 row tiles), K = 1024, 8 segments over 8 integer
    adapters (B signatures) -- the GPU output is bit-identical to the oracle rounded once to bf16
    (T = 520: ragged token tail)."""
    proj = synth.Projection("gate_up", "column", 1024, (3584, 3584))
    n, i = 2, 1
    ads, X, w_loc, ids, ref = _column_case(3300 + T, proj, n, i, T, 16, "8seg", integer=True)
    y, info = _run_column(dev, proj, n, i, 16, ads, X, w_loc, ids)
    assert info["bn"] == bn, info
    refb = ol.bf16_round(ref)
    assert np.array_equal(y, refb), f"{np.count_nonzero(y != refb)} mismatches"
