"""GPU parity of the lean decode kernel (kernels_decode.cuh, bdlora_last_launch_info kind 3) against the fp64
oracle: every T <= 16 forward whose batch fits the kernel's K-local LoRA capacity (BD / NFS pools), and the
v-precomputed mode behind bdlora_base_expand (S-LoRA's expand after its collective).  Covers whole tiles,
split-K tiles finished by the last contributor, stream-K grids over tiles of different slices, tiles that
straddle a slice boundary, ragged M, several adapters in one batch, id -1 tokens, and exact integer mode."""
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


def _assert_tol(y, ref, what):
    ok, m, l1 = ol.within_tolerance(y, ref)
    assert ok, f"{what}: max-rel {m:.3e} (<=2e-2), l1-rel {l1:.3e} (<=5e-3)"


def _run(case, i, dev, expect_kind=3):
    import torch

    import paper_2510_23346_b200 as bd

    pool = H.make_pool(case, i)
    X, W, ids = H.device_inputs(case, i, dev)
    T = X.shape[0]
    Y = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    col = case.proj.parallel == "column"
    if case.sharding == "nfs":
        (bd.nfs_column_forward if col else bd.nfs_row_partial)(pool, X, W, ids, Y, ws)
    else:
        (bd.bdlora_column_forward if col else bd.bdlora_row_partial)(pool, X, W, ids, Y, ws)
    info = bd.bdlora_last_launch_info()
    torch.cuda.synchronize()
    pool.close()
    if expect_kind is not None:
        assert info["kind"] == expect_kind, info
    return _np(Y), info


def _ref(case, i):
    ads = case.oracle_adapters()
    if case.proj.parallel == "column":
        full = ol.column_layer(case.X.f64, case.W.f64, case.proj.d_out, ads, case.ids, case.sharding, case.n)
        return ol.column_device_output(full, case.n, i)
    if case.sharding == "nfs":
        return ol.row_partial_nfs(case.X.f64, case.W.f64, ads, case.ids, case.n, i)
    return ol.row_partial_bd(case.X.f64, case.W.f64, ads, case.ids, case.n, i)


P8 = synth.arch_projections("llama-3.1-8b")
P70 = synth.arch_projections("llama-3.1-70b")


@pytest.mark.parametrize("pi", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_decode_8b_bs1_every_projection(dev, pi, n):
    """configs[1]: 8B, T = 1, one rank-16 adapter, every projection, first and last tp_rank."""
    proj = P8[pi]
    case = H.make_case(5000 + 10 * pi + n, proj, "bd", n, 1, ranks=[16], ids=np.zeros(1, np.int32))
    for i in sorted({0, n - 1}):
        y, info = _run(case, i, dev)
        _assert_tol(y, _ref(case, i), f"{proj.name} N={n} rank {i} grid {info['grid']}")


@pytest.mark.parametrize("pi", [0, 1, 3])
def test_decode_70b_bs1_tp8(dev, pi):
    """configs[3] at batch 1: 70B, rank 32 (r/N = 4), TP = 8."""
    proj = P70[pi]
    case = H.make_case(5100 + pi, proj, "bd", 8, 1, ranks=[32], ids=np.zeros(1, np.int32))
    y, _ = _run(case, 5, dev)
    _assert_tol(y, _ref(case, 5), f"70B {proj.name}")


@pytest.mark.parametrize("T,ranks,cap_ids", [(16, [16], "one"), (4, [8, 8, 8, 8], "mixed"), (2, [16, 16], "mixed"),
                                             (16, [32], "none_and_one"), (7, [8, 16], "mixed")])
@pytest.mark.parametrize("n", [1, 4])
def test_decode_multi_token_multi_adapter(dev, T, ranks, cap_ids, n):
    """Up to 16 tokens, several adapters and id -1 tokens in one batch (K-local capacity: at most 32 local rank
    rows over the batch's distinct adapters), 8B QKV (3 slices) and down (row)."""
    rng = synth.rng_for(5200 + T + n, 1)
    if cap_ids == "one":
        ids = np.zeros(T, np.int32)
    elif cap_ids == "none_and_one":
        ids = np.where(rng.random(T) < 0.3, -1, 0).astype(np.int32)
    else:
        ids = synth.ids_runs(rng, T, len(ranks), p_none=0.15, mean_run=1.5)
    for proj in (P8[0], P8[3]):
        case = H.make_case(5200 + T + n, proj, "bd", n, T, ranks=ranks, ids=ids)
        rs_max = max(ranks) // n
        kind = 3 if min(T, len(ranks)) * rs_max <= 32 else None
        y, _ = _run(case, n - 1, dev, expect_kind=kind)
        _assert_tol(y, _ref(case, n - 1), f"{proj.name} T={T} ranks={ranks} N={n}")


def test_decode_slice_straddling_tiles(dev):
    """Slices narrower than a 128-row tile (q | k | v = 512 | 64 | 64 at N = 1 and 32-column k / v at N = 2):
    one tile holds rows of two or three slices, each with its own A_j, B_j."""
    proj = synth.Projection("qkv", "column", 1024, (512, 64, 64))
    for n in (1, 2):
        case = H.make_case(5300 + n, proj, "bd", n, 3, ranks=[8, 16], ids=np.array([1, 0, 1], np.int32))
        for i in range(n):
            y, _ = _run(case, i, dev)
            _assert_tol(y, _ref(case, i), f"straddle N={n} rank {i}")


def test_decode_ragged_m(dev):
    """M not a multiple of 128 (last tile partly outside W: TMA zero fill, rows skipped on store)."""
    proj = synth.Projection("odd", "column", 512, (200, 72))
    case = H.make_case(5400, proj, "bd", 1, 5, ranks=[8])
    y, _ = _run(case, 0, dev)
    _assert_tol(y, _ref(case, 0), "ragged M")


@pytest.mark.parametrize("n", [1, 8])
def test_decode_nfs(dev, n):
    """NFS-LoRA pools (A_1 / B_2 replicated, full local rank) through the K-local kernel."""
    for proj in (P8[0], P8[1]):
        case = H.make_case(5500 + n, proj, "nfs", n, 2, ranks=[16], ids=np.array([0, 0], np.int32))
        y, _ = _run(case, n - 1, dev)
        _assert_tol(y, _ref(case, n - 1), f"nfs {proj.name} N={n}")


@pytest.mark.parametrize("n", [1, 2, 8])
@pytest.mark.parametrize("T", [1, 5, 16])
def test_decode_integer_bit_exact(dev, n, T):
    """P10: integer inputs, s a power of two -- the K-local split (each contributor's v_seg B in its partial) and
    the deterministic fix-up are exact, so the output is bit-identical to the oracle rounded once."""
    for proj, ranks in ((synth.Projection("qkv", "column", 2048, (1024, 512, 512)), [8, 16]),
                        (synth.Projection("down", "row", 4096, (1024,)), [16, 8])):
        case = H.make_case(5600 + n + T, proj, "bd", n, T, ranks=ranks, integer=True)
        for i in sorted({0, n - 1}):
            y, _ = _run(case, i, dev)
            ref = ol.bf16_round(_ref(case, i))
            assert np.array_equal(y, ref), f"{proj.name} N={n} T={T} rank {i}: {np.count_nonzero(y != ref)} mismatches"


@pytest.mark.parametrize("T", [1, 12])
def test_decode_v_precomputed_mode(dev, T):
    """bdlora_base_expand at T <= 16 runs the decode kernel with v from the preceding shrink (S-LoRA's expand
    after its collective, emulated here at N = 2 by concatenating both ranks' shrink outputs)."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = P8[0]
    n = 2
    case = H.make_case(5700 + T, proj, "slora", n, T, ranks=[16, 32])
    pools = [H.make_pool(case, i) for i in range(n)]
    vs = []
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        v = torch.zeros(bd.bdlora_v_elems(p, T), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(p, X, ids, v, bd.make_workspace(p, T))
        vs.append(v)
    vg = torch.cat(vs)
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        Y = torch.empty(T, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_base_expand(p, X, W, ids, vg, Y, bd.make_workspace(p, T))
        assert bd.bdlora_last_launch_info()["kind"] == 3
        torch.cuda.synchronize()
        _assert_tol(_np(Y), _ref(case, i), f"slora v-mode rank {i}")
    for p in pools:
        p.close()


# ----------------------------------------------------------------------------- 17..64 tokens (BN = 64 tiles)
# configs[3] batch 64: one resident adapter per pool -> the decode kernel with 64-token tiles, the tensor-core
# K-local shrink (BD / NFS) or staged-B expand of a precomputed v (S-LoRA).

@pytest.mark.parametrize("T", [17, 40, 64])
@pytest.mark.parametrize("pi,n", [(0, 8), (1, 8), (2, 8), (3, 8), (0, 1), (3, 2)])
def test_decode_bn64_one_adapter(dev, T, pi, n):
    """70B shapes at TP = N, rank 32 (r/N <= 16 at N >= 2; N = 1 uses the 8B QKV with rank 16), ids 0 with
    some -1 tokens: every projection, first and last tp_rank, BN = 64 asserted."""
    rng = synth.rng_for(5800 + T + pi + n, 1)
    ids = np.where(rng.random(T) < 0.2, -1, 0).astype(np.int32)
    proj = P70[pi] if n > 1 else P8[pi]
    r = 32 if n > 1 else 16
    case = H.make_case(5800 + 10 * pi + n + T, proj, "bd", n, T, ranks=[r], ids=ids)
    for i in sorted({0, n - 1}):
        y, info = _run(case, i, dev)
        assert info["bn"] == 64, info
        _assert_tol(y, _ref(case, i), f"{proj.name} N={n} T={T} rank {i}")


@pytest.mark.parametrize("T", [33, 64])
def test_decode_bn64_integer_bit_exact(dev, T):
    """P10 at 64-token tiles: column (3 slices, 128-aligned) and row, N = 4, bit-identical to the oracle."""
    for proj in (synth.Projection("qkv", "column", 2048, (1024, 512, 512)), synth.Projection("down", "row", 4096, (1024,))):
        case = H.make_case(5900 + T, proj, "bd", 4, T, ranks=[32], integer=True, ids=np.zeros(T, np.int32))
        for i in (0, 3):
            y, info = _run(case, i, dev)
            assert info["bn"] == 64, info
            ref = ol.bf16_round(_ref(case, i))
            assert np.array_equal(y, ref), f"{proj.name} T={T} rank {i}: {np.count_nonzero(y != ref)} mismatches"


@pytest.mark.parametrize("T", [24, 64])
def test_decode_bn64_nfs_and_slora(dev, T):
    """NFS-LoRA (K-local) and S-LoRA (v precomputed, staged B) at 64-token tiles, one adapter per pool."""
    import torch

    import paper_2510_23346_b200 as bd

    ids = np.zeros(T, np.int32)
    case = H.make_case(5950 + T, P70[1], "nfs", 8, T, ranks=[16], ids=ids)
    y, info = _run(case, 7, dev)
    assert info["bn"] == 64
    _assert_tol(y, _ref(case, 7), "nfs row")
    proj = P70[0]
    n = 2
    case = H.make_case(5960 + T, proj, "slora", n, T, ranks=[16], ids=ids)
    pools = [H.make_pool(case, i) for i in range(n)]
    vs = []
    for i, p in enumerate(pools):
        X, W, idt = H.device_inputs(case, i, dev)
        v = torch.zeros(bd.bdlora_v_elems(p, T), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(p, X, idt, v, bd.make_workspace(p, T))
        vs.append(v)
    vg = torch.cat(vs)
    for i, p in enumerate(pools):
        X, W, idt = H.device_inputs(case, i, dev)
        Y = torch.empty(T, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_base_expand(p, X, W, idt, vg, Y, bd.make_workspace(p, T))
        info = bd.bdlora_last_launch_info()
        assert info["kind"] == 3 and info["bn"] == 64, info
        torch.cuda.synchronize()
        _assert_tol(_np(Y), _ref(case, i), f"slora v-mode T={T} rank {i}")
    for p in pools:
        p.close()


# ----------------------------------------------------------------------------- many adapters, T <= 64 (lora 4)
# configs[4]-shaped batches: more distinct adapters than the K-local capacity -> one grid-wide shrink launch
# (dec_shrink_kernel, every distinct adapter's A rows read once) + the decode kernel expanding the precomputed v
# in its epilogue, each split contributor taking a share of the tile's rank rows through 64-row B chunks.

MT_COL = synth.Projection("qkv_s", "column", 1024, (1024, 256, 256))
MT_ROW = synth.Projection("down_s", "row", 2048, (1024,))


def _mt_ids(seed, T, n_ad):
    rng = synth.rng_for(seed, 2)
    ids = rng.integers(0, n_ad, T).astype(np.int32)
    ids[rng.random(T) < 0.1] = -1
    return ids


@pytest.mark.parametrize("T", [3, 17, 64])
@pytest.mark.parametrize("proj,n", [(MT_COL, 1), (MT_COL, 2), (MT_ROW, 2), (MT_ROW, 8)])
def test_decode_multi_adapter_vs_oracle(dev, T, proj, n):
    """12 resident adapters of ranks 8..128 (mixed), uniform ids with -1 tokens: BN = 64 asserted, every rank of
    the batch's groups through the chunked expand, first and last tp_rank."""
    ranks = [[8, 16, 32, 64, 128][a % 5] for a in range(12)]
    case = H.make_case(6000 + T + 10 * n + len(proj.d_out), proj, "bd", n, T, ranks=ranks, ids=_mt_ids(6000 + T, T, 12))
    for i in sorted({0, n - 1}):
        y, info = _run(case, i, dev)
        assert info["bn"] == 64, info
        _assert_tol(y, _ref(case, i), f"{proj.name} N={n} T={T} rank {i} grid {info['grid']} cluster {info['cluster']}")


@pytest.mark.parametrize("T", [8, 64])
def test_decode_multi_adapter_many_chunks(dev, T):
    """24 adapters up to rank 128 at N = 4 (about 600 expand rows per tile: several 64-row B chunks per
    contributor), all distinct ids at T = 8 and uniform ids at T = 64."""
    proj = synth.Projection("qkv_m", "column", 4096, (2048, 512, 512))
    ranks = [[8, 16, 32, 64, 128][a % 5] for a in range(24)]
    ids = np.arange(T, dtype=np.int32) * 3 % 24 if T == 8 else _mt_ids(6100, T, 24)
    case = H.make_case(6100 + T, proj, "bd", 4, T, ranks=ranks, ids=ids)
    for i in (0, 3):
        y, info = _run(case, i, dev)
        assert info["bn"] == 64, info
        _assert_tol(y, _ref(case, i), f"many chunks T={T} rank {i}")


@pytest.mark.parametrize("T", [5, 64])
def test_decode_multi_adapter_integer_bit_exact(dev, T):
    """P10 through the multi-adapter path: integer inputs, power-of-two scales, per-adapter B signatures --
    routing, the shrink and the share-split expand are exact, so the output is bit-identical."""
    ranks = [8, 16, 32, 8, 16, 32, 64, 8, 16, 32]
    for proj, n in ((MT_COL, 2), (MT_ROW, 4)):
        case = H.make_case(6200 + T + n, proj, "bd", n, T, ranks=ranks, integer=True, ids=_mt_ids(6200 + T, T, 10))
        for i in sorted({0, n - 1}):
            y, info = _run(case, i, dev)
            assert info["bn"] == 64, info
            ref = ol.bf16_round(_ref(case, i))
            assert np.array_equal(y, ref), f"{proj.name} N={n} T={T} rank {i}: {np.count_nonzero(y != ref)} mismatches"


@pytest.mark.parametrize("T", [9, 48])
def test_decode_multi_adapter_slora_expand(dev, T):
    """S-LoRA column at N = 2 with 8 mixed-rank adapters: the grid-wide shrink writes each rank's v chunk, the
    all-gather is emulated by concatenation, bdlora_base_expand expands C = N chunks of v (lora 4)."""
    import torch

    import paper_2510_23346_b200 as bd

    n = 2
    ranks = [8, 16, 32, 64, 16, 8, 32, 64]
    case = H.make_case(6300 + T, MT_COL, "slora", n, T, ranks=ranks, ids=_mt_ids(6300 + T, T, 8))
    pools = [H.make_pool(case, i) for i in range(n)]
    vs = []
    for i, p in enumerate(pools):
        X, W, idt = H.device_inputs(case, i, dev)
        v = torch.zeros(bd.bdlora_v_elems(p, T), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(p, X, idt, v, bd.make_workspace(p, T))
        vs.append(v)
    vg = torch.cat(vs)
    for i, p in enumerate(pools):
        X, W, idt = H.device_inputs(case, i, dev)
        Y = torch.empty(T, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_base_expand(p, X, W, idt, vg, Y, bd.make_workspace(p, T))
        info = bd.bdlora_last_launch_info()
        assert info["kind"] == 3 and info["bn"] == 64, info
        torch.cuda.synchronize()
        _assert_tol(_np(Y), _ref(case, i), f"slora lora-4 T={T} rank {i}")
    for p in pools:
        p.close()


@pytest.mark.parametrize("T", [24, 64])
@pytest.mark.parametrize("integer", [False, True])
def test_decode_bn64_streamk_slices(dev, T, integer):
    """64-token tiles of a one-adapter pool on a stream-K grid (160 tiles > #SM: no cluster, CTAs owning parts of
    two tiles, one of them at the gate | up slice boundary): the tensor-core K-local shrink takes each stage's A
    box from its own tile's slice and double-buffers v_seg with the accumulator."""
    proj = synth.Projection("gu_wide", "column", 256, (10240, 10240))
    rng = synth.rng_for(6400 + T, 1)
    ids = np.where(rng.random(T) < 0.2, -1, 0).astype(np.int32)
    case = H.make_case(6400 + T + integer, proj, "bd", 1, T, ranks=[16], ids=ids, integer=integer)
    y, info = _run(case, 0, dev)
    assert info["bn"] == 64 and info["cluster"] == 1, info
    ref = _ref(case, 0)
    if integer:
        ref = ol.bf16_round(ref)
        assert np.array_equal(y, ref), f"T={T}: {np.count_nonzero(y != ref)} mismatches"
    else:
        _assert_tol(y, ref, f"stream-K bn64 T={T}")
