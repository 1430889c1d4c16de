"""GPU parity of the C-ABI path against the fp64 oracle (SURVEY §8(c) step 7 tolerance:
max|y - y_ref| <= 2e-2 max|y_ref| and sum|y - y_ref| / sum|y_ref| <= 5e-3), element by element on
seeded inputs.  TP degrees are emulated on one GPU: every tp_rank's device-local call runs on
cuda:0 and is compared with the oracle's block for that rank (column) or the oracle's per-rank
partial and their sum (row).  The S-LoRA collectives are emulated in the test through the
phase entry points (bdlora_lora_shrink / bdlora_base_expand); the NCCL path itself needs >1 GPU."""
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


def run_column(case: H.Case, i: int, dev, fwd="bd"):
    import torch

    import paper_2510_23346_b200 as bd

    pool = H.make_pool(case, i)
    X, W, ids = H.device_inputs(case, i, dev)
    T = X.shape[0]
    Y = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    (bd.nfs_column_forward if case.sharding == "nfs" else bd.bdlora_column_forward)(pool, X, W, ids, Y, ws)
    torch.cuda.synchronize()
    pool.close()
    return Y


def run_row_partial(case: H.Case, i: int, dev):
    import torch

    import paper_2510_23346_b200 as bd

    pool = H.make_pool(case, i)
    X, W, ids = H.device_inputs(case, i, dev)
    T = X.shape[0]
    P = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    (bd.nfs_row_partial if case.sharding == "nfs" else bd.bdlora_row_partial)(pool, X, W, ids, P, ws)
    torch.cuda.synchronize()
    pool.close()
    return P


# ----------------------------------------------------------------------------- a2: segments

@pytest.mark.parametrize("T", [0, 1, 2, 17, 1024, 1500, 5000])
def test_segments_bit_exact(dev, T):
    import torch

    import paper_2510_23346_b200 as bd

    rng = synth.rng_for(T, 1)
    ids = synth.ids_runs(rng, T, 5, p_none=0.2, mean_run=3.0) if T else np.zeros(0, np.int32)
    ss, sl, si, n = bd.bdlora_build_segments(torch.from_numpy(ids).to(dev))
    torch.cuda.synchronize()
    n = int(n.item())
    got = list(zip(ss[:n].tolist(), sl[:n].tolist(), si[:n].tolist()))
    assert got == ol.segments(ids.tolist())


# ----------------------------------------------------------------------------- column BD

@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("T", [1, 3, 37])
def test_column_bd_8b_qkv(dev, n, T):
    """8B QKV shapes (4096 -> 4096|1024|1024), r=16, mixed ids with -1, every tp_rank."""
    proj = synth.arch_projections("llama-3.1-8b")[0]
    case = H.make_case(100 + n * 10 + T, proj, "bd", n, T, ranks=[16, 16, 32])
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", n)
    for i in range(n):
        Y = run_column(case, i, dev)
        _assert_tol(_np(Y), ol.column_device_output(ref_full, n, i), f"N={n} rank {i} T={T}")


def test_column_bd_tiny_config0(dev):
    """configs[0]: tiny column 256 -> 512, r=8, 4 adapters, 16 tokens mixed ids, TP=2."""
    proj = synth.tiny_pair()[0]
    ids = np.array([0, 0, 1, 1, 1, 2, 3, 3, 0, 2, 2, 1, 3, 3, 3, 0], np.int32)
    case = H.make_case(5, proj, "bd", 2, 16, ranks=[8, 8, 8, 8], ids=ids)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 2)
    for i in range(2):
        _assert_tol(_np(run_column(case, i, dev)), ol.column_device_output(ref_full, 2, i), f"rank {i}")


@pytest.mark.parametrize("which", ["W0", "A0"])
def test_column_lora_and_base_isolated(dev, which):
    """Step 7 (ii) W = 0 isolates the LoRA path; (iii) A = 0 the base path."""
    proj = synth.arch_projections("llama-3.1-8b")[2]  # gate_up
    n, T = 4, 9
    if which == "W0":
        case = H.make_case(31, proj, "bd", n, T, ranks=[16, 32], w_zero=True)
    else:
        case = H.make_case(32, proj, "bd", n, T, ranks=[16, 32], zero={0: "A", 1: "A"})
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", n)
    for i in range(n):
        _assert_tol(_np(run_column(case, i, dev)), ol.column_device_output(ref_full, n, i), f"{which} rank {i}")


def test_zero_adapter_bit_identical_to_base(dev):
    """P5: a B = 0 adapter gives output bit-identical to the no-adapter (id -1) output."""
    import torch

    proj = synth.arch_projections("llama-3.1-8b")[0]
    T = 8
    case = H.make_case(41, proj, "bd", 2, T, ranks=[16], ids=np.zeros(T, np.int32), zero={0: "B"})
    y0 = run_column(case, 1, dev)
    case.ids = -np.ones(T, np.int32)
    y1 = run_column(case, 1, dev)
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))


# ----------------------------------------------------------------------------- row BD

@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("T", [1, 37])
def test_row_bd_8b_down(dev, n, T):
    """8B down (14336 -> 4096): per-rank partials vs the oracle's Alg. 1 partial, and their sum
    (the all-reduce, emulated) vs the unsharded oracle."""
    proj = synth.arch_projections("llama-3.1-8b")[3]
    case = H.make_case(200 + n * 10 + T, proj, "bd", n, T, ranks=[16, 32, 16])
    ads = case.oracle_adapters()
    acc = None
    for i in range(n):
        P = run_row_partial(case, i, dev)
        _assert_tol(_np(P), ol.row_partial_bd(case.X.f64, case.W.f64, ads, case.ids, n, i), f"N={n} partial {i}")
        acc = _np(P) if acc is None else acc + _np(P)
    _assert_tol(acc, ol.row_layer(case.X.f64, case.W.f64, ads, case.ids, "bd", n), f"N={n} sum")


def test_row_forward_n1_no_comm(dev):
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.tiny_pair()[1]
    case = H.make_case(51, proj, "bd", 1, 16, ranks=[8, 8])
    pool = H.make_pool(case, 0)
    X, W, ids = H.device_inputs(case, 0, dev)
    Y = torch.empty(16, pool.m_loc, dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, 16)
    bd.bdlora_row_forward(pool, None, X, W, ids, Y, ws)
    torch.cuda.synchronize()
    _assert_tol(_np(Y), ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "bd", 1), "row N=1")


# ----------------------------------------------------------------------------- S-LoRA (phases)

def _slora_column_emulated(case: H.Case, dev):
    """Every rank: shrink -> (all-gather emulated by concatenating the ranks' v) -> base+expand."""
    import torch

    import paper_2510_23346_b200 as bd

    n = case.n
    T = len(case.ids)
    pools = [H.make_pool(case, i) for i in range(n)]
    vs = []
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        v = torch.zeros(bd.bdlora_v_elems(p, T), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(p, X, ids, v, bd.make_workspace(p, T))
        vs.append(v)
    vg = torch.cat(vs)  # [N][T][J][Rc]
    outs = []
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        Y = torch.empty(T, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_base_expand(p, X, W, ids, vg, Y, bd.make_workspace(p, T))
        outs.append(Y)
    torch.cuda.synchronize()
    for p in pools:
        p.close()
    return outs, vg


@pytest.mark.parametrize("n", [1, 2, 8])
def test_slora_column_8b_qkv(dev, n):
    proj = synth.arch_projections("llama-3.1-8b")[0]
    T = 13
    case = H.make_case(300 + n, proj, "slora", n, T, ranks=[16, 32, 16])
    ads = case.oracle_adapters()
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, ads, case.ids, "slora", n)
    outs, vg = _slora_column_emulated(case, dev)
    for i in range(n):
        _assert_tol(_np(outs[i]), ol.column_device_output(ref_full, n, i), f"slora col N={n} rank {i}")
    # the all-gathered intermediate equals X A (full rank) within fp32 accumulation (step 6)
    J, Rc = len(proj.d_out), case.max_rank // n
    v = vg.cpu().numpy().reshape(n, T, J, Rc)
    for j in range(J):
        refv = ol.slora_column_gathered_v(case.X.f64, ads, case.ids, j)
        for t, vec in refv.items():
            r = ads[int(case.ids[t])]["rank"]
            got = np.concatenate([v[c, t, j, :r // n] for c in range(n)])
            assert np.allclose(got, vec, rtol=1e-4, atol=1e-4 * np.abs(vec).max())


@pytest.mark.parametrize("n", [1, 2, 8])
def test_slora_row_8b_o(dev, n):
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[1]
    T = 11
    case = H.make_case(400 + n, proj, "slora", n, T, ranks=[16, 32])
    ads = case.oracle_adapters()
    pools = [H.make_pool(case, i) for i in range(n)]
    v = None
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        vi = torch.zeros(bd.bdlora_v_elems(p, T), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(p, X, ids, vi, bd.make_workspace(p, T))
        v = vi if v is None else v + vi  # all-reduce after matmul_5, emulated
    acc = None
    for i, p in enumerate(pools):
        X, W, ids = H.device_inputs(case, i, dev)
        P = torch.empty(T, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_base_expand(p, X, W, ids, v, P, bd.make_workspace(p, T))
        acc = P.float() if acc is None else acc + P.float()  # base all-reduce, emulated
    torch.cuda.synchronize()
    _assert_tol(acc.cpu().numpy(), ol.row_layer(case.X.f64, case.W.f64, ads, case.ids, "slora", n), f"slora row N={n}")
    for p in pools:
        p.close()


# ----------------------------------------------------------------------------- NFS-LoRA

@pytest.mark.parametrize("n", [1, 2, 8])
@pytest.mark.parametrize("T", [1, 5, 37])
def test_nfs_column_8b_qkv(dev, n, T):
    """NFS-LoRA column layer (A_1 replicated, B_1 column-sharded; no LoRA collective): every device's
    block vs the oracle.  Ranks not divisible by N are legal for NFS (12 at N = 8)."""
    proj = synth.arch_projections("llama-3.1-8b")[0]
    case = H.make_case(1100 + 10 * n + T, proj, "nfs", n, T, ranks=[16, 12, 8])
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "nfs", n)
    for i in sorted({0, n - 1}):
        _assert_tol(_np(run_column(case, i, dev)), ol.column_device_output(ref_full, n, i), f"N={n} rank {i}")


@pytest.mark.parametrize("n", [1, 2, 8])
@pytest.mark.parametrize("T", [1, 37])
def test_nfs_row_8b_o(dev, n, T):
    """NFS-LoRA row layer (A_2 row-sharded, B_2 replicated): per-rank partials vs the oracle's, and their
    sum (the base all-reduce, emulated) vs the unsharded layer."""
    proj = synth.arch_projections("llama-3.1-8b")[1]
    case = H.make_case(1200 + 10 * n + T, proj, "nfs", n, T, ranks=[16, 24])
    ads = case.oracle_adapters()
    acc = None
    for i in range(n):
        P = _np(run_row_partial(case, i, dev))
        _assert_tol(P, ol.row_partial_nfs(case.X.f64, case.W.f64, ads, case.ids, n, i), f"N={n} partial {i}")
        acc = P if acc is None else acc + P
    _assert_tol(acc, ol.row_layer(case.X.f64, case.W.f64, ads, case.ids, "nfs", n), f"N={n} sum")


@pytest.mark.parametrize("n", [1, 4])
@pytest.mark.parametrize("T", [9, 21])
def test_nfs_integer_mode_bit_exact(dev, n, T):
    """P10 for NFS-LoRA: column device blocks and row partials bit-identical to the oracle rounded once."""
    col = synth.Projection("qkv", "column", 1024, (512, 256, 256))
    case = H.make_case(1300 + n + T, col, "nfs", n, T, ranks=[8, 16, 8, 32], integer=True)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, col.d_out, case.oracle_adapters(), case.ids, "nfs", n)
    for i in range(n):
        got, ref = _np(run_column(case, i, dev)), ol.bf16_round(ol.column_device_output(ref_full, n, i))
        assert np.array_equal(got, ref), f"column rank {i}: {np.count_nonzero(got != ref)} mismatches"
    row = synth.Projection("down", "row", 1024, (512,))
    case = H.make_case(1400 + n + T, row, "nfs", n, T, ranks=[8, 16, 32], integer=True)
    ads = case.oracle_adapters()
    for i in range(n):
        got = _np(run_row_partial(case, i, dev))
        ref = ol.bf16_round(ol.row_partial_nfs(case.X.f64, case.W.f64, ads, case.ids, n, i))
        assert np.array_equal(got, ref), f"row rank {i}: {np.count_nonzero(got != ref)} mismatches"


# ----------------------------------------------------------------------------- downward-compatible BD

def _run_blocks(case, nl, i, dev):
    """Pool with tp_size = nl loading case's N_h-format adapters through bdlora_load_adapter_blocks."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = case.proj
    par = bd.COLUMN if proj.parallel == "column" else bd.ROW
    pool = bd.bdlora_create_pool(par, bd.SHARD_BD, nl, i, proj.d_in, proj.d_out, case.capacity, case.max_rank)
    for a, ad in case.adapters.items():
        bd.bdlora_load_adapter_blocks(pool, a, ad.rank, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                                      [H.torch_bf16(x.bits) for x in ad.B], case.n)
    X = H.torch_bf16(H.x_shard(case.X, proj, nl, i), dev)
    W = H.torch_bf16(H.base_shard_T(case.W, proj, nl, i), dev)
    ids = torch.from_numpy(case.ids).to(dev)
    T = X.shape[0]
    Y = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    (bd.bdlora_column_forward if par == bd.COLUMN else bd.bdlora_row_partial)(pool, X, W, ids, Y, ws)
    torch.cuda.synchronize()
    pool.close()
    return Y


@pytest.mark.parametrize("nh,nl", [(8, 1), (8, 2), (8, 4), (4, 2)])
@pytest.mark.parametrize("T", [1, 37])
def test_downward_compatible_serving(dev, nh, nl, T):
    """Adapters trained for N_h devices served on N_l | N_h devices: column device blocks and
    row partials vs the oracle of the N_h-block adapter read off in the N_l layout."""
    qkv, down = synth.arch_projections("llama-3.1-8b")[0], synth.arch_projections("llama-3.1-8b")[3]
    case = H.make_case(1500 + 10 * nh + nl + T, qkv, "bd", nh, T, ranks=[16, 32, 8])
    ref_full = ol.column_layer(case.X.f64, case.W.f64, qkv.d_out, case.oracle_adapters(), case.ids, "bd", nh)
    for i in sorted({0, nl - 1}):
        _assert_tol(_np(_run_blocks(case, nl, i, dev)), ol.column_device_output(ref_full, nl, i), f"col {nh}->{nl} dev {i}")
    case = H.make_case(1600 + 10 * nh + nl + T, down, "bd", nh, T, ranks=[16, 32])
    ads = case.oracle_adapters()
    acc = None
    for i in range(nl):
        P = _np(_run_blocks(case, nl, i, dev))
        _assert_tol(P, ol.row_partial_bd_blocks(case.X.f64, case.W.f64, ads, case.ids, nh, nl, i), f"row {nh}->{nl} dev {i}")
        acc = P if acc is None else acc + P
    _assert_tol(acc, ol.row_layer(case.X.f64, case.W.f64, ads, case.ids, "bd", nh), f"row {nh}->{nl} sum")


def test_downward_compatible_integer_bit_exact(dev):
    """P10 for downward-compatible serving: N_h = 8 adapters on N_l = 2, bit-identical to the oracle."""
    col = synth.Projection("qkv", "column", 1024, (512, 256, 256))
    case = H.make_case(1700, col, "bd", 8, 9, ranks=[8, 16, 32], integer=True)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, col.d_out, case.oracle_adapters(), case.ids, "bd", 8)
    for i in range(2):
        got, ref = _np(_run_blocks(case, 2, i, dev)), ol.bf16_round(ol.column_device_output(ref_full, 2, i))
        assert np.array_equal(got, ref), f"dev {i}: {np.count_nonzero(got != ref)} mismatches"
    row = synth.Projection("down", "row", 1024, (512,))
    case = H.make_case(1701, row, "bd", 8, 9, ranks=[8, 16, 32], integer=True)
    ads = case.oracle_adapters()
    for i in range(2):
        got = _np(_run_blocks(case, 2, i, dev))
        ref = ol.bf16_round(ol.row_partial_bd_blocks(case.X.f64, case.W.f64, ads, case.ids, 8, 2, i))
        assert np.array_equal(got, ref), f"row dev {i}: {np.count_nonzero(got != ref)} mismatches"


@pytest.mark.parametrize("T", [64, 150])
def test_downward_compatible_long_batches(dev, T):
    """Downward-compatible serving beyond one 64-token decode batch (the library runs such pools in chunks of
    <= 64 tokens): N_h = 8 adapters on N_l = 1 and 2, several adapters, id -1 tokens, vs the oracle."""
    qkv, down = synth.arch_projections("llama-3.1-8b")[0], synth.arch_projections("llama-3.1-8b")[3]
    for nl in (1, 2):
        case = H.make_case(1800 + T + nl, qkv, "bd", 8, T, ranks=[16, 32, 8])
        ref_full = ol.column_layer(case.X.f64, case.W.f64, qkv.d_out, case.oracle_adapters(), case.ids, "bd", 8)
        _assert_tol(_np(_run_blocks(case, nl, nl - 1, dev)), ol.column_device_output(ref_full, nl, nl - 1),
                    f"col 8->{nl} T={T}")
        case = H.make_case(1900 + T + nl, down, "bd", 8, T, ranks=[16, 32])
        P = _np(_run_blocks(case, nl, 0, dev))
        _assert_tol(P, ol.row_partial_bd_blocks(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, 8, nl, 0),
                    f"row 8->{nl} T={T}")


def test_downward_compatible_stores_no_zeros(dev):
    """P:389 / P:1082: the local blocks of a downward-compatible adapter are stored compactly -- resident bytes
    are exactly those of the m = N_h / N_l diagonal blocks (COLUMN: B_j [r/N_h, d_out_j/N_l]; ROW: A
    [r/N_l, d_in/N_h]), rounded up to whole K-rows; and one pool holds one block count."""
    import paper_2510_23346_b200 as bd

    qkv, down = synth.arch_projections("llama-3.1-8b")[0], synth.arch_projections("llama-3.1-8b")[3]
    nh, r = 8, 32
    for nl in (1, 2, 4):
        for proj in (qkv, down):
            case = H.make_case(2000 + nl, proj, "bd", nh, 1, ranks=[r])
            par = bd.COLUMN if proj.parallel == "column" else bd.ROW
            pool = bd.bdlora_create_pool(par, bd.SHARD_BD, nl, 0, proj.d_in, proj.d_out, 2, r)
            ad = case.adapters[0]
            bd.bdlora_load_adapter_blocks(pool, 0, r, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                                          [H.torch_bf16(x.bits) for x in ad.B], nh)
            resident, _ = bd.bdlora_pool_bytes(pool)
            K = proj.d_in if par == bd.COLUMN else proj.d_in // nl
            if par == bd.COLUMN:
                elems = sum((r // nl) * K + (r // nh) * (dj // nl) for dj in proj.d_out)
                dense = sum((r // nl) * K + (r // nl) * (dj // nl) for dj in proj.d_out)
            else:
                elems = (r // nl) * (K // (nh // nl)) + (r // nl) * proj.d_out[0]
                dense = (r // nl) * K + (r // nl) * proj.d_out[0]
            assert resident == -(-elems // K) * K * 2, (nl, proj.name, resident, elems)
            if nh // nl > 1:
                assert resident < dense * 2
                # a native (one-block) adapter cannot join a pool holding m > 1 blocks per device
                with pytest.raises(bd.BdloraError):
                    bd.bdlora_load_adapter(pool, 1, r, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                                           [H.torch_bf16(x.bits) for x in ad.B])
            pool.close()


# ----------------------------------------------------------------------------- Alg. 2

def test_alg2_column_forward_gather(dev):
    """Alg. 2: column forward + all-gather of the device outputs.  On one GPU: N = 1 (the gather is the
    identity) vs the oracle's full output, and the N > 1 contract (a communicator is required)."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.tiny_pair()[0]
    case = H.make_case(1800, proj, "bd", 1, 16, ranks=[8, 8, 16])
    pool = H.make_pool(case, 0)
    X, W, ids = H.device_inputs(case, 0, dev)
    Y = torch.full((16, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, 16)
    bd.bdlora_column_forward_gather(pool, None, X, W, ids, Y, ws)
    torch.cuda.synchronize()
    ref = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 1)[0]
    _assert_tol(_np(Y), ref, "Alg. 2 N=1")
    pool.close()
    case2 = H.make_case(1801, proj, "bd", 2, 16, ranks=[8])
    pool2 = H.make_pool(case2, 1)
    X2, W2, ids2 = H.device_inputs(case2, 1, dev)
    Y2 = torch.empty(16, 2 * pool2.m_loc, dtype=torch.bfloat16, device=dev)
    with pytest.raises(bd.BdloraError) as ei:
        bd.bdlora_column_forward_gather(pool2, None, X2, W2, ids2, Y2, bd.make_workspace(pool2, 16))
    assert ei.value.code == 1
    pool2.close()


# ----------------------------------------------------------------------------- P10 integer mode

@pytest.mark.parametrize("sharding", ["bd", "slora"])
@pytest.mark.parametrize("n", [1, 4])
def test_integer_mode_bit_exact_column(dev, sharding, n):
    """P10: {-1,0,1} inputs, s a power of two: every partial sum is exact, so the GPU output must be
    bit-identical to the oracle rounded once to bf16, for every rank; routing errors show up
    through each adapter's B signature."""
    proj = synth.Projection("qkv", "column", 1024, (512, 256, 256))
    T = 21
    case = H.make_case(500 + n, proj, sharding, n, T, ranks=[8, 16, 8, 32], integer=True)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, sharding, n)
    if sharding == "bd":
        outs = [run_column(case, i, dev) for i in range(n)]
    else:
        outs, _ = _slora_column_emulated(case, dev)
    for i in range(n):
        ref = ol.bf16_round(ol.column_device_output(ref_full, n, i))
        got = _np(outs[i])
        assert np.array_equal(got, ref), f"rank {i}: {np.count_nonzero(got != ref)} mismatches"


@pytest.mark.parametrize("n", [1, 2, 4])
def test_integer_mode_bit_exact_row_partials(dev, n):
    proj = synth.Projection("down", "row", 1024, (512,))
    T = 19
    case = H.make_case(600 + n, proj, "bd", n, T, ranks=[8, 16, 32], integer=True)
    ads = case.oracle_adapters()
    for i in range(n):
        ref = ol.bf16_round(ol.row_partial_bd(case.X.f64, case.W.f64, ads, case.ids, n, i))
        got = _np(run_row_partial(case, i, dev))
        assert np.array_equal(got, ref), f"rank {i}: {np.count_nonzero(got != ref)} mismatches"


# ----------------------------------------------------------------------------- multi-tenant / pool

def test_multitenant_mixed_ranks_ragged_arena(dev):
    """C4-like: 16 resident adapters r in {8,16,32,64,128}, uniform ids over them, T=64, TP=8
    (70B-gate_up-like but narrower), ragged arena with unload / reload."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.Projection("gate_up", "column", 2048, (3584, 3584))
    n, T = 8, 64
    ranks = [[8, 16, 32, 64, 128][k % 5] for k in range(16)]
    rng = synth.rng_for(7, 7)
    ids = synth.ids_uniform(rng, T, 16)
    case = H.make_case(700, proj, "bd", n, T, ranks=ranks, ids=ids)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", n)
    i = 5
    pool = H.make_pool(case, i, arena_bytes=64 << 20)
    # unload + reload a few slots to exercise the ragged allocator
    for a in (3, 7, 11):
        bd.bdlora_unload_adapter(pool, a)
    for a in (11, 3, 7):
        ad = case.adapters[a]
        bd.bdlora_load_adapter(pool, a, ad.rank, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                               [H.torch_bf16(x.bits) for x in ad.B])
    X, W, idt = H.device_inputs(case, i, dev)
    Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
    bd.bdlora_column_forward(pool, X, W, idt, Y, bd.make_workspace(pool, T))
    torch.cuda.synchronize()
    _assert_tol(_np(Y), ol.column_device_output(ref_full, n, i), "multi-tenant")
    res, arena = bd.bdlora_pool_bytes(pool)
    assert 0 < res <= arena
    pool.close()


def test_device_resident_factor_loading(dev):
    """Loading from device pointers gives the same result as from host pointers."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.tiny_pair()[1]
    case = H.make_case(61, proj, "bd", 2, 16, ranks=[8, 8])
    p_host = H.make_pool(case, 1)
    p_dev = bd.bdlora_create_pool(bd.ROW, bd.SHARD_BD, 2, 1, proj.d_in, proj.d_out, 2, 8)
    for a, ad in case.adapters.items():
        bd.bdlora_load_adapter(p_dev, a, ad.rank, ad.scale, [H.torch_bf16(x.bits, dev) for x in ad.A],
                               [H.torch_bf16(x.bits, dev) for x in ad.B])
    X, W, ids = H.device_inputs(case, 1, dev)
    outs = []
    for p in (p_host, p_dev):
        P = torch.empty(16, p.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_row_partial(p, X, W, ids, P, bd.make_workspace(p, 16))
        outs.append(P)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    p_host.close()
    p_dev.close()


# ----------------------------------------------------------------------------- errors / edge cases

def test_error_paths(dev):
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.tiny_pair()[0]
    case = H.make_case(71, proj, "bd", 2, 4, ranks=[8])
    pool = H.make_pool(case, 0)
    X, W, ids = H.device_inputs(case, 0, dev)
    Y = torch.empty(4, pool.m_loc, dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, 4)
    with pytest.raises(bd.BdloraError) as e:
        bd.slora_column_forward(pool, None, X, W, ids, Y, ws)
    assert e.value.code == 5
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_row_partial(pool, X, W, ids, Y, ws)
    assert e.value.code == 5
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_column_forward(pool, X, W, ids, Y, ws[:128])
    assert e.value.code == 1
    a = case.adapters[0]
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_load_adapter(pool, 0, 16, 1.0, [H.torch_bf16(x.bits) for x in a.A], [H.torch_bf16(x.bits) for x in a.B])
    assert e.value.code == 3  # rank > max_rank
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_load_adapter(pool, 5, 8, 1.0, [H.torch_bf16(x.bits) for x in a.A], [H.torch_bf16(x.bits) for x in a.B])
    assert e.value.code == 3  # slot out of range
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_load_adapter(pool, 0, 7, 1.0, [H.torch_bf16(x.bits) for x in a.A], [H.torch_bf16(x.bits) for x in a.B])
    assert e.value.code == 2  # N does not divide r
    with pytest.raises(bd.BdloraError) as e:
        bd.bdlora_unload_adapter(pool, 0) or bd.bdlora_unload_adapter(pool, 0)
    assert e.value.code == 4
    # T = 0 is a no-op
    bd.bdlora_column_forward(pool, X[:0], W, ids[:0], Y[:0], ws)
    pool.close()


# ----------------------------------------------------------------------------- launch paths

@pytest.mark.parametrize("pdl", [True, False])
def test_pdl_on_off_identical(dev, pdl):
    """Programmatic-dependent-launch chaining changes only scheduling, never values."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[2]
    case = H.make_case(81, proj, "bd", 8, 5, ranks=[16, 32])
    bd.bdlora_set_pdl(pdl)
    try:
        y = run_column(case, 3, dev)
    finally:
        bd.bdlora_set_pdl(True)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 8)
    _assert_tol(_np(y), ol.column_device_output(ref_full, 8, 3), f"pdl={pdl}")


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("pi,n,T", [(0, 1, 1), (0, 8, 5), (2, 1, 16), (2, 4, 3), (3, 2, 7), (1, 1, 1), (3, 8, 12)])
def test_decode_lora_schedules(dev, mode, pi, n, T):
    """Decode (T <= 16) single-kernel forward under the three LoRA schedules of bdlora_set_decode_lora
    (0 global shrink, 1 auto, 2 K-local: each K-range contributor adds s (X_seg A_seg) B to its partial,
    Alg. 1/2 regrouped over K) -- all against the oracle.  8B shapes: QKV whole/split-K tiles, gate_up
    stream-K, O and down row partials (split-K)."""
    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[pi]
    case = H.make_case(900 + 31 * pi + 7 * n + T, proj, "bd", n, T, ranks=[16, 32, 8])
    ads = case.oracle_adapters()
    bd.bdlora_set_decode_lora(mode)
    try:
        for i in sorted({0, n - 1}):
            if proj.parallel == "column":
                ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, ads, case.ids, "bd", n)
                _assert_tol(_np(run_column(case, i, dev)), ol.column_device_output(ref_full, n, i),
                            f"mode={mode} rank {i}")
            else:
                _assert_tol(_np(run_row_partial(case, i, dev)),
                            ol.row_partial_bd(case.X.f64, case.W.f64, ads, case.ids, n, i), f"mode={mode} rank {i}")
    finally:
        bd.bdlora_set_decode_lora(1)


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("n", [1, 4])
def test_integer_mode_bit_exact_decode(dev, mode, n):
    """P10 at decode sizes (T <= 16, single-kernel forward) under the global and the K-local LoRA
    schedule: bit-identical to the oracle rounded once to bf16 on every rank."""
    import paper_2510_23346_b200 as bd

    proj = synth.Projection("qkv", "column", 1024, (512, 256, 256))
    case = H.make_case(700 + n, proj, "bd", n, 9, ranks=[8, 16, 8, 32], integer=True)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", n)
    bd.bdlora_set_decode_lora(mode)
    try:
        for i in range(n):
            ref = ol.bf16_round(ol.column_device_output(ref_full, n, i))
            got = _np(run_column(case, i, dev))
            assert np.array_equal(got, ref), f"mode={mode} rank {i}: {np.count_nonzero(got != ref)} mismatches"
    finally:
        bd.bdlora_set_decode_lora(1)


def test_cuda_core_gemv_path_k_not_multiple_of_64(dev):
    """K % 64 != 0 takes the CUDA-core GEMV kernel (still on the GPU): parity on a ragged K."""
    proj = synth.Projection("odd", "column", 200, (96, 32))
    case = H.make_case(82, proj, "bd", 2, 7, ranks=[8, 16])
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 2)
    for i in range(2):
        _assert_tol(_np(run_column(case, i, dev)), ol.column_device_output(ref_full, 2, i), f"rank {i}")


@pytest.mark.parametrize("T", [129, 300])
def test_prefill_token_tiles(dev, T):
    """More tokens than one 256-wide token tile (n_tiles > 1) and a ragged token tail, segments of
    requests (SGMV-shaped ids), TP=8 rank 3 of 8B gate_up-like shapes (narrowed)."""
    proj = synth.Projection("gate_up", "column", 1024, (2048, 2048))
    ids = synth.ids_segments(T, 3)
    case = H.make_case(83 + T, proj, "bd", 8, T, ranks=[64, 32, 64], ids=ids)
    ref_full = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 8)
    _assert_tol(_np(run_column(case, 3, dev)), ol.column_device_output(ref_full, 8, 3), f"T={T}")


# ----------------------------------------------------------------------------- full-size, sampled

def _sampled_check(y_dev, X, W_cols, col_index, ads_dense, ids, rng, n_samples=96, what=""):
    """Compare n_samples random outputs of a full-size device output against the oracle computed one by
    one (oracle.lora_layer_sampled): W_cols[:, q] is the base weight column of local output column
    col_index[q] (paper orientation)."""
    T, M = y_dev.shape
    ts = rng.integers(0, T, size=n_samples)
    cs = rng.integers(0, M, size=n_samples)
    got = y_dev[ts, cs].astype(np.float64)
    # oracle.lora_layer_sampled, one output at a time (dW column = A B[:, c] materialised)
    out = np.empty(n_samples)
    for k, (t, c) in enumerate(zip(ts, cs)):
        out[k] = ol.lora_layer_sampled(X, W_cols, ads_dense, ids, [(int(t), int(col_index[c]))])[0]
    _assert_tol(got, out, what)


def test_full_size_bench_config_8b_decode(dev):
    """The bench's own workload at full size and in its launch configuration: Llama-3.1-8B layer,
    decode T=1, rank 16, TP=1 -- every projection, sampled outputs vs the oracle one by one."""
    import torch

    import paper_2510_23346_b200 as bd

    rng_s = np.random.default_rng(5)
    for k, proj in enumerate(synth.arch_projections("llama-3.1-8b")):
        case = H.make_case(900 + k, proj, "bd", 1, 1, ranks=[16], ids=np.zeros(1, np.int32))
        pool = H.make_pool(case, 0)
        X, W, ids = H.device_inputs(case, 0, dev)
        Y = torch.empty(1, pool.m_loc, dtype=torch.bfloat16, device=dev)
        ws = bd.make_workspace(pool, 1)
        if proj.parallel == "column":
            bd.bdlora_column_forward(pool, X, W, ids, Y, ws)
        else:
            bd.bdlora_row_forward(pool, None, X, W, ids, Y, ws)
        torch.cuda.synchronize()
        ads = case.oracle_adapters()
        Wf = case.W.f64
        if proj.parallel == "column":
            # local columns are [q|k|v] or [gate|up] = full columns at N=1; per slice factors
            y = _np(Y)
            col0 = 0
            for j, dj in enumerate(proj.d_out):
                dense = {a: (d["scale"],) + ol.dense_factors("column", "bd", d["A"], d["B"], 1)[j] for a, d in ads.items()}
                _sampled_check(y[:, col0:col0 + dj], case.X.f64, Wf[:, col0:col0 + dj], np.arange(dj), dense,
                               case.ids, rng_s, 48, f"{proj.name} slice {j}")
                col0 += dj
        else:
            dense = {a: (d["scale"],) + ol.dense_factors("row", "bd", d["A"], d["B"], 1)[0] for a, d in ads.items()}
            _sampled_check(_np(Y), case.X.f64, Wf, np.arange(proj.d_out[0]), dense, case.ids, rng_s, 96, proj.name)
        pool.close()


def test_full_size_multitenant_70b_gate_up_tp8(dev):
    """configs[4] at full size on one emulated rank: Llama-3.1-70B gate_up (8192 -> 2 x 28672) at TP=8,
    64 decode tokens over 128 resident adapters of mixed rank {8..128}, uniform ids; sampled outputs."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-70b")[2]
    n, i, T = 8, 5, 64
    ranks = [[8, 16, 32, 64, 128][k % 5] for k in range(128)]
    rng = synth.rng_for(910, 1)
    ids = synth.ids_uniform(rng, T, 128)
    ads = {a: synth.make_adapter(rng, proj, "bd", r, n, synth.rs_scale(16.0, r, n, "bd")) for a, r in enumerate(ranks)}
    X = synth.make_x(rng, T, proj.d_in)
    # only device i's base columns are generated (column-parallel: W_i = column block i of each slice)
    w_loc = [synth.bf16_normal(rng, (proj.d_in, dj // n), 1 / np.sqrt(proj.d_in)) for dj in proj.d_out]
    pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, n, i, proj.d_in, proj.d_out, 128, 128, device=0)
    for a, ad in ads.items():
        bd.bdlora_load_adapter(pool, a, ad.rank, ad.scale, [H.torch_bf16(x.bits) for x in ad.A],
                               [H.torch_bf16(x.bits) for x in ad.B])
    Wt = H.torch_bf16(np.ascontiguousarray(np.concatenate([w.bits for w in w_loc], axis=1).T), dev)
    Xd = H.torch_bf16(X.bits, dev)
    Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
    bd.bdlora_column_forward(pool, Xd, Wt, torch.from_numpy(ids).to(dev), Y, bd.make_workspace(pool, T))
    torch.cuda.synchronize()
    y = _np(Y)
    used = sorted(set(ids.tolist()))
    rng_s = np.random.default_rng(6)
    col0 = 0
    for j, dj in enumerate(proj.d_out):
        w = dj // n
        dense = {}
        for a in used:
            A, B = ol.dense_factors("column", "bd", [x.f64 for x in ads[a].A], [x.f64 for x in ads[a].B], n)[j]
            dense[a] = (ads[a].scale, A, B)
        # local column c of slice j is full column i*w + c; W_cols holds only the local block
        Wfull_cols = np.zeros((proj.d_in, dj))
        Wfull_cols[:, i * w:(i + 1) * w] = w_loc[j].f64
        _sampled_check(y[:, col0:col0 + w], X.f64, Wfull_cols, i * w + np.arange(w), dense, ids, rng_s, 64,
                       f"70B gate_up slice {j}")
        col0 += w
    pool.close()


@pytest.mark.parametrize("n,T,ranks", [(4, 37, [16, 16, 32]), (8, 64, [8, 24, 64, 128]), (1, 200, [16, 48])])
def test_shrink_v_against_oracle(dev, n, T, ranks):
    """The shrink's fp32 intermediate v (tensor-core path for T > 16, CUDA-core below) equals
    s_a x_t A_j[:, chunk i] for every token and slice (~1e-5 relative)."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[0]
    case = H.make_case(950 + n + T, proj, "bd", n, T, ranks=ranks)
    J, Rc = 3, max(ranks) // n
    for i in (0, n - 1):
        pool = H.make_pool(case, i)
        X, W, ids = H.device_inputs(case, i, dev)
        v = torch.full((bd.bdlora_v_elems(pool, T),), float("nan"), dtype=torch.float32, device=dev)
        bd.bdlora_lora_shrink(pool, X, ids, v, bd.make_workspace(pool, T))
        torch.cuda.synchronize()
        vv = v.cpu().numpy().reshape(T, J, Rc).astype(np.float64)
        for t in range(T):
            a = int(case.ids[t])
            if a < 0:
                continue
            ad = case.adapters[a]
            rs = ad.rank // n
            for j in range(J):
                ref = ad.scale * (case.X.f64[t] @ ad.A[j].f64[:, i * rs:(i + 1) * rs])
                assert np.allclose(vv[t, j, :rs], ref, rtol=1e-3, atol=1e-4 * (np.abs(ref).max() + 1)), (i, t, j)
        pool.close()
