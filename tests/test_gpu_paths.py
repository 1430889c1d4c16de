"""GPU parity of the ABI entry points that the bench times but the per-projection tests reach only through
other calls, of the chained decode step, of the workspace contract and of large batches -- all against the
fp64 oracle (SURVEY §8(c) step 7 tolerance unless a test says bit-exact)."""
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


def _fwd(fn, case, dev, comm=None, T=None):
    import torch

    import paper_2510_23346_b200 as bd

    pool = H.make_pool(case, 0)
    X, W, ids = H.device_inputs(case, 0, dev)
    T = X.shape[0]
    Y = torch.full((T, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    if fn in (bd.slora_column_forward, bd.slora_row_forward, bd.nfs_row_forward, bd.bdlora_row_forward):
        fn(pool, comm, X, W, ids, Y, ws)
    else:
        fn(pool, X, W, ids, Y, ws)
    torch.cuda.synchronize()
    pool.close()
    return _np(Y)


# ----------------------------------------------------------------------------- ABI entry points at N = 1
# N = 1: every sharding is plain LoRA (P3, P4) and no collective is issued (comm may be NULL), so the
# full forwards -- including the code between the shrink and the GEMM that the collectives sit in --
# run on one GPU.

@pytest.mark.parametrize("T", [1, 9, 40])
def test_slora_column_forward_n1(dev, T):
    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[0]
    case = H.make_case(4000 + T, proj, "slora", 1, T, ranks=[16, 32, 8])
    ref = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "slora", 1)
    _assert_tol(_fwd(bd.slora_column_forward, case, dev), ol.column_device_output(ref, 1, 0), f"T={T}")


@pytest.mark.parametrize("T", [1, 9, 40])
def test_slora_row_forward_n1(dev, T):
    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[1]
    case = H.make_case(4100 + T, proj, "slora", 1, T, ranks=[16, 24])
    ref = ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "slora", 1)
    _assert_tol(_fwd(bd.slora_row_forward, case, dev), ref, f"T={T}")


@pytest.mark.parametrize("T", [1, 9, 40])
def test_nfs_row_forward_n1(dev, T):
    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[3]
    case = H.make_case(4200 + T, proj, "nfs", 1, T, ranks=[16, 12])
    ref = ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "nfs", 1)
    _assert_tol(_fwd(bd.nfs_row_forward, case, dev), ref, f"T={T}")


def test_slora_entry_points_integer_bit_exact(dev):
    """P10 through slora_column_forward / slora_row_forward themselves (N = 1)."""
    import paper_2510_23346_b200 as bd

    col = synth.Projection("qkv", "column", 1024, (512, 256, 256))
    case = H.make_case(4300, col, "slora", 1, 21, ranks=[8, 16, 32], integer=True)
    ref = ol.bf16_round(ol.column_device_output(
        ol.column_layer(case.X.f64, case.W.f64, col.d_out, case.oracle_adapters(), case.ids, "slora", 1), 1, 0))
    got = _fwd(bd.slora_column_forward, case, dev)
    assert np.array_equal(got, ref), f"{np.count_nonzero(got != ref)} mismatches"
    row = synth.Projection("down", "row", 1024, (512,))
    case = H.make_case(4301, row, "slora", 1, 21, ranks=[8, 16, 32], integer=True)
    ref = ol.bf16_round(ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "slora", 1))
    got = _fwd(bd.slora_row_forward, case, dev)
    assert np.array_equal(got, ref), f"{np.count_nonzero(got != ref)} mismatches"


# ----------------------------------------------------------------------------- bf16 all-reduce model (H8)

def _ring_bf16_sum(parts):
    """What a bf16 ring all-reduce can return: partials summed one at a time with a bf16 rounding after each
    add (the reduction runs in the wire dtype).  Order: rank order, a valid ring order for one chunk."""
    acc = ol.bf16_round(parts[0])
    for p in parts[1:]:
        acc = ol.bf16_round(acc + p)
    return acc


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("T", [1, 37])
def test_row_partials_bf16_allreduce(dev, n, T):
    """bdlora_row_forward all-reduces the bf16 row partials with ncclBfloat16 (reading R7): the layer output is
    then the partials summed in bf16.  Emulated on one GPU with each rank's partial from the library, reduced
    in bf16 (ring model) -- the result must still meet the tolerance against the unsharded oracle, at the
    8B O and down shapes and the largest N."""
    for proj in synth.arch_projections("llama-3.1-8b")[1::2]:
        case = H.make_case(4400 + n * 10 + T, proj, "bd", n, T, ranks=[16, 32])
        import torch

        import paper_2510_23346_b200 as bd

        parts = []
        for i in range(n):
            pool = H.make_pool(case, i)
            X, W, ids = H.device_inputs(case, i, dev)
            P = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
            bd.bdlora_row_partial(pool, X, W, ids, P, bd.make_workspace(pool, T))
            torch.cuda.synchronize()
            parts.append(_np(P))
            pool.close()
        y = _ring_bf16_sum(parts)
        _assert_tol(y, ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "bd", n),
                    f"{proj.name} N={n} T={T} bf16 ring sum")


# ----------------------------------------------------------------------------- the chained decode step (8(f) row 3)

def _chain_model(seed, L, d_h=512, d_i=1024, d_kv=128, r=16, n=1):
    projs = synth.llama_projections(d_h, d_i, d_kv)
    rng = synth.rng_for(seed, 31)
    layers = []
    for layer in range(L):
        ent = []
        for p in projs:
            W = synth.make_base(rng, p)
            ad = synth.make_adapter(rng, p, "bd", r, n, synth.rs_scale(16.0, r, n, "bd"))
            ent.append((p, W, ad))
        layers.append(ent)
    return projs, layers


def _oracle_chain(x0, layers, T, n=1):
    """Layer-by-layer oracle of the chain bench.time_decode_step runs: QKV -> q slice -> O -> gate_up -> gate
    slice -> down -> next layer, every projection output rounded to bf16 (the activations are bf16, R7)."""
    x = x0
    outs = []
    ids = np.zeros(T, np.int32)
    for ent in layers:
        (pq, Wq, aq), (po, Wo, ao), (pg, Wg, ag), (pd, Wd, adn) = ent
        oa = lambda ad: {0: {"rank": ad.rank, "scale": ad.scale, "A": [a.f64 for a in ad.A],  # noqa: E731
                             "B": [b.f64 for b in ad.B]}}
        yq = ol.bf16_round(np.concatenate(ol.column_layer(x, Wq.f64, pq.d_out, oa(aq), ids, "bd", n), axis=1))
        yo = ol.bf16_round(ol.row_layer(yq[:, :po.d_in], Wo.f64, oa(ao), ids, "bd", n))
        yg = ol.bf16_round(np.concatenate(ol.column_layer(yo, Wg.f64, pg.d_out, oa(ag), ids, "bd", n), axis=1))
        yd = ol.bf16_round(ol.row_layer(yg[:, :pd.d_in], Wd.f64, oa(adn), ids, "bd", n))
        outs.append((yq, yo, yg, yd))
        x = yd
    return outs


@pytest.mark.parametrize("T", [1, 3])
@pytest.mark.parametrize("pdl", [True, False])
def test_decode_chain_graph_replay(dev, T, pdl):
    """4 decoder layers (narrowed Llama shapes, one adapter per layer) chained through their real inputs,
    captured in ONE CUDA graph and replayed twice, with programmatic dependent launch on and off.  Every
    projection output of every layer is compared with the oracle chain (PDL may only change scheduling)."""
    import torch

    import paper_2510_23346_b200 as bd

    L = 4
    projs, layers = _chain_model(4500 + T, L)
    rng = synth.rng_for(4501 + T, 1)
    x0 = synth.make_x(rng, T, projs[0].d_in)
    ref = _oracle_chain(x0.f64, layers, T)
    pools, Ws, Ys, wss = [], [], [], []
    for k, p in enumerate(projs):
        par = bd.COLUMN if p.parallel == "column" else bd.ROW
        pool = bd.bdlora_create_pool(par, bd.SHARD_BD, 1, 0, p.d_in, p.d_out, L, 16, device=0)
        for layer in range(L):
            _, W, ad = layers[layer][k]
            bd.bdlora_load_adapter(pool, layer, ad.rank, ad.scale, [H.torch_bf16(a.bits) for a in ad.A],
                                   [H.torch_bf16(b.bits) for b in ad.B])
        pools.append(pool)
        Ws.append([H.torch_bf16(np.ascontiguousarray(layers[layer][k][1].bits.T), dev) for layer in range(L)])
        Ys.append([torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev) for _ in range(L)])
        wss.append(bd.make_workspace(pool, T))
    ids = [torch.full((T,), layer, dtype=torch.int32, device=dev) for layer in range(L)]
    xin = H.torch_bf16(x0.bits, dev)
    xo = torch.empty(T, projs[1].d_in, dtype=torch.bfloat16, device=dev)
    xd = torch.empty(T, projs[3].d_in, dtype=torch.bfloat16, device=dev)

    def step():
        x = xin
        for layer in range(L):
            bd.bdlora_column_forward(pools[0], x, Ws[0][layer], ids[layer], Ys[0][layer], wss[0])
            xo.copy_(Ys[0][layer][:, :projs[1].d_in])  # attention placeholder: the q slice
            bd.bdlora_row_forward(pools[1], None, xo, Ws[1][layer], ids[layer], Ys[1][layer], wss[1])
            bd.bdlora_column_forward(pools[2], Ys[1][layer], Ws[2][layer], ids[layer], Ys[2][layer], wss[2])
            xd.copy_(Ys[2][layer][:, :projs[3].d_in])  # SiLU(gate)*up placeholder: the gate slice
            bd.bdlora_row_forward(pools[3], None, xd, Ws[3][layer], ids[layer], Ys[3][layer], wss[3])
            x = Ys[3][layer]

    bd.bdlora_set_pdl(pdl)
    try:
        step()  # eager run: the graph replay below must reproduce it bit for bit
        torch.cuda.synchronize()
        eager = [[y.clone() for y in Yl] for Yl in Ys]
        for Yl in Ys:
            for y in Yl:
                y.fill_(float("nan"))
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                step()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        g.replay()
        torch.cuda.synchronize()
    finally:
        bd.bdlora_set_pdl(True)
    for layer in range(L):
        for k in range(4):
            what = f"layer {layer} proj {projs[k].name} T={T} pdl={pdl}"
            # scheduling (graph replay, PDL) never changes a bit: every kernel reduces in a fixed order
            assert torch.equal(Ys[k][layer].view(torch.int16), eager[k][layer].view(torch.int16)), what + " != eager"
            # against the oracle chain: the GPU output of projection d (1-based depth in the chain) carries the
            # rounding of the d - 1 projections before it; independent roundings add in quadrature, so the
            # bound is sqrt(d) x the single-projection tolerance (reading R18)
            d = 4 * layer + k + 1
            ok, m, l1 = ol.within_tolerance(_np(Ys[k][layer]), ref[layer][k], max_rel=2e-2 * d ** 0.5,
                                            l1_rel=5e-3 * d ** 0.5)
            assert ok, f"{what}: max-rel {m:.3e} (<= {2e-2 * d ** 0.5:.2e}), l1-rel {l1:.3e} (<= {5e-3 * d ** 0.5:.2e})"
    for p in pools:
        p.close()


# ----------------------------------------------------------------------------- workspace contract (bdlora.h)

def test_workspace_reused_for_smaller_batches(dev):
    """A workspace sized for T = 64 serves T = 1, 3, 37, 64, 5 in turn (counter region at fixed offsets, left
    zero by every call), after bdlora_workspace_init on a buffer full of garbage."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[3]  # down: split-K tiles use the counters at every T
    case = H.make_case(4600, proj, "bd", 4, 64, ranks=[16, 32])
    pool = H.make_pool(case, 1)
    X, W, ids = H.device_inputs(case, 1, dev)
    ws = torch.full((bd.bdlora_workspace_bytes(pool, 64),), 0xA5, dtype=torch.uint8, device=dev)
    bd.bdlora_workspace_init(pool, ws)
    ads = case.oracle_adapters()
    for T in (1, 3, 37, 64, 5):
        P = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_row_partial(pool, X[:T].contiguous(), W, ids[:T].contiguous(), P, ws)
        torch.cuda.synchronize()
        ref = ol.row_partial_bd(case.X.f64[:T], case.W.f64, ads, case.ids[:T], 4, 1)
        _assert_tol(_np(P), ref, f"T={T}")
    pool.close()


# ----------------------------------------------------------------------------- batches beyond one route chunk

@pytest.mark.parametrize("d_in", [256, 200])
def test_forward_above_4096_tokens(dev, d_in):
    """T = 5000 > 4096 (the routing chunk): the shrink runs in chunks of <= 4096 tokens; d_in = 200 takes the
    CUDA-core shrink + GEMV path (K % 64 != 0), 256 the tensor-core one.  Mixed ids with -1 runs."""
    import paper_2510_23346_b200 as bd

    proj = synth.Projection("col", "column", d_in, (384,))
    case = H.make_case(4700 + d_in, proj, "bd", 2, 5000, ranks=[8, 16, 8, 32])
    ref = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 2)
    import torch

    pool = H.make_pool(case, 1)
    X, W, ids = H.device_inputs(case, 1, dev)
    Y = torch.full((5000, pool.m_loc), float("nan"), dtype=torch.bfloat16, device=dev)
    bd.bdlora_column_forward(pool, X, W, ids, Y, bd.make_workspace(pool, 5000))
    torch.cuda.synchronize()
    pool.close()
    _assert_tol(_np(Y), ol.column_device_output(ref, 2, 1), f"T=5000 d_in={d_in}")
