"""GPU parity of the fused row GEMM + all-reduce (include/bdlora.h "fused row all-reduce"):
Alg. 1 end to end with the base all-reduce done by the decode kernel's peer pushes and the
per-rank reduce kernel -- no NCCL.

One GPU: N ranks are emulated in one process with bdlora_peer_create_local (every rank's receive buffer mapped
directly instead of through CUDA IPC).  Every rank's push is issued before any rank's reduce (the emulation's
ordering rule), then every rank's Y is compared with the unsharded oracle row layer, and all ranks' outputs
must be bit-identical (the reduction runs in rank order on every rank).  The N > 1 multi-process path (IPC
handles exchanged over NCCL) is exercised by tests/test_gpu_multi.py when more than one GPU is present."""
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


def _setup(case, n, T):
    import torch

    import paper_2510_23346_b200 as bd

    pools = [H.make_pool(case, i) for i in range(n)]
    peers = bd.bdlora_peer_create_local(n, 16 * pools[0].m_loc)
    ins = [H.device_inputs(case, i, torch.device("cuda", 0)) for i in range(n)]
    wss = [bd.make_workspace(p, T) for p in pools]
    Ys = [torch.full((T, pools[0].m_loc), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    return pools, peers, ins, wss, Ys


def _call_all(pools, peers, ins, wss, Ys):
    import paper_2510_23346_b200 as bd

    for i, p in enumerate(pools):  # every rank's push first (one-device emulation rule)
        X, W, ids = ins[i]
        bd.bdlora_row_partial_push(p, peers[i], X, W, ids, wss[i])
    for i in range(len(pools)):
        bd.bdlora_peer_reduce(peers[i], Ys[i])


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("pi,T", [(1, 1), (3, 1), (1, 5), (3, 16)])
def test_fused_row_allreduce_vs_oracle(dev, n, pi, T):
    """8B O / down at TP = N: every rank's Y = AllReduce_i(P_i) against the unsharded oracle; all ranks equal."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[pi]
    ids = np.zeros(T, np.int32) if T == 1 else None
    case = H.make_case(6000 + 10 * n + pi + T, proj, "bd", n, T, ranks=[16], ids=ids)
    pools, peers, ins, wss, Ys = _setup(case, n, T)
    _call_all(pools, peers, ins, wss, Ys)
    torch.cuda.synchronize()
    assert all(bd.bdlora_peer_error(q) == 0 for q in peers)
    ref = ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "bd", n)
    for i in range(n):
        _assert_tol(_np(Ys[i]), ref, f"{proj.name} N={n} T={T} rank {i}")
        assert torch.equal(Ys[i].view(torch.int16), Ys[0].view(torch.int16)), f"rank {i} differs from rank 0"
    for q in peers:
        q.close()
    for p in pools:
        p.close()


@pytest.mark.parametrize("n", [2, 4])
def test_fused_row_allreduce_integer_bit_exact(dev, n):
    """P10: integer inputs -- the fp32 sum of exact partials rounded once equals the oracle rounded once."""
    import torch

    proj = synth.Projection("down", "row", 2048, (1024,))
    case = H.make_case(6100 + n, proj, "bd", n, 7, ranks=[8, 16], integer=True)
    pools, peers, ins, wss, Ys = _setup(case, n, 7)
    _call_all(pools, peers, ins, wss, Ys)
    torch.cuda.synchronize()
    ref = ol.bf16_round(ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "bd", n))
    for i in range(n):
        got = _np(Ys[i])
        assert np.array_equal(got, ref), f"rank {i}: {np.count_nonzero(got != ref)} mismatches"
    for q in peers:
        q.close()
    for p in pools:
        p.close()


def test_fused_row_allreduce_repeated_calls_graph(dev):
    """The call parity alternates and the counters re-arm: five calls in a row captured in one CUDA graph,
    replayed twice, each call with different X (the result of every call checked)."""
    import torch

    import paper_2510_23346_b200 as bd

    n, T = 4, 3
    proj = synth.arch_projections("llama-3.1-8b")[1]
    cases = [H.make_case(6200 + c, proj, "bd", n, T, ranks=[16]) for c in range(5)]
    pools = [H.make_pool(cases[0], i) for i in range(n)]
    peers = bd.bdlora_peer_create_local(n, T * pools[0].m_loc)
    wss = [bd.make_workspace(p, T) for p in pools]
    W = [H.device_inputs(cases[0], i, dev)[1] for i in range(n)]
    Xs = [[H.device_inputs(c, i, dev)[0] for i in range(n)] for c in cases]
    ids = torch.from_numpy(cases[0].ids).to(dev)
    Ys = [[torch.empty(T, pools[0].m_loc, dtype=torch.bfloat16, device=dev) for _ in range(n)] for _ in cases]

    def run():
        for c in range(len(cases)):
            for i in range(n):
                bd.bdlora_row_partial_push(pools[i], peers[i], Xs[c][i], W[i], ids, wss[i])
            for i in range(n):
                bd.bdlora_peer_reduce(peers[i], Ys[c][i])

    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            run()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        for Yc in Ys:
            for y in Yc:
                y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert all(bd.bdlora_peer_error(q) == 0 for q in peers)
        for c, case in enumerate(cases):
            # all cases share adapters and W with case 0 (the pools were loaded from case 0)
            ref = ol.row_layer(case.X.f64, cases[0].W.f64, cases[0].oracle_adapters(), cases[0].ids, "bd", n)
            for i in range(n):
                _assert_tol(_np(Ys[c][i]), ref, f"call {c} rank {i}")
    for q in peers:
        q.close()
    for p in pools:
        p.close()


def test_fused_row_allreduce_contract_errors(dev):
    """Shapes the fused path does not serve and mismatched peers are rejected before any launch."""
    import torch

    import paper_2510_23346_b200 as bd

    proj = synth.arch_projections("llama-3.1-8b")[1]
    case = H.make_case(6300, proj, "bd", 2, 32, ranks=[16])
    pools = [H.make_pool(case, i) for i in range(2)]
    peers = bd.bdlora_peer_create_local(2, 64 * pools[0].m_loc)
    X, W, ids = H.device_inputs(case, 0, dev)
    ws = bd.make_workspace(pools[0], 32)
    with pytest.raises(bd.BdloraError) as e:  # T = 32 > 16: decode batches only
        bd.bdlora_row_partial_push(pools[0], peers[0], X, W, ids, ws)
    assert e.value.code == 3
    with pytest.raises(bd.BdloraError) as e:  # peer of rank 1 with the pool of rank 0
        bd.bdlora_row_partial_push(pools[0], peers[1], X[:4].contiguous(), W, ids[:4].contiguous(), ws)
    assert e.value.code == 1
    col = H.make_case(6301, synth.arch_projections("llama-3.1-8b")[0], "bd", 2, 4, ranks=[16])
    cp = H.make_pool(col, 0)
    Xc, Wc, idc = H.device_inputs(col, 0, dev)
    with pytest.raises(bd.BdloraError) as e:  # column pools have no all-reduce
        bd.bdlora_row_partial_push(cp, peers[0], Xc, Wc, idc, bd.make_workspace(cp, 4))
    assert e.value.code == 5
    for q in peers:
        q.close()
    for p in pools + [cp]:
        p.close()
