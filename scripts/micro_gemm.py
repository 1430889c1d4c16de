"""Micro-benchmark of the base GEMM + fused expand kernel alone (bdlora_base_expand) vs cuBLAS
(torch.matmul) on decode shapes: separates fixed per-launch cost from streaming bandwidth.
Weights rotate over replicas totalling > 3 x L2 so every launch streams from HBM."""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402

dev = torch.device("cuda", 0)
L2 = 126 << 20


def bench(fn, reps, iters=40):
    """GPU time per call: `iters` calls captured in one CUDA graph, replayed (no host overhead)."""
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def run(M, K, T, lora=True, rank=16):
    pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, 1, 0, K, [M], 1, rank)
    A = (torch.randn(K, rank, device=dev) / math.sqrt(K)).to(torch.bfloat16)
    B = (torch.randn(rank, M, device=dev) / 4).to(torch.bfloat16)
    bd.bdlora_load_adapter(pool, 0, rank, 1.0, [A], [B])
    nrep = max(1, math.ceil(3 * L2 / (M * K * 2)))
    Ws = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(nrep)]
    X = torch.randn(T, K, device=dev).to(torch.bfloat16)
    ids = torch.zeros(T, dtype=torch.int32, device=dev) if lora else -torch.ones(T, dtype=torch.int32, device=dev)
    Y = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    v = torch.zeros(bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)
    bd.bdlora_lora_shrink(pool, X, ids, v, ws)
    us = bench(lambda i: bd.bdlora_base_expand(pool, X, Ws[i % nrep], ids, v, Y, ws), nrep)
    us_fwd = bench(lambda i: bd.bdlora_column_forward(pool, X, Ws[i % nrep], ids, Y, ws), nrep)
    us_sh = bench(lambda i: bd.bdlora_lora_shrink(pool, X, ids, v, ws), nrep)
    us_cublas = bench(lambda i: torch.matmul(X, Ws[i % nrep].t()), nrep)
    nids = -torch.ones(T, dtype=torch.int32, device=dev)
    us_base = bench(lambda i: bd.bdlora_column_forward(pool, X, Ws[i % nrep], nids, Y, ws), nrep)
    gb = (M * K * 2) / 1e9
    out = dict(M=M, K=K, T=T, lora=lora, us_gemm=us, us_fwd=us_fwd, us_shrink=us_sh, us_cublas=us_cublas, us_fwd_nolora=us_base,
               gbs_gemm=gb / (us * 1e-6), gbs_cublas=gb / (us_cublas * 1e-6))
    pool.close()
    return out


if __name__ == "__main__":
    res = []
    shapes = [(4096, 4096), (6144, 4096), (28672, 4096), (4096, 14336), (768, 4096), (4096, 512), (4096, 1792)]
    for M, K in shapes:
        for T in (1,):
            r = run(M, K, T)
            res.append(r)
            print(json.dumps(r), flush=True)
    r = run(6144, 4096, 1, lora=False)
    print(json.dumps(r), flush=True)
