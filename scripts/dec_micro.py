"""Decode-kernel micro-benchmark: one projection's bdlora_column_forward / row_partial timed back to back in a
CUDA graph (weights rotated over >= 3 x L2), and one traced launch (per-CTA %globaltimer stamps + %smid).
usage: python scripts/dec_micro.py [M K T rank]..."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402

dev = torch.device("cuda", 0)
L2 = 126 << 20


def bench(fn, iters=40):
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


def run(M, K, T, rank):
    pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, 1, 0, K, [M], 1, rank)
    A = (torch.randn(K, rank, device=dev) / math.sqrt(K)).to(torch.bfloat16)
    B = (torch.randn(rank, M, device=dev) / 4).to(torch.bfloat16)
    bd.bdlora_load_adapter(pool, 0, rank, 1.0, [A], [B])
    nrep = max(2, math.ceil(3 * L2 / (M * K * 2)))
    Ws = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(nrep)]
    X = torch.randn(T, K, device=dev).to(torch.bfloat16)
    ids = torch.zeros(T, dtype=torch.int32, device=dev)
    if os.environ.get("NOLORA"):
        ids = -torch.ones(T, dtype=torch.int32, device=dev)
    Y = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
    ws = bd.make_workspace(pool, T)
    us = bench(lambda i: bd.bdlora_column_forward(pool, X, Ws[i % nrep], ids, Y, ws))
    info = bd.bdlora_last_launch_info()
    tr = torch.zeros(1024 * 32, dtype=torch.int64, device=dev)
    bd.bdlora_debug_trace(tr)
    for r in range(2):
        bd.bdlora_column_forward(pool, X, Ws[r % nrep], ids, Y, ws)
        torch.cuda.synchronize()
    bd.bdlora_debug_trace(None)
    t = tr.view(1024, 32).cpu().numpy()[: info["grid"]]
    t0 = t[:, 0].min()
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    sm = t[:, 31]
    per_sm = np.bincount(sm.astype(np.int64), minlength=148)
    gb = M * K * 2 / 1e9
    print(f"M={M} K={K} T={T} r={rank}: {us:.2f} us/launch ({gb / (us * 1e-6):.0f} GB/s)  info={info}")
    print(f"   CTAs on distinct SMs {np.count_nonzero(per_sm)} (max per SM {per_sm.max()})")
    for k, nm in [(0, "entry"), (1, "ring0 issued"), (2, "first mma"), (3, "epi pre-wait"), (4, "acc ready"),
                  (9, "tc v read"), (11, "peers started"), (12, "pushed"), (6, "reduced"), (7, "epi end"),
                  (8, "producer end")]:
        if (t[:, k] <= 0).all():
            continue
        c = rel(k)
        print(f"   {nm:14s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} us")
    end = rel(7)
    order = np.argsort(-end)[:4]
    names = ["entry", "ring0", "mma0", "pre", "acc", "-", "fin", "end", "prod"]
    print("   slowest CTAs:", " ".join(f"{nm:>6s}" for nm in names), "sm")
    for c in order:
        print("   ", f"{c:4d}", " ".join(f"{rel(k)[c]:6.2f}" if t[c, k] > 0 else "     -" for k in range(9)), int(sm[c]))
    pool.close()


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    shapes = [tuple(args[i:i + 4]) for i in range(0, len(args), 4)] or [
        (28672, 4096, 1, 16), (6144, 4096, 1, 16), (4096, 4096, 1, 16), (768, 4096, 1, 2), (4096, 512, 1, 2),
        (3584, 4096, 1, 2), (4096, 1792, 1, 2)]
    for s in shapes:
        run(*s)
