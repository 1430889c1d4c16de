"""Per-CTA %globaltimer trace of BD decode forwards of one TP rank (one adapter, T tokens), chained in a CUDA
graph (PDL on) over rotating weights: median stamps per launch (us from the first launch's first stamp).
usage: python scripts/bd_trace.py ARCH PROJ_INDEX N T RANK"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402
import synth  # noqa: E402

arch, k, n, T, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
dev = torch.device("cuda", 0)
proj = synth.arch_projections(arch)[k]
par = bd.COLUMN if proj.parallel == "column" else bd.ROW
pool = bd.bdlora_create_pool(par, bd.SHARD_BD, n, 0, proj.d_in, proj.d_out, 1, r)
g = torch.Generator(device=dev)
g.manual_seed(0)
A, B = [], []
for dj in proj.d_out:
    if par == bd.COLUMN:
        A.append((torch.randn(proj.d_in, r, generator=g, device=dev) / 64).to(torch.bfloat16))
        B.append((torch.randn(r // n, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
    else:
        A.append((torch.randn(proj.d_in, r // n, generator=g, device=dev) / 64).to(torch.bfloat16))
        B.append((torch.randn(r, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
bd.bdlora_load_adapter(pool, 0, r, 1.0, A, B)
nrep = max(2, math.ceil(3 * (126 << 20) / (pool.m_loc * pool.k_loc * 2)))
Ws = [(torch.randn(pool.m_loc, pool.k_loc, generator=g, device=dev) / 64).to(torch.bfloat16) for _ in range(nrep)]
X = torch.randn(T, pool.k_loc, generator=g, device=dev).to(torch.bfloat16)
ids = torch.zeros(T, dtype=torch.int32, device=dev)
Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
L = 6
bufs = [torch.zeros(2048 * 32, dtype=torch.int64, device=dev) for _ in range(L)]
fwd = bd.bdlora_column_forward if par == bd.COLUMN else bd.bdlora_row_partial


def step(rec):
    for i in range(L):
        if rec:
            bd.bdlora_debug_trace(bufs[i])
        fwd(pool, X, Ws[i % nrep], ids, Y, ws)
    bd.bdlora_debug_trace(None)


step(False)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(gr, stream=s):
        step(True)
torch.cuda.current_stream().wait_stream(s)
gr.replay()
torch.cuda.synchronize()
for b in bufs:
    b.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.replay()
e1.record()
torch.cuda.synchronize()
info = bd.bdlora_last_launch_info()
print(f"{arch} {proj.name} TP{n} T={T} r={r}: {e0.elapsed_time(e1) * 1e3 / L:.2f} us per launch (traced)  {info}")
ts = [b.view(2048, 32).cpu().numpy() for b in bufs]
t0 = min(t[t[:, 0] > 1e12, 0].min() for t in ts)
slots = [0, 1, 13, 2, 14, 15, 3, 4, 9, 11, 12, 6, 7, 8]
print("launch CTAs " + " ".join(f"{s:>6d}" for s in slots) + "   max(7)")
for i, t in enumerate(ts):
    t = t[t[:, 0] > 1e12]
    row = []
    for c in slots:
        col = t[:, c]
        col = col[col > 1e12]
        row.append(f"{np.median((col - t0) / 1e3):6.2f}" if len(col) else "     -")
    e7 = t[:, 7][t[:, 7] > 1e12]
    print(f"{i:6d} {len(t):4d} " + " ".join(row) + f"   {((e7.max() - t0) / 1e3) if len(e7) else float('nan'):6.2f}")
