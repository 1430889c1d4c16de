"""Timeline of a CUDA-graph chain of decode forwards (PDL on): each launch records per-CTA %globaltimer stamps
into its own trace buffer (the buffer pointer is baked into the captured launch), so the overlap between
consecutive projections is visible.  usage: python scripts/dec_chain_trace.py [M K rank]... (one projection
per triple, chained in order, repeated twice)"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402

dev = torch.device("cuda", 0)
args = [int(a) for a in sys.argv[1:]] or [6144 // 8, 4096, 2, 4096, 512, 2, 28672 // 8, 4096, 2, 4096, 1792, 2]
shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)]
nolora = bool(os.environ.get("NOLORA"))
projs = []
for M, K, r in shapes:
    pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, 1, 0, K, [M], 1, r)
    A = (torch.randn(K, r, device=dev) / math.sqrt(K)).to(torch.bfloat16)
    B = (torch.randn(r, M, device=dev) / 4).to(torch.bfloat16)
    bd.bdlora_load_adapter(pool, 0, r, 1.0, [A], [B])
    nrep = max(2, math.ceil(3 * (126 << 20) / (M * K * 2) / 4))
    Ws = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(nrep)]
    projs.append(dict(pool=pool, Ws=Ws, X=torch.randn(1, K, device=dev).to(torch.bfloat16),
                      Y=torch.empty(1, M, dtype=torch.bfloat16, device=dev), ws=bd.make_workspace(pool, 1)))
ids = torch.full((1,), -1 if nolora else 0, dtype=torch.int32, device=dev)
order = list(range(len(projs))) * 3
bufs = [torch.zeros(1024 * 32, dtype=torch.int64, device=dev) for _ in order]


def step(record):
    for k, pi in enumerate(order):
        p = projs[pi]
        if record:
            bd.bdlora_debug_trace(bufs[k])
        bd.bdlora_column_forward(p["pool"], p["X"], p["Ws"][k % len(p["Ws"])], ids, p["Y"], p["ws"])
    bd.bdlora_debug_trace(None)


step(False)
torch.cuda.synchronize()
for rec, name in ((False, "untraced"), (True, "traced")):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step(rec)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 1e3 / len(order):.2f} us per projection over {len(order)} launches")
t_all = [b.view(1024, 32).cpu().numpy() for b in bufs]
t0 = min(t[t[:, 0] > 0, 0].min() for t in t_all)
print("launch  M      CTAs  start(min)  ring0  mma0(med)  pre-wait(med)  acc(med)  v-smem  dot  peers  pushed  reduce  end(med)  end(max)   [us]")
for k, (pi, t) in enumerate(zip(order, t_all)):
    t = t[t[:, 0] > 0]
    f = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1e3  # noqa: E731
    print(f"{k:5d} {shapes[pi][0]:6d} {len(t):5d} {f(0).min():9.2f} {np.median(f(1)):7.2f} {np.median(f(2)):9.2f} "
          f"{np.median(f(3)):12.2f} {np.median(f(4)):9.2f} " +
          " ".join(f"{np.median(f(c)):6.2f}" if (t[:, c] > 0).any() else "     -" for c in (9, 10, 11, 12, 6)) +
          f" {np.median(f(7)):9.2f} {f(7).max():9.2f}")
