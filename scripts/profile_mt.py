"""configs[4] single projection on one emulated rank (for ncu / tracing):
python scripts/profile_mt.py [proj_index 0..3] [tp] [T] [trace]"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402
import synth  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 64
trace = len(sys.argv) > 4 and sys.argv[4] == "trace"
dev = torch.device("cuda", 0)
proj = synth.arch_projections("llama-3.1-70b")[k]
ranks = [[8, 16, 32, 64, 128][a % 5] for a in range(128)]
par = bd.COLUMN if proj.parallel == "column" else bd.ROW
pool = bd.bdlora_create_pool(par, bd.SHARD_BD, n, 0, proj.d_in, proj.d_out, 128, 128)
g = torch.Generator(device=dev)
g.manual_seed(0)
for a, r in enumerate(ranks):
    A, B = [], []
    for dj in proj.d_out:
        if proj.parallel == "column":
            A.append((torch.randn(proj.d_in, r, generator=g, device=dev) / 64).to(torch.bfloat16))
            B.append((torch.randn(r // n, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
        else:
            A.append((torch.randn(proj.d_in, r // n, generator=g, device=dev) / 64).to(torch.bfloat16))
            B.append((torch.randn(r, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
    bd.bdlora_load_adapter(pool, a, r, 1.0, A, B)
W = (torch.randn(pool.m_loc, pool.k_loc, generator=g, device=dev) / 64).to(torch.bfloat16)
X = torch.randn(T, pool.k_loc, generator=g, device=dev).to(torch.bfloat16)
ids = torch.from_numpy(synth.ids_uniform(synth.rng_for(0, 3), T, 128)).to(dev)
Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
fwd = (lambda: bd.bdlora_column_forward(pool, X, W, ids, Y, ws)) if par == bd.COLUMN else \
      (lambda: bd.bdlora_row_partial(pool, X, W, ids, Y, ws))
for _ in range(3):
    fwd()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    fwd()
e.record()
torch.cuda.synchronize()
print(f"{proj.name} TP{n} T={T}: {s.elapsed_time(e) / 10 * 1e3:.1f} us/call (eager)")
if trace:
    tr = torch.zeros(148 * 32, dtype=torch.int64, device=dev)
    bd.bdlora_debug_trace(tr)
    fwd()
    torch.cuda.synchronize()
    bd.bdlora_debug_trace(None)
    t = tr.view(148, 32).cpu().numpy().astype("int64")
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = ["entry", "setup", "tma0", "data0", "mma_last", "epi_first", "epi_last", "epi_end", "exit"] + [""] * 10 + \
        ["lx_pre", "p0_meta", "p0_empty", "p0_issued", "p0_landed", "p1_meta", "p1_empty", "p1_issued", "p1_landed",
         "p0_a_issued"]
    for kk, nm in enumerate(names):
        if not nm or (t[:, kk] <= 0).all():
            continue
        col = (t[:, kk][t[:, kk] > 0] - t0) / 1e3
        print(f"{nm:10s} min {col.min():8.2f} med {np.median(col):8.2f} max {col.max():8.2f}")

if len(sys.argv) > 4 and sys.argv[4] == "parts":
    # component timing: shrink alone, GEMM + expand alone, GEMM without LoRA
    v = torch.zeros(bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)
    nids = -torch.ones(T, dtype=torch.int32, device=dev)

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps * 1e3

    print(f"  shrink (route + tc shrink): {timeit(lambda: bd.bdlora_lora_shrink(pool, X, ids, v, ws)):.1f} us")
    print(f"  base_expand (GEMM + expand): {timeit(lambda: bd.bdlora_base_expand(pool, X, W, ids, v, Y, ws)):.1f} us")
    print(f"  base_expand, ids = -1:      {timeit(lambda: bd.bdlora_base_expand(pool, X, W, nids, v, Y, ws)):.1f} us")
    print(f"  forward, ids = -1:          {timeit(lambda: fwd_nolora()) if False else 0:.1f}")
