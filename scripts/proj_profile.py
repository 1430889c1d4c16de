"""One adapted projection of one TP rank (device-local forward), timed in a CUDA graph with the weights rotated
over >= 3 x L2, plus its launch record -- for ncu launch lists and A/B runs.
usage: python scripts/proj_profile.py ARCH PROJ_INDEX N T RANKS N_ADAPTERS IDS [REPS]
  ARCH llama-3.1-8b | llama-3.1-70b;  RANKS comma list (cycled over the slots);  IDS single | uniform | segments"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402
import synth  # noqa: E402

arch, k, n, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ranks_l = [int(x) for x in sys.argv[5].split(",")]
n_ad, ids_kind = int(sys.argv[6]), sys.argv[7]
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 20
dev = torch.device("cuda", 0)
proj = synth.arch_projections(arch)[k]
ranks = [ranks_l[a % len(ranks_l)] for a in range(n_ad)]
par = bd.COLUMN if proj.parallel == "column" else bd.ROW
# SHARDING=slora: the S-LoRA device-local phases (shrink + v-precomputed expand, no collective)
slora = os.environ.get("SHARDING", "bd") == "slora"
pool = bd.bdlora_create_pool(par, bd.SHARD_SLORA if slora else bd.SHARD_BD, n, 0, proj.d_in, proj.d_out, n_ad, max(ranks))
g = torch.Generator(device=dev)
g.manual_seed(0)
for a, r in enumerate(ranks):
    A, B = [], []
    for dj in proj.d_out:
        if proj.parallel == "column":
            A.append((torch.randn(proj.d_in, r, generator=g, device=dev) / 64).to(torch.bfloat16))
            B.append((torch.randn(r if slora else r // n, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
        else:
            A.append((torch.randn(proj.d_in, r if slora else r // n, generator=g, device=dev) / 64).to(torch.bfloat16))
            B.append((torch.randn(r, dj, generator=g, device=dev) / 8).to(torch.bfloat16))
    bd.bdlora_load_adapter(pool, a, r, 1.0, A, B)
nrep = max(2, math.ceil(3 * (126 << 20) / (pool.m_loc * pool.k_loc * 2)))
Ws = [(torch.randn(pool.m_loc, pool.k_loc, generator=g, device=dev) / 64).to(torch.bfloat16) for _ in range(nrep)]
X = torch.randn(T, pool.k_loc, generator=g, device=dev).to(torch.bfloat16)
rng = synth.rng_for(0, 3)
ids_np = {"single": lambda: np.zeros(T, np.int32), "uniform": lambda: synth.ids_uniform(rng, T, n_ad),
          "segments": lambda: synth.ids_segments(T, n_ad)}[ids_kind]()
ids = torch.from_numpy(ids_np).to(dev)
Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
if slora:
    vbuf = torch.zeros((n if par == bd.COLUMN else 1) * bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)


def fwd(i):
    W = Ws[i % nrep]
    if slora:
        only = os.environ.get("ONLY", "")  # shrink | expand: time one phase alone
        if only != "expand":
            bd.bdlora_lora_shrink(pool, X, ids, vbuf, ws)
        if only != "shrink":
            bd.bdlora_base_expand(pool, X, W, ids, vbuf, Y, ws)
    elif par == bd.COLUMN:
        bd.bdlora_column_forward(pool, X, W, ids, Y, ws)
    else:
        bd.bdlora_row_partial(pool, X, W, ids, Y, ws)


for i in range(3):
    fwd(i)
torch.cuda.synchronize()
if os.environ.get("EAGER"):
    for i in range(reps):
        fwd(i)
    torch.cuda.synchronize()
    print("eager launches done")
    sys.exit(0)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    for i in range(reps):
        fwd(i)
gr.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
gr.replay()
e.record()
torch.cuda.synchronize()
us = s.elapsed_time(e) / reps * 1e3
print(f"{arch} {proj.name} TP{n} T={T} ranks={ranks_l} adapters={n_ad} ids={ids_kind}: {us:.2f} us  "
      f"M={pool.m_loc} K={pool.k_loc} last={bd.bdlora_last_launch_info()} distinct={len(set(ids_np.tolist()) - {-1})}")

if os.environ.get("TRACE"):
    # per-CTA %globaltimer stamps of the last decode-kernel launch (slots: kernels_decode.cuh DEC_TRACE)
    tr = torch.zeros(1024 * 32, dtype=torch.int64, device=dev)
    bd.bdlora_debug_trace(tr)
    fwd(0)
    torch.cuda.synchronize()
    bd.bdlora_debug_trace(None)
    info = bd.bdlora_last_launch_info()
    t = tr.view(1024, 32).cpu().numpy()[: info["grid"]]
    t0 = t[:, 0].min()
    names = {0: "entry", 1: "ring0 issued", 2: "first mma", 13: "groups built", 3: "epi pre-wait", 14: "v staged",
             15: "lora done", 4: "acc ready", 9: "tc v read", 11: "cluster peers", 12: "pushed", 6: "reduced",
             7: "epi end", 8: "producer end"}
    for k, nm in names.items():
        col = t[:, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        c = (col - t0) / 1e3
        print(f"   {nm:14s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} us")
