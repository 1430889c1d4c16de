"""Per-CTA %globaltimer trace of one multi-adapter decode expand (lora 4) launch: S-LoRA or BD pool, one TP rank,
after its shrink.  Prints the slowest CTAs' stamps (us from the launch's first stamp).
usage: python scripts/mt_trace.py ARCH PROJ_INDEX N T RANKS N_ADAPTERS [slora|bd]"""
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
n_ad = int(sys.argv[6])
slora = (sys.argv[7] if len(sys.argv) > 7 else "slora") == "slora"
dev = torch.device("cuda", 0)
proj = synth.arch_projections(arch)[k]
ranks = [ranks_l[a % len(ranks_l)] for a in range(n_ad)]
par = bd.COLUMN if proj.parallel == "column" else bd.ROW
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
W = (torch.randn(pool.m_loc, pool.k_loc, generator=g, device=dev) / 64).to(torch.bfloat16)
X = torch.randn(T, pool.k_loc, generator=g, device=dev).to(torch.bfloat16)
ids = torch.from_numpy(synth.ids_uniform(synth.rng_for(0, 3), T, n_ad)).to(dev)
Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
v = torch.zeros((n if par == bd.COLUMN else 1) * bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)
tr = torch.zeros(2048 * 32, dtype=torch.int64, device=dev)
for it in range(3):
    bd.bdlora_lora_shrink(pool, X, ids, v, ws)
    if it == 2:
        bd.bdlora_debug_trace(tr)
    bd.bdlora_base_expand(pool, X, W, ids, v, Y, ws)
    bd.bdlora_debug_trace(None)
torch.cuda.synchronize()
info = bd.bdlora_last_launch_info()
grid = info["grid"]
t = tr[: grid * 32].view(grid, 32).cpu().numpy().astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
t[:, 31] = 0
rel = np.where(t > 1e12, (t - t0) / 1e3, np.nan)
end = np.nanmax(rel, axis=1)
order = np.argsort(-end)
np.set_printoptions(linewidth=250, precision=1, suppress=True)
print(info)
print("slots: 0 start 1 setup 13 groups 2 first-full 14 mt-start 16+2c chunk c staged 17+2c chunk c MMA 15 mt-end 3 4 acc 7 end")
for c in list(order[:6]) + list(order[-2:]):
    row = rel[c]
    print(f"cta {c:4d} end {end[c]:7.2f}  " + " ".join(f"{s}:{row[s]:.1f}" for s in range(32) if not np.isnan(row[s])))
