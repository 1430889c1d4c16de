"""Compare the tensor-core shrink's v with numpy (debug)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd
import synth
from tests import _harness as H

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 37
proj = synth.arch_projections("llama-3.1-8b")[0]
case = H.make_case(100 + n * 10 + T, proj, "bd", n, T, ranks=[16, 16, 32])
for i in range(n):
    pool = H.make_pool(case, i)
    X, W, ids = H.device_inputs(case, i, dev)
    ws = bd.make_workspace(pool, T)
    v = torch.full((bd.bdlora_v_elems(pool, T),), float("nan"), dtype=torch.float32, device=dev)
    bd.bdlora_lora_shrink(pool, X, ids, v, ws)
    torch.cuda.synchronize()
    J, Rc = 3, 32 // n
    vv = v.cpu().numpy().reshape(T, J, Rc)
    bad = 0
    for t in range(T):
        a = int(case.ids[t])
        if a < 0:
            continue
        ad = case.adapters[a]
        rs = ad.rank // n
        for j in range(J):
            A = ad.A[j].f64[:, i * rs:(i + 1) * rs]
            ref = ad.scale * (case.X.f64[t] @ A)
            got = vv[t, j, :rs]
            if not np.allclose(got, ref, rtol=2e-3, atol=2e-3 * np.abs(ref).max()):
                bad += 1
                if bad < 6:
                    print(f"rank {i} t={t} a={a} j={j} got {got[:4]} ref {ref[:4]}")
    print(f"rank {i}: bad (t,j) pairs = {bad}")
    pool.close()

# identify which A column produced the wrong values (N from argv)
pool = H.make_pool(case, 0)
X, W, ids = H.device_inputs(case, 0, dev)
ws = bd.make_workspace(pool, T)
v = torch.full((bd.bdlora_v_elems(pool, T),), float("nan"), dtype=torch.float32, device=dev)
bd.bdlora_lora_shrink(pool, X, ids, v, ws)
torch.cuda.synchronize()
J, Rc = 3, 32 // n
vv = v.cpu().numpy().reshape(T, J, Rc)
t = 1
a = int(case.ids[t])
ad = case.adapters[a]
rs = ad.rank // n
cands = {}
for a2, ad2 in case.adapters.items():
    for j2 in range(J):
        for col in range(ad2.rank):
            cands[(a2, j2, col)] = ad2.scale * (case.X.f64[t] @ ad2.A[j2].f64[:, col])
for k in range(rs):
    g = vv[t, 2, k]
    best = min(cands.items(), key=lambda kv: abs(kv[1] / ad.scale * ad.scale - g))
    print("t", t, "a", a, "k", k, "got", g, "closest", best[0], best[1])
print("scales", {a2: ad2.scale for a2, ad2 in case.adapters.items()})
