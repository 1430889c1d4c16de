"""Debug the tensor-core expand: W = 0 isolates the LoRA term."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd
import synth
from oracle import lora as ol
from tests import _harness as H

dev = torch.device("cuda", 0)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 37
proj = synth.Projection("p", "column", 256, (256,))
case = H.make_case(7, proj, "bd", 1, T, ranks=[16], ids=np.zeros(T, np.int32), w_zero=True)
pool = H.make_pool(case, 0)
X, W, ids = H.device_inputs(case, 0, dev)
Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
bd.bdlora_column_forward(pool, X, W, ids, Y, bd.make_workspace(pool, T))
torch.cuda.synchronize()
y = Y.float().cpu().numpy()
ref = ol.column_layer(case.X.f64, case.W.f64, proj.d_out, case.oracle_adapters(), case.ids, "bd", 1)[0]
print("max|y|", np.abs(y).max(), "max|ref|", np.abs(ref).max())
print("y[0,:6]  ", y[0, :6])
print("ref[0,:6]", ref[0, :6])
print("y[1,:6]  ", y[1, :6])
print("ref[1,:6]", ref[1, :6])
# least squares ratio
r = (y * ref).sum() / (ref * ref).sum()
print("ratio", r, "resid", np.abs(y - r * ref).max())
# check transposition hypotheses: does y match ref with rows/cols permuted within 8-blocks?
for name, cand in [("ref", ref)]:
    print(name, ol.within_tolerance(y, cand))
# per column / per token error pattern
err = np.abs(y - ref)
print("err per token (first 20):", np.round(err.max(axis=1)[:20], 3))
print("err per col block of 8:", np.round(err.max(axis=0).reshape(-1, 8).max(axis=1)[:32], 3))
