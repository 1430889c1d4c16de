"""Run one projection's device-local forward a few times (for ncu --set full captures).
usage: python scripts/profile_one.py M K T [rank] [phase: fwd|gemm]"""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402

M, K, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rank = int(sys.argv[4]) if len(sys.argv) > 4 else 16
phase = sys.argv[5] if len(sys.argv) > 5 else "fwd"
dev = torch.device("cuda", 0)
pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, 1, 0, K, [M], 1, rank)
A = (torch.randn(K, rank, device=dev) / math.sqrt(K)).to(torch.bfloat16)
B = (torch.randn(rank, M, device=dev) / 4).to(torch.bfloat16)
bd.bdlora_load_adapter(pool, 0, rank, 1.0, [A], [B])
W = torch.randn(M, K, device=dev).to(torch.bfloat16)
X = torch.randn(T, K, device=dev).to(torch.bfloat16)
ids = torch.zeros(T, dtype=torch.int32, device=dev)
Y = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
v = torch.zeros(bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)
bd.bdlora_lora_shrink(pool, X, ids, v, ws)
for i in range(4):
    if phase == "gemm":
        bd.bdlora_base_expand(pool, X, W, ids, v, Y, ws)
    else:
        bd.bdlora_column_forward(pool, X, W, ids, Y, ws)
torch.cuda.synchronize()
print("ok")
