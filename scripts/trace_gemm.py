"""Per-CTA timeline of one GEMM launch (bdlora_debug_trace): where does the time go?"""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402

dev = torch.device("cuda", 0)
M, K, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rank = 16
pool = bd.bdlora_create_pool(bd.COLUMN, bd.SHARD_BD, 1, 0, K, [M], 1, rank)
A = (torch.randn(K, rank, device=dev) / math.sqrt(K)).to(torch.bfloat16)
B = (torch.randn(rank, M, device=dev) / 4).to(torch.bfloat16)
bd.bdlora_load_adapter(pool, 0, rank, 1.0, [A], [B])
nrep = max(1, math.ceil(3 * (126 << 20) / (M * K * 2)))
Ws = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(nrep)]
X = torch.randn(T, K, device=dev).to(torch.bfloat16)
ids = torch.zeros(T, dtype=torch.int32, device=dev)
Y = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
ws = bd.make_workspace(pool, T)
v = torch.zeros(bd.bdlora_v_elems(pool, T), dtype=torch.float32, device=dev)
bd.bdlora_lora_shrink(pool, X, ids, v, ws)
tr = torch.zeros(148 * 32, dtype=torch.int64, device=dev)
for i in range(6):
    bd.bdlora_base_expand(pool, X, Ws[i % nrep], ids, v, Y, ws)
torch.cuda.synchronize()
fused = len(sys.argv) > 4 and sys.argv[4] == "fused"
shrink_only = len(sys.argv) > 4 and sys.argv[4] == "shrink"
bd.bdlora_debug_trace(tr)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
  s.record()
  if fused:
    bd.bdlora_column_forward(pool, X, Ws[rep % nrep], ids, Y, ws)
  elif shrink_only:
    bd.bdlora_lora_shrink(pool, X, ids, v, ws)
  else:
    bd.bdlora_base_expand(pool, X, Ws[rep % nrep], ids, v, Y, ws)
  e.record()
  torch.cuda.synchronize()
bd.bdlora_debug_trace(None)
t = tr.view(148, 32).cpu().numpy().astype("int64")
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
names = ["entry", "setup", "tma0", "data0", "mma_last", "epi_first", "epi_last", "epi_end", "exit", "fin_beg",
         "fin_end", "arrived", "part_beg", "shr_done", "v_ready", "lora1",
         "vseg_smem", "lr_done", "chunk_in", "v_staged", "lc_g", "lc_j", "lc_mask", "lc_vec"]
print(f"M={M} K={K} T={T} event time {s.elapsed_time(e)*1e3:.1f} us, CTAs {used.sum()}")
for k, nm in enumerate(names):
    if (t[:, k] <= 0).all():
        continue
    col = (t[:, k] - t0) / 1e3
    print(f"{nm:10s} min {col.min():7.2f}  med {sorted(col)[len(col)//2]:7.2f}  max {col.max():7.2f} us")
order = (t[:, 8] - t0).argsort()[::-1][:6]
print("slowest CTAs (us):", " ".join(names))
for c in order:
    print(c, " ".join(f"{(t[c, k] - t0) / 1e3 if t[c, k] > 0 else -1:6.2f}" for k in range(len(names))))
