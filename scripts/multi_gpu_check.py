"""N-GPU check of every collective path, one process per GPU (torchrun --nproc-per-node N):
bdlora_row_forward (NCCL bf16 all-reduce), bdlora_row_forward_fused (peer-memory all-reduce),
bdlora_column_forward_gather (Alg. 2 all-gather), slora_column_forward / slora_row_forward (S-LoRA's extra
all-gather / all-reduce), NFS-LoRA row; every output against the fp64 oracle, and the collective call log
(BD-LoRA: zero LoRA collectives, §8(d) step 9).  Rank 0 prints one JSON line.  Used by tests/test_gpu_multi.py."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_23346_b200 as bd  # noqa: E402
import synth  # noqa: E402
from oracle import lora as ol  # noqa: E402
from tests import _harness as H  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    comm = bd.comm_from_process_group(local)
    out = {"world": world, "checks": {}}

    def check(name, y, ref):
        ok, m, l1 = ol.within_tolerance(y.float().cpu().numpy().astype(np.float64), ref)
        out["checks"][name] = {"ok": bool(ok), "max_rel": m, "l1_rel": l1}

    p8 = synth.arch_projections("llama-3.1-8b")
    for T in (1, 9):
        # BD row: NCCL path and fused peer path
        case = H.make_case(7000 + T, p8[1], "bd", world, T, ranks=[16, 32])
        pool = H.make_pool(case, rank, device=local)
        X, W, ids = H.device_inputs(case, rank, dev)
        ws = bd.make_workspace(pool, T)
        ref = ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "bd", world)
        Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
        bd.bdlora_row_forward(pool, comm, X, W, ids, Y, ws)
        torch.cuda.synchronize()
        check(f"bd_row_nccl_T{T}", Y, ref)
        peer = bd.bdlora_peer_create(comm, 16 * pool.m_loc)
        Yf = torch.empty_like(Y)
        for _ in range(3):  # parity alternation
            bd.bdlora_row_forward_fused(pool, peer, X, W, ids, Yf, ws)
        torch.cuda.synchronize()
        check(f"bd_row_fused_T{T}", Yf, ref)
        out["checks"][f"bd_row_fused_T{T}"]["peer_error"] = bd.bdlora_peer_error(peer)
        g = [torch.empty_like(Yf) for _ in range(world)]
        dist.all_gather(g, Yf)
        out["checks"][f"bd_row_fused_T{T}"]["identical_on_all_ranks"] = all(torch.equal(g[0], x) for x in g)
        peer.close()
        pool.close()
        # Alg. 2 column + all-gather
        col = synth.tiny_pair()[0]
        case = H.make_case(7100 + T, col, "bd", world, T, ranks=[8, 16])
        pool = H.make_pool(case, rank, device=local)
        X, W, ids = H.device_inputs(case, rank, dev)
        Yg = torch.empty(T, pool.m_loc * world, dtype=torch.bfloat16, device=dev)
        bd.bdlora_column_forward_gather(pool, comm, X, W, ids, Yg, bd.make_workspace(pool, T))
        torch.cuda.synchronize()
        check(f"bd_alg2_gather_T{T}", Yg,
              ol.column_layer(case.X.f64, case.W.f64, col.d_out, case.oracle_adapters(), case.ids, "bd", world)[0])
        pool.close()
        # S-LoRA column and row
        for pi, fn in ((0, bd.slora_column_forward), (1, bd.slora_row_forward)):
            proj = p8[pi]
            case = H.make_case(7200 + 10 * pi + T, proj, "slora", world, T, ranks=[16, 32])
            pool = H.make_pool(case, rank, device=local)
            X, W, ids = H.device_inputs(case, rank, dev)
            Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
            fn(pool, comm, X, W, ids, Y, bd.make_workspace(pool, T))
            torch.cuda.synchronize()
            ads = case.oracle_adapters()
            if proj.parallel == "column":
                ref = ol.column_device_output(ol.column_layer(case.X.f64, case.W.f64, proj.d_out, ads, case.ids, "slora",
                                                              world), world, rank)
            else:
                ref = ol.row_layer(case.X.f64, case.W.f64, ads, case.ids, "slora", world)
            check(f"slora_{proj.parallel}_T{T}", Y, ref)
            pool.close()
        # NFS row
        case = H.make_case(7300 + T, p8[3], "nfs", world, T, ranks=[16])
        pool = H.make_pool(case, rank, device=local)
        X, W, ids = H.device_inputs(case, rank, dev)
        Y = torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev)
        bd.nfs_row_forward(pool, comm, X, W, ids, Y, bd.make_workspace(pool, T))
        torch.cuda.synchronize()
        check(f"nfs_row_T{T}", Y, ol.row_layer(case.X.f64, case.W.f64, case.oracle_adapters(), case.ids, "nfs", world))
        pool.close()
    out["comm_stats"] = bd.bdlora_comm_stats(comm)
    comm.close()
    dist.barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
