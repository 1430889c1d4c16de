"""Multi-process host logic of the N > 1 path on CPU (gloo, world size 2, 127.0.0.1):
the NCCL unique-id bootstrap over torch.distributed, the bench's max-over-ranks timing reduction,
Alg. 1's row-layer all-reduce emulated with gloo over the oracle's per-rank partials
(sum of device partials == unsharded layer), and Alg. 2's all-gather of the column blocks
(rank-order concatenation == unsharded column output)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_23346_b200 as bd
        import bench
        import synth
        from oracle import lora as ol

        # 1) unique-id bootstrap: every rank ends up with rank 0's 128 bytes
        uid = bd.broadcast_unique_id()
        ids_all = [None] * world
        dist.all_gather_object(ids_all, uid)
        # 2) max over ranks
        mx = bench.reduce_max(float(rank + 1) * 1.5)
        # 3) Alg. 1 row layer: each rank its partial, all-reduce (sum) == unsharded oracle
        proj = synth.tiny_pair()[1]
        rng = synth.rng_for(3, 3)
        ads = {}
        for a in range(3):
            ad = synth.make_adapter(rng, proj, "bd", 8, world, 2.0)
            ads[a] = {"rank": 8, "scale": ad.scale, "A": [x.f64 for x in ad.A], "B": [x.f64 for x in ad.B]}
        X = synth.make_x(rng, 9, proj.d_in).f64
        W = synth.make_base(rng, proj).f64
        ids = np.array([0, 1, 2, -1, 0, 0, 1, 2, 2], np.int32)
        P = torch.from_numpy(ol.row_partial_bd(X, W, ads, ids, world, rank))
        dist.all_reduce(P)
        full = ol.row_layer(X, W, ads, ids, "bd", world)
        err = float(np.max(np.abs(P.numpy() - full)))
        # 4) Alg. 2: every rank's column block, all-gathered in rank order, is the unsharded
        #    column output [Y_0 | Y_1] (n_slices = 1) -- for one token (the in-place gather of
        #    bdlora_column_forward_gather) and for several
        col = synth.tiny_pair()[0]
        cads = {}
        for a in range(3):
            ad = synth.make_adapter(rng, col, "bd", 8, world, 2.0)
            cads[a] = {"rank": 8, "scale": ad.scale, "A": [x.f64 for x in ad.A], "B": [x.f64 for x in ad.B]}
        Wc = synth.make_base(rng, col).f64
        gerr = 0.0
        for T in (1, 9):
            Xc = synth.make_x(rng, T, col.d_in).f64
            cid = ids[:T]
            yfull = ol.column_layer(Xc, Wc, col.d_out, cads, cid, "bd", world)
            mine = torch.from_numpy(np.ascontiguousarray(ol.column_device_output(yfull, world, rank)))
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            gathered = torch.cat(parts, dim=1).numpy()
            gerr = max(gerr, float(np.max(np.abs(gathered - np.concatenate(yfull, axis=1)))))
        q.put((rank, uid, ids_all, mx, max(err, gerr)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_bootstrap_and_alg1_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort()
    (r0, uid0, all0, mx0, e0), (r1, uid1, all1, mx1, e1) = res
    assert uid0 == uid1 and len(uid0) == 128 and all0[0] == all0[1]
    assert mx0 == mx1 == 3.0
    assert e0 < 1e-12 and e1 < 1e-12
