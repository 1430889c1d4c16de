#!/usr/bin/env python
"""bench.py -- BD-LoRA tensor-parallel multi-adapter LoRA layer on B200 (arXiv 2510.23346).

A "step" = one pass of the whole hot path over one batch: the four adapted projections of one
Llama decoder layer -- QKV (column), O (row), gate_up (column), down (row) -- each running
shrink (X A[a]) -> base GEMM + fused expand/add (matmul_1..6, add_1/2), plus the base model's
own all-reduce after each row layer when N > 1 (the ONLY collective of BD-LoRA).

Default workload (N=1) = BASELINE.json configs[1]: Llama-3.1-8B layer shapes, decode batch 1,
rank 16, TP = N.  Other configs are parity-test cases; `--workload` selects them for exploration.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl reference]`; for N>1 the
driver launches it under torchrun (one rank per GPU; TP degree = N).  Rank 0 prints ONE JSON line.
Timing: W eager warm-up steps, then the K timed steps captured in one CUDA graph and replayed once,
bracketed by barrier + cuda.synchronize, CUDA events on the launching stream, max over ranks.
Per-step weights exceed the 126 MB L2 (or rotate over >= 3 x L2 of replicas), so no L2 flush is
needed between steps (said in `config.l2`).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

BASELINE_METRIC = "LoRA-layer µs & tokens/s vs S-LoRA at TP=1/2/4/8; % of HBM/tensor roofline"
L2_BYTES = 126 * 1024 * 1024

WORKLOADS = {
    # configs[1] -- the bench line
    "8b-decode-bs1-r16": dict(arch="llama-3.1-8b", T=1, ranks=[16], n_adapters=1, ids="single",
                              desc="configs[1]: Llama-3.1-8B layer shapes (h=4096, ff=14336, GQA 32/8), decode batch 1, rank 16"),
    # configs[1] variants: 64 resident adapters with 1 active; the paper's parameter-matched pairing
    # (BD 2r vs S-LoRA r, 0.86x the parameters)
    "8b-decode-bs1-r16-64resident": dict(arch="llama-3.1-8b", T=1, ranks=[16], n_adapters=64, ids="single",
                                         desc="configs[1] variant: 64 resident rank-16 adapters, 1 active, decode batch 1"),
    "8b-decode-bs1-bd32-vs-slora16": dict(arch="llama-3.1-8b", T=1, ranks=[32], slora_ranks=[16], n_adapters=1,
                                          ids="single",
                                          desc="configs[1] parameter-matched pair: BD-LoRA rank 32 vs S-LoRA rank 16 "
                                               "(P:801-805), decode batch 1"),
    # configs[3]
    "70b-decode-bs64-r32": dict(arch="llama-3.1-70b", T=64, ranks=[32], n_adapters=1, ids="single",
                                desc="configs[3]: Llama-3.1-70B layer shapes, decode batch 64, rank 32"),
    "70b-decode-bs1-r32": dict(arch="llama-3.1-70b", T=1, ranks=[32], n_adapters=1, ids="single",
                               desc="configs[3]: Llama-3.1-70B layer shapes, decode batch 1, rank 32"),
    # configs[4] and its id-distribution variants (every request a different adapter)
    "70b-multitenant": dict(arch="llama-3.1-70b", T=64, ranks=[8, 16, 32, 64, 128], n_adapters=128, ids="uniform",
                            desc="configs[4]: 64 requests over 128 resident adapters (r in 8..128), Llama-3.1-70B shapes"),
    "70b-multitenant-zipf": dict(arch="llama-3.1-70b", T=64, ranks=[8, 16, 32, 64, 128], n_adapters=128, ids="zipf",
                                 desc="configs[4] variant: Zipf(1.0) adapter popularity over 128 resident adapters"),
    "70b-multitenant-distinct": dict(arch="llama-3.1-70b", T=64, ranks=[8, 16, 32, 64, 128], n_adapters=128,
                                     ids="distinct",
                                     desc="configs[4] variant: all 64 requests use different adapters (P:730-731)"),
}
# configs[2]: the rank sweep, one request (1 segment) and 8 requests x 128 tokens over 8 adapters (8 segments)
for _r in (8, 32, 64, 128, 256):
    WORKLOADS[f"8b-prefill-1024-r{_r}"] = dict(
        arch="llama-3.1-8b", T=1024, ranks=[_r], n_adapters=1, ids="single",
        desc=f"configs[2]: Llama-3.1-8B prefill 1024 tokens, rank {_r}, one segment")
    WORKLOADS[f"8b-prefill-8x128-r{_r}"] = dict(
        arch="llama-3.1-8b", T=1024, ranks=[_r], n_adapters=8, ids="segments", n_requests=8,
        desc=f"configs[2]: Llama-3.1-8B prefill, 8 requests x 128 tokens over 8 rank-{_r} adapters (8 segments)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ============================================================================ helpers

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def reduce_max(x: float, device=None) -> float:
    """Max over ranks of a host float (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ============================================================================ layer construction

class Projection:
    """One adapted projection on one device: base weight replicas, pool(s), buffers.

    Weight replicas: at least `replicas` (the layer's count) and at least 3 x L2 of this projection's own
    bytes, so the projection timed ALONE also streams its weights from HBM."""

    def __init__(self, bd, torch, proj, sharding, n, i, ranks_of_slots, scale_of_slots, T, dev, replicas, gen,
                 w_replicas=None, keep_slots=()):
        self.proj, self.sharding, self.n, self.i = proj, sharding, n, i
        par = bd.COLUMN if proj.parallel == "column" else bd.ROW
        sh = {"bd": bd.SHARD_BD, "slora": bd.SHARD_SLORA, "nfs": bd.SHARD_NFS}[sharding]
        cap = len(ranks_of_slots)
        self.pool = bd.bdlora_create_pool(par, sh, n, i, proj.d_in, proj.d_out, cap, max(ranks_of_slots), device=dev.index)
        k, m = self.pool.k_loc, self.pool.m_loc
        self.k, self.m = k, m
        self.kept = {}  # slot -> (rank, scale, A list, B list) in the load format (bench self-check)
        # adapters: factors generated in the load format on the device (synthetic, seeded), then sliced
        for a, (r, s) in enumerate(zip(ranks_of_slots, scale_of_slots)):
            A, B = [], []
            for dj in proj.d_out:
                if proj.parallel == "column":
                    A.append((torch.randn(proj.d_in, r, generator=gen, device=dev) / math.sqrt(proj.d_in)).to(torch.bfloat16))
                    rb = r // n if sharding == "bd" else r
                    B.append((torch.randn(rb, dj, generator=gen, device=dev) / (s * math.sqrt(r / n))).to(torch.bfloat16))
                else:
                    ra = r // n if sharding == "bd" else r
                    A.append((torch.randn(proj.d_in, ra, generator=gen, device=dev) / math.sqrt(proj.d_in)).to(torch.bfloat16))
                    B.append((torch.randn(r, dj, generator=gen, device=dev) / (s * math.sqrt(r / n))).to(torch.bfloat16))
            bd.bdlora_load_adapter(self.pool, a, r, s, A, B)
            if a in keep_slots:
                self.kept[a] = (r, s, A, B)
            del A, B
        pbytes = 2 * k * m
        self.n_reps = max(replicas, math.ceil(3 * L2_BYTES / pbytes))
        if w_replicas is None:
            w_replicas = [(torch.randn(m, k, generator=gen, device=dev) / math.sqrt(proj.d_in)).to(torch.bfloat16)
                          for _ in range(self.n_reps)]
        self.W = w_replicas
        self.X = (torch.randn(T, k, generator=gen, device=dev)).to(torch.bfloat16)
        self.Y = torch.empty(T, m, dtype=torch.bfloat16, device=dev)
        self.ws = bd.make_workspace(self.pool, T)

    peer = None  # fused row all-reduce peer group (N > 1, decode batches): bdlora_row_forward_fused

    def run(self, bd, comm, ids, rep, X=None, Y=None):
        X = self.X if X is None else X
        Y = self.Y if Y is None else Y
        W = self.W[rep % len(self.W)]
        if self.sharding == "bd":
            if self.proj.parallel == "column":
                bd.bdlora_column_forward(self.pool, X, W, ids, Y, self.ws)
            elif self.peer is not None:
                bd.bdlora_row_forward_fused(self.pool, self.peer, X, W, ids, Y, self.ws)
            else:
                bd.bdlora_row_forward(self.pool, comm, X, W, ids, Y, self.ws)
        elif self.sharding == "nfs":
            if self.proj.parallel == "column":
                bd.nfs_column_forward(self.pool, X, W, ids, Y, self.ws)
            else:
                bd.nfs_row_forward(self.pool, comm, X, W, ids, Y, self.ws)
        else:
            if self.proj.parallel == "column":
                bd.slora_column_forward(self.pool, comm, X, W, ids, Y, self.ws)
            else:
                bd.slora_row_forward(self.pool, comm, X, W, ids, Y, self.ws)

    def close(self):
        if self.peer is not None:
            self.peer.close()
        self.pool.close()


def make_ids(torch, wl, T, seed, dev):
    import numpy as np

    import synth

    rng = synth.rng_for(seed, 3)
    if wl["ids"] == "single":
        ids = np.zeros(T, np.int32)
    elif wl["ids"] == "uniform":
        ids = synth.ids_uniform(rng, T, wl["n_adapters"])
    elif wl["ids"] == "zipf":
        ids = synth.ids_zipf(rng, T, wl["n_adapters"])
    elif wl["ids"] == "distinct":
        ids = synth.ids_distinct(rng, T, wl["n_adapters"])
    elif wl["ids"] == "segments":
        ids = synth.ids_segments(T, wl["n_requests"])
    else:
        raise ValueError(wl["ids"])
    return torch.from_numpy(ids).to(dev), ids


def slot_ranks(wl, sharding="bd"):
    ranks = wl.get("slora_ranks", wl["ranks"]) if sharding == "slora" else wl["ranks"]
    return [ranks[k % len(ranks)] for k in range(wl["n_adapters"])]


def build_layer(bd, torch, wl, sharding, n, i, dev, seed=0, replicas=None, share_w=None, keep_slots=()):
    import synth

    projs = synth.arch_projections(wl["arch"])
    T = wl["T"]
    ranks = slot_ranks(wl, sharding)
    scales = [synth.rs_scale(16.0, r, n, sharding) for r in ranks]
    from paper_2510_23346_b200 import accounting as acc

    per_step = sum(acc.proj_bytes(p.parallel, sharding, p.d_in, p.d_out, n, T, []) for p in projs)
    if replicas is None:
        replicas = max(1, math.ceil(3 * L2_BYTES / per_step))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + seed)
    layer = []
    for k, p in enumerate(projs):
        wr = share_w[k].W if share_w is not None else None
        layer.append(Projection(bd, torch, p, sharding, n, i, ranks, scales, T, dev, replicas, gen, w_replicas=wr,
                                keep_slots=keep_slots))
    return layer, replicas


def algorithmic(wl, sharding, n, ids_np):
    """Per-projection algorithmic bytes and FLOPs of one step on one device."""
    import synth
    from paper_2510_23346_b200 import accounting as acc

    ranks = slot_ranks(wl, sharding)
    touched = sorted(set(int(a) for a in ids_np.tolist() if a >= 0))
    rt = [ranks[a] for a in touched]
    tok = [ranks[a] if a >= 0 else 0 for a in ids_np.tolist()]
    out = {}
    for p in synth.arch_projections(wl["arch"]):
        out[p.name] = (acc.proj_bytes(p.parallel, sharding, p.d_in, p.d_out, n, wl["T"], rt),
                       acc.proj_flops(p.parallel, sharding, p.d_in, p.d_out, n, tok))
    return out


# ============================================================================ timing

def graph_time(torch, body, steps, barrier, use_graph=True):
    """Capture `steps` calls of body(k) in ONE CUDA graph, replay once (warm), then time one replay with
    CUDA events on the launching stream, bracketed by barrier + synchronize.  Returns total ms."""
    g = None
    if use_graph:
        s = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(s)
        with torch.cuda.stream(side):
            body(0)  # warm the capture stream
        s.wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(steps):
                body(k)
        g.replay()
        torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    start.record()
    if g is not None:
        g.replay()
    else:
        for k in range(steps):
            body(k)
    end.record()
    torch.cuda.synchronize()
    barrier()
    return start.elapsed_time(end)


def time_layer(bd, torch, layer, comm, ids, steps, warmup, use_graph, barrier):
    """Returns (total_ms of `steps` layer steps, per-projection isolated us, launches per step)."""
    l0 = bd.bdlora_kernel_launches()
    for p in layer:
        p.run(bd, comm, ids, 0)
    launches = bd.bdlora_kernel_launches() - l0
    for w in range(max(0, warmup - 1)):
        for p in layer:
            p.run(bd, comm, ids, w + 1)
    torch.cuda.synchronize()

    def step(k):
        for p in layer:
            p.run(bd, comm, ids, k)

    total = graph_time(torch, step, steps, barrier, use_graph)
    # each projection alone, same launch configuration, weights rotated like in the step
    per = []
    for p in layer:
        ms = graph_time(torch, lambda k, p=p: p.run(bd, comm, ids, k), steps, barrier, use_graph)
        per.append(ms / steps * 1e3)
    return total, per, launches
def time_e2e(bd, torch, layer, comm, ids_np, steps, warmup, barrier):
    """Same step through the public API with HOST buffers: every step uploads its inputs (every
    projection's activations + the ids, packed) from pinned host memory, runs the four forwards and
    downloads the four outputs -- all inside the timed region (graph-captured).  As a server does, the
    transfers run on a copy stream, double-buffered: step k+1's upload overlaps step k's forwards and step
    k's download overlaps step k+1's.  Returns (ms, h2d bytes, d2h bytes) per the whole run."""
    dev = layer[0].X.device
    T = layer[0].X.shape[0]
    xs = [p.X.numel() for p in layer]
    ys = [p.Y.numel() for p in layer]
    nin = sum(xs) + 2 * T  # bf16 elements; ids (int32) packed as 2 bf16 slots each
    h_in = [torch.empty(nin, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    d_in = [torch.empty(nin, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    h_out = [torch.empty(sum(ys), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    d_out = [torch.empty(sum(ys), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    views = []
    for b in range(2):
        off, dx = 0, []
        for p, n in zip(layer, xs):
            h_in[b][off:off + n].copy_(p.X.reshape(-1).cpu())
            dx.append(d_in[b][off:off + n].view(p.X.shape))
            off += n
        h_in[b][off:off + 2 * T].view(torch.int32).copy_(torch.from_numpy(ids_np.copy()))
        did = d_in[b][off:off + 2 * T].view(torch.int32)
        off, dy = 0, []
        for p, n in zip(layer, ys):
            dy.append(d_out[b][off:off + n].view(p.Y.shape))
            off += n
        views.append((dx, did, dy))
    copy = torch.cuda.Stream()
    ev = {name: [torch.cuda.Event() for _ in range(2)] for name in ("in_ready", "in_free", "out_ready", "out_free")}

    def run(nsteps):
        # the stream current at CALL time: under torch.cuda.graph that is the capture stream, so the copy
        # stream forks from it and joins back -- every H2D / D2H copy and event wait is captured in the graph
        compute = torch.cuda.current_stream()
        copy.wait_stream(compute)  # fork
        for k in range(nsteps):
            b = k % 2
            dx, did, dy = views[b]
            with torch.cuda.stream(copy):
                if k >= 2:
                    copy.wait_event(ev["in_free"][b])
                d_in[b].copy_(h_in[b], non_blocking=True)
                ev["in_ready"][b].record(copy)
            compute.wait_event(ev["in_ready"][b])
            if k >= 2:
                compute.wait_event(ev["out_free"][b])
            for p, x, y in zip(layer, dx, dy):
                p.run(bd, comm, did, k, X=x, Y=y)
            ev["in_free"][b].record(compute)
            ev["out_ready"][b].record(compute)
            with torch.cuda.stream(copy):
                copy.wait_event(ev["out_ready"][b])
                h_out[b].copy_(d_out[b], non_blocking=True)
                ev["out_free"][b].record(copy)
        compute.wait_stream(copy)  # join

    run(max(warmup, 2))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g):
        run(steps)
    census = graph_census(g)
    g.instantiate()
    g.replay()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    start.record()
    g.replay()
    end.record()
    torch.cuda.synchronize()
    barrier()
    return start.elapsed_time(end), nin * 2, sum(ys) * 2, census


def graph_census(g):
    """Node types of a captured CUDA graph (proves the e2e graph holds the per-step H2D/D2H copies)."""
    try:
        from cuda.bindings import runtime as rt

        h = rt.cudaGraph_t(init_value=int(g.raw_cuda_graph()))
        err, _, n = rt.cudaGraphGetNodes(h, 0)
        err, nodes, n = rt.cudaGraphGetNodes(h, n)
        out = {}
        for nd in nodes[:n]:
            e2, ty = rt.cudaGraphNodeGetType(nd)
            name = str(ty).split(".")[-1].replace("cudaGraphNodeType", "").lower()
            out[name] = out.get(name, 0) + 1
        return out
    except Exception as e:  # pragma: no cover
        return {"error": repr(e)[:200]}


# ============================================================================ oracle legs

def oracle_step_sample(wl, seed=0):
    """Build the bounded oracle sample: one token through the full (unsharded) layer with its adapter."""
    import numpy as np

    import synth

    rng = synth.rng_for(seed, 11)
    ranks = slot_ranks(wl)
    r = ranks[0]
    sample = []
    for p in synth.arch_projections(wl["arch"]):
        W = synth.make_base(rng, p)
        ad = synth.make_adapter(rng, p, "bd", r, 1, synth.rs_scale(16.0, r, 1, "bd"))
        ads = {0: {"rank": r, "scale": ad.scale, "A": [a.f64 for a in ad.A], "B": [b.f64 for b in ad.B]}}
        X = synth.make_x(rng, 1, p.d_in)
        sample.append((p, W.f64, ads, X.f64))
    return sample, np.zeros(1, np.int32)


def run_oracle_step(sample, ids):
    from oracle import lora as ol

    for p, W, ads, X in sample:
        if p.parallel == "column":
            ol.column_layer(X, W, p.d_out, ads, ids, "bd", 1)
        else:
            ol.row_layer(X, W, ads, ids, "bd", 1)


def oracle_check_bench_output(bd, torch, layer, ids, ids_np, n_samples=24, seed=0):
    """Part of the cpu_baseline leg (the oracle runs only there): re-run each projection of the timed BD
    layer once, eagerly, in the bench's own launch configuration (pools, T, workspace, replica 0), and
    compare `n_samples` sampled outputs per projection with the fp64 oracle computed one by one
    (oracle.lora_layer_sampled).  N = 1 only, where the device output is the unsharded layer and the
    load format of every factor is its dense form.  Returns the worst errors seen."""
    import numpy as np

    from oracle import lora as ol

    rng = np.random.default_rng(seed)
    worst_rel, n_tot, ok = 0.0, 0, True
    per = {}
    for p in layer:
        p.run(bd, None, ids, 0)
        torch.cuda.synchronize()
        T, M = p.Y.shape
        X = p.X.float().cpu().numpy().astype(np.float64)
        ts = rng.integers(0, T, size=n_samples)
        cs = rng.integers(0, M, size=n_samples)
        got = p.Y[torch.from_numpy(ts).to(p.Y.device), torch.from_numpy(cs).to(p.Y.device)].float().cpu().numpy()
        ref = np.empty(n_samples)
        col0 = np.cumsum([0] + list(p.proj.d_out))
        for q, (t, c) in enumerate(zip(ts.tolist(), cs.tolist())):
            j = int(np.searchsorted(col0, c, side="right") - 1)
            wcol = p.W[0][c].float().cpu().numpy().astype(np.float64)[:, None]  # W[:, c] (paper orientation)
            ads = {}
            a = int(ids_np[t])
            if a >= 0:
                r, sc, A, B = p.kept[a]
                Aj = A[j].float().cpu().numpy().astype(np.float64)
                Bc = B[j][:, c - col0[j]].float().cpu().numpy().astype(np.float64)[:, None]
                ads[a] = (sc, Aj, Bc)
            ref[q] = ol.lora_layer_sampled(X, wcol, ads, ids_np, [(t, 0)])[0]
        good, m, l1 = ol.within_tolerance(got, ref)
        ok = ok and good
        worst_rel = max(worst_rel, m)
        n_tot += n_samples
        per[p.proj.name] = {"max_rel": m, "l1_rel": l1, "ok": good}
    return {"ok": ok, "samples": n_tot, "worst_max_rel": worst_rel, "per_projection": per,
            "tolerance": "max|y-ref| <= 2e-2 max|ref|, sum|y-ref|/sum|ref| <= 5e-3 (SURVEY 8(c) step 7)"}


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count()


def cpu_baseline(wl, max_steps=3, budget_s=25.0):
    sample, ids = oracle_step_sample(wl)
    run_oracle_step(sample, ids)  # warm
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (time.perf_counter() - t0) < budget_s:
        run_oracle_step(sample, ids)
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": 1.0 / dt, "unit": "tokens/s", "cores": cores_used(), "kind": "oracle",
            "sample": f"{n} step(s) of 1 token through the full unsharded {wl['arch']} layer (QKV+O+gate_up+down, "
                      f"r={slot_ranks(wl)[0]}, materialised dW, numpy fp64/OpenBLAS); {dt * 1e3:.0f} ms/token"}


def run_reference(args, wl):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    sample, ids = oracle_step_sample(wl)
    for _ in range(args.warmup):
        run_oracle_step(sample, ids)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run_oracle_step(sample, ids)
    dt = (time.perf_counter() - t0) / args.steps
    v = 1.0 / dt  # one token per step
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["desc"] + " -- bounded sample: 1 token per step through the unsharded layer",
                       "tp": 1, "T_per_step": 1},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores_used(), "kind": "oracle",
                             "sample": "1 token per step, full unsharded layer, numpy fp64"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ============================================================================ main (ours)

def run_ours(args, wl):
    import torch

    world, rank, local = dist_env()
    n = world
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

        def barrier():
            dist.barrier()
    else:
        def barrier():
            pass

    import paper_2510_23346_b200 as bd

    bd.bdlora_device_check(local)
    comm = bd.comm_from_process_group(local) if world > 1 else None
    T = wl["T"]
    ids, ids_np = make_ids(torch, wl, T, 0, dev)
    hbm_peak, tf_peak, tf_sus, peak_src = measured_peaks()

    # ---------------- BD-LoRA layer (the step) ----------------
    keep = sorted(set(int(a) for a in ids_np.tolist() if a >= 0)) if world == 1 else ()
    layer, reps = build_layer(bd, torch, wl, "bd", n, rank, dev, keep_slots=keep)
    fused_ar = world > 1 and T <= 16 and not args.no_fused_ar
    if fused_ar:  # the row layers' base all-reduce fused into the decode kernel over NVLink peer memory
        for p in layer:
            if p.proj.parallel == "row":
                p.peer = bd.bdlora_peer_create(comm, T * p.m)
    clocks = ClockSampler(local)
    clocks.start()
    total_ms, per, launches = time_layer(bd, torch, layer, comm, ids, args.steps, args.warmup, not args.no_graph, barrier)
    clk = clocks.stop()
    total_ms = reduce_max(total_ms, dev)
    ms_step = total_ms / args.steps
    value = T / (ms_step * 1e-3)
    names = [p.proj.name for p in layer]
    proj_us = dict(zip(names, per))
    alg = algorithmic(wl, "bd", n, ids_np)

    # dominant kernel = the base GEMM + fused expand of the projection with the most time
    dom = max(names, key=lambda nm: proj_us[nm])
    dom_mean_us = per[names.index(dom)]
    dom_bytes, dom_flops = alg[dom]
    bound = "hbm" if dom_flops / dom_bytes < (tf_peak * 1e12) / (hbm_peak * 1e9) else "tensor"
    if bound == "hbm":
        achieved = dom_bytes / (dom_mean_us * 1e-6) / 1e9
        peak = hbm_peak
        unit = "GB/s"
    else:
        achieved = dom_flops / (dom_mean_us * 1e-6) / 1e12
        peak = tf_peak
        unit = "TFLOP/s"
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tr = json.load(f)
            traffic = tr.get(args.workload, {}).get(f"tp{n}", {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                "traffic": traffic,
                "traffic_source": ("ncu --set full capture of this kernel and shape, profiles/traffic.json "
                                   "(not measured in this run)") if traffic is not None else None,
                "kernel": f"{dom} projection (shrink + base GEMV/GEMM with fused expand)",
                "algorithmic_bytes": dom_bytes, "algorithmic_flops": dom_flops, "mean_us": dom_mean_us,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)" if bound == "hbm" else peak_src}
    layer_bytes = sum(b for b, _ in alg.values())
    layer_frac = layer_bytes / (ms_step * 1e-3) / 1e9 / hbm_peak

    # ---------------- sampled oracle check of this run's own output (cpu_baseline leg, N = 1) ----------------
    self_check = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        self_check = oracle_check_bench_output(bd, torch, layer, ids, ids_np)
        if not self_check["ok"]:
            log("bench self-check FAILED:", json.dumps(self_check))

    # ---------------- S-LoRA comparison (same box, same W) ----------------
    slora = None
    if not args.skip_slora:
        sl_layer, _ = build_layer(bd, torch, wl, "slora", n, rank, dev, share_w=layer)
        s_total, s_per, _ = time_layer(bd, torch, sl_layer, comm, ids, args.steps, args.warmup, not args.no_graph, barrier)
        s_total = reduce_max(s_total, dev)
        s_bytes = sum(b for b, _ in algorithmic(wl, "slora", n, ids_np).values())
        slora = {"ms_per_step": s_total / args.steps, "tokens_per_s": T / (s_total / args.steps * 1e-3),
                 "proj_us": dict(zip(names, s_per)), "ranks": wl.get("slora_ranks", wl["ranks"]),
                 "layer_hbm_frac": s_bytes / (s_total / args.steps * 1e-3) / 1e9 / hbm_peak,
                 "bd_speedup": (s_total / total_ms)}
        if comm is not None:
            slora["collectives"] = bd.bdlora_comm_stats(comm)
        for p in sl_layer:
            p.close()
        del sl_layer

    # ---------------- NFS-LoRA comparison (same box, same W) ----------------
    nfs = None
    if not args.skip_slora:
        nf_layer, _ = build_layer(bd, torch, wl, "nfs", n, rank, dev, share_w=layer)
        f_total, f_per, _ = time_layer(bd, torch, nf_layer, comm, ids, args.steps, args.warmup, not args.no_graph, barrier)
        f_total = reduce_max(f_total, dev)
        f_bytes = sum(b for b, _ in algorithmic(wl, "nfs", n, ids_np).values())
        nfs = {"ms_per_step": f_total / args.steps, "tokens_per_s": T / (f_total / args.steps * 1e-3),
               "proj_us": dict(zip(names, f_per)),
               "layer_hbm_frac": f_bytes / (f_total / args.steps * 1e-3) / 1e9 / hbm_peak,
               "bd_speedup": (f_total / total_ms)}
        for p in nf_layer:
            p.close()
        del nf_layer

    # ---------------- e2e through the public API with host buffers ----------------
    e2e_ms, h2d, d2h, census = time_e2e(bd, torch, layer, comm, ids_np, args.steps, args.warmup, barrier)
    e2e_ms = reduce_max(e2e_ms, dev)
    e2e = {"value": T / (e2e_ms / args.steps * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
           "graph_nodes": census, "graph_memcpy_nodes_expected": 2 * args.steps}
    collectives = bd.bdlora_comm_stats(comm) if comm is not None else None
    for p in layer:
        p.close()
    del layer
    torch.cuda.empty_cache()

    # ---------------- emulated TP shards on one GPU (N=1 only) ----------------
    tp_emulated = None
    if world == 1 and not args.skip_tp_emulation:
        tp_emulated = {}
        for tpn in (2, 4, 8):
            row = {}
            for sh in ("bd", "slora", "nfs"):
                em, _ = build_layer(bd, torch, wl, sh, tpn, 0, dev, seed=tpn)
                # device-local work only (no collectives on one GPU): BD row = partial; S-LoRA = phases
                tt, pp, _ = time_layer_local(bd, torch, em, ids, max(10, args.steps), args.warmup, tpn)
                row[sh] = {"us_per_layer": tt * 1e3, "proj_us": {nm: u for nm, u in zip(names, pp)},
                           "hbm_frac": sum(b for b, _ in algorithmic(wl, sh, tpn, ids_np).values()) / (tt * 1e-3) / 1e9 / hbm_peak}
                for p in em:
                    p.close()
                del em
                torch.cuda.empty_cache()
            tp_emulated[f"tp{tpn}"] = row

    # ---------------- whole decode step, batch-1 workloads ----------------
    decode_step = None
    if T == 1 and args.decode_layers > 0:
        L = args.decode_layers
        us = time_decode_step(bd, torch, wl, n, rank, dev, comm, max(3, args.steps // 10), args.warmup, L)
        decode_step = {"layers": L, "us_per_token": us, "tokens_per_s": 1e6 / us,
                       "note": "QKV->O->gate_up->down per layer chained through real inputs (attention / SiLU "
                               "placeholders), one CUDA graph, PDL; per output token at batch 1"}
        if world == 1 and not args.skip_tp_emulation:
            decode_step["tp_emulated_1gpu"] = {
                f"tp{tpn}": time_decode_step(bd, torch, wl, tpn, 0, dev, None, max(3, args.steps // 10), args.warmup,
                                             L, local_only=True) for tpn in (2, 4, 8)}

    cpu = None
    if rank == 0 and not args.skip_cpu:
        cpu = cpu_baseline(wl)

    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded torch.randn bf16; random-init factors)",
            "config": {"workload": wl["desc"] + f", TP={n}", "tp": n, "T": T, "ranks": wl["ranks"],
                       "resident_adapters": wl["n_adapters"], "sharding": "BD-LoRA",
                       "l2": f"inputs larger than L2: {reps} weight replica(s) rotated, "
                             f"{reps * layer_bytes / 1e6:.0f} MB per rotation >= 3 x 126 MB L2",
                       "cuda_graph": not args.no_graph, "parallelism": f"tp{n}",
                       "row_allreduce": ("fused peer-memory (bdlora_row_forward_fused)" if fused_ar else
                                         "ncclAllReduce bf16" if world > 1 else "none (N = 1)")},
            "layer_us": ms_step * 1e3, "proj_us": proj_us, "layer_hbm_frac": layer_frac,
            "layer_algorithmic_bytes": layer_bytes,
            "slora": slora, "nfs": nfs, "collectives": collectives, "tp_emulated_1gpu": tp_emulated,
            "roofline": roofline, "cpu_baseline": cpu, "self_check": self_check, "e2e": e2e, "decode_step": decode_step,
            "gpu_launches": launches * args.steps, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def time_decode_step(bd, torch, wl, n, rank, dev, comm, steps, warmup, layers, local_only=False):
    """the whole decode step: `layers` decoder layers, each QKV -> [attention
    placeholder] -> O -> gate_up -> [SiLU*up placeholder] -> down, chained through their REAL inputs (each
    projection reads the previous one's output) in one CUDA graph with programmatic dependent launch.
    Placeholders (the sharding method does not touch them): O reads the q slice of QKV's output,
    down reads the gate slice of gate_up's output (contiguous views at T = 1); no residual, norm or KV cache.
    Every layer has its own base weights and its own rank-r adapter (slot = layer in one pool per
    projection).  local_only: device-local work of rank 0 of an N-way TP group on one GPU (row layers as
    partials, no all-reduce).  Returns us per decode step (= per output token at batch 1)."""
    import synth

    T = wl["T"]
    if T != 1:
        return None
    projs = synth.arch_projections(wl["arch"])
    r = wl["ranks"][0]
    s = synth.rs_scale(16.0, r, n, "bd")
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321)
    pools, Ws, Ys, wss = [], [], [], []
    for p in projs:
        par = bd.COLUMN if p.parallel == "column" else bd.ROW
        pool = bd.bdlora_create_pool(par, bd.SHARD_BD, n, rank, p.d_in, p.d_out, layers, r, device=dev.index)
        for layer in range(layers):
            A, B = [], []
            for dj in p.d_out:
                if p.parallel == "column":
                    A.append((torch.randn(p.d_in, r, generator=gen, device=dev) / math.sqrt(p.d_in)).to(torch.bfloat16))
                    B.append((torch.randn(r // n, dj, generator=gen, device=dev) / (s * math.sqrt(r / n))).to(torch.bfloat16))
                else:
                    A.append((torch.randn(p.d_in, r // n, generator=gen, device=dev) / math.sqrt(p.d_in)).to(torch.bfloat16))
                    B.append((torch.randn(r, dj, generator=gen, device=dev) / (s * math.sqrt(r / n))).to(torch.bfloat16))
            bd.bdlora_load_adapter(pool, layer, r, s, A, B)
        pools.append(pool)
        Ws.append([(torch.randn(pool.m_loc, pool.k_loc, generator=gen, device=dev) / math.sqrt(p.d_in)).to(torch.bfloat16)
                   for _ in range(layers)])
        Ys.append(torch.empty(T, pool.m_loc, dtype=torch.bfloat16, device=dev))
        wss.append(bd.make_workspace(pool, T))
    ids = [torch.full((T,), layer, dtype=torch.int32, device=dev) for layer in range(layers)]
    x0 = torch.randn(T, pools[0].k_loc, generator=gen, device=dev).to(torch.bfloat16)
    q_cols, gate_cols = pools[1].k_loc, pools[3].k_loc

    def step(k):
        x = x0 if k == 0 else Ys[3]
        for layer in range(layers):
            i = ids[layer]
            bd.bdlora_column_forward(pools[0], x, Ws[0][layer], i, Ys[0], wss[0])
            xo = Ys[0][:, :q_cols]  # attention placeholder: the q slice
            if local_only or comm is None:
                bd.bdlora_row_partial(pools[1], xo, Ws[1][layer], i, Ys[1], wss[1])
            else:
                bd.bdlora_row_forward(pools[1], comm, xo, Ws[1][layer], i, Ys[1], wss[1])
            bd.bdlora_column_forward(pools[2], Ys[1], Ws[2][layer], i, Ys[2], wss[2])
            xd = Ys[2][:, :gate_cols]  # SiLU(gate) * up placeholder: the gate slice
            if local_only or comm is None:
                bd.bdlora_row_partial(pools[3], xd, Ws[3][layer], i, Ys[3], wss[3])
            else:
                bd.bdlora_row_forward(pools[3], comm, xd, Ws[3][layer], i, Ys[3], wss[3])
            x = Ys[3]

    for w in range(warmup):
        step(1)
    torch.cuda.synchronize()
    ms = graph_time(torch, step, steps, lambda: None)
    for pool in pools:
        pool.close()
    del Ws
    torch.cuda.empty_cache()
    return ms / steps * 1e3


def time_layer_local(bd, torch, layer, ids, steps, warmup, tpn):
    """Device-local per-rank work of one TP shard on one GPU (no collectives): BD / NFS column forward,
    BD / NFS row partial, S-LoRA shrink + base_expand.  Graph-captured; returns (ms/step, proj us list)."""
    dev = layer[0].X.device
    vbufs = {}

    def run(p, k):
        W = p.W[k % len(p.W)]
        if p.sharding == "bd":
            if p.proj.parallel == "column":
                bd.bdlora_column_forward(p.pool, p.X, W, ids, p.Y, p.ws)
            else:
                bd.bdlora_row_partial(p.pool, p.X, W, ids, p.Y, p.ws)
        elif p.sharding == "nfs":
            if p.proj.parallel == "column":
                bd.nfs_column_forward(p.pool, p.X, W, ids, p.Y, p.ws)
            else:
                bd.nfs_row_partial(p.pool, p.X, W, ids, p.Y, p.ws)
        else:
            if id(p) not in vbufs:
                T = p.X.shape[0]
                c = tpn if p.proj.parallel == "column" else 1
                vbufs[id(p)] = torch.zeros(c * bd.bdlora_v_elems(p.pool, T), dtype=torch.float32, device=dev)
            v = vbufs[id(p)]
            bd.bdlora_lora_shrink(p.pool, p.X, ids, v, p.ws)
            bd.bdlora_base_expand(p.pool, p.X, W, ids, v, p.Y, p.ws)

    for w in range(warmup):
        for p in layer:
            run(p, w)
    torch.cuda.synchronize()
    nobar = lambda: None  # noqa: E731
    total = graph_time(torch, lambda k: [run(p, k) for p in layer], steps, nobar)
    per = [graph_time(torch, lambda k, p=p: run(p, k), steps, nobar) / steps * 1e3 for p in layer]
    return total / steps, per, None


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="8b-decode-bs1-r16")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph")
    ap.add_argument("--skip-slora", action="store_true", help="skip the S-LoRA and NFS-LoRA comparison legs")
    ap.add_argument("--skip-tp-emulation", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-fused-ar", action="store_true",
                    help="N > 1: BD row layers all-reduce with NCCL instead of the fused peer-memory path")
    ap.add_argument("--decode-layers", type=int, default=None,
                    help="layers of the whole-decode-step leg (batch-1 workloads; default: the model's depth; 0 = off)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.decode_layers is None:
        args.decode_layers = {"llama-3.1-8b": 32}.get(wl["arch"], 0)  # 70B x 80 layers at TP1 would not fit beside the rest
    world, _, _ = dist_env()
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus={args.gpus}; TP degree follows WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())
