"""Multi-GPU collective paths (one process per GPU under torchrun): NCCL row all-reduce, the fused peer-memory
all-reduce, Alg. 2's all-gather, S-LoRA's extra collectives and NFS-LoRA's row, all against the fp64 oracle,
plus the collective call log (BD-LoRA issues only the base all-reduce: zero LoRA-tagged collectives, SURVEY
§8(d) step 9).  Skipped on a machine with fewer than 2 GPUs -- this environment's boxes have one; the
single-GPU tests emulate the same reductions (tests/test_gpu_fused_ar.py, tests/test_gpu_paths.py)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_collectives(n):
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs, found {_ngpu()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29561", os.path.join(ROOT, "scripts", "multi_gpu_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    bad = {k: v for k, v in out["checks"].items() if not v["ok"]}
    assert not bad, bad
    for k, v in out["checks"].items():
        if k.startswith("bd_row_fused"):
            assert v["peer_error"] == 0 and v["identical_on_all_ranks"], (k, v)
    st = out["comm_stats"]
    # the BD / NFS paths add no LoRA collective; the S-LoRA calls above account for exactly 2 per T
    assert st["lora_allgather_calls"] == 2 and st["lora_allreduce_calls"] == 2, st
