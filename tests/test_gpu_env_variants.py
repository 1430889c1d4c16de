"""The schedule knobs of the GEMM (read once per process from the environment) change only scheduling,
never values: re-run a parity subset against the fp64 oracle in a subprocess under each alternative
schedule -- global split-K fix-up instead of the cluster/DSMEM reduce, no cluster shrinking, stream-K
over every SM, the single-kernel forward at T = 64 (grid-wide shrink + tensor-core expand), the
CUDA-core expand, no K-local LoRA."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# decode (fused, split-K/cluster, stream-K), T = 64 multi-adapter, prefill token tiles, exact integer mode
SUBSET = ("decode_lora_schedules or integer_mode_bit_exact_decode or integer_mode_bit_exact_row or multitenant "
          "or prefill_token_tiles or full_size_bench")

VARIANTS = {
    "global_fixup": {"BDLORA_CLUSTER": "0"},
    "no_cluster_shrink": {"BDLORA_CLUSTER_SHRINK": "0"},
    "streamk_all_sms": {"BDLORA_STREAMK_CTAS": "148"},
    "fused_t64": {"BDLORA_FUSED_MAX_T": "64"},
    "cuda_core_expand": {"BDLORA_TC_EXPAND": "0"},
    "no_k_local": {"BDLORA_LOCAL": "0"},
    "single_kernel_decode_forward": {"BDLORA_DECODE": "0"},  # the round-1 decode path instead of the lean kernel
}

# the lean decode kernel's own knobs: a subset of tests/test_gpu_decode.py that covers every split / reduction
# style (whole tiles, cluster DSMEM, global fix-up, stream-K), both token-tile widths and every LoRA mode
DEC_SUBSET = ("(test_decode_8b_bs1_every_projection and (8-1 or 1-2 or 2-0)) or "
              "(test_decode_integer_bit_exact and (5-8 or 16-2)) or "
              "(test_decode_bn64_one_adapter and (0-8-64 or 2-8-64 or 0-1-64)) or "
              "(test_decode_bn64_streamk_slices and True) or (test_decode_multi_adapter_vs_oracle and 17) or "
              "test_decode_multi_adapter_integer_bit_exact or test_decode_v_precomputed_mode")
DEC_VARIANTS = {
    "dec_streamk_all_sms": {"BDLORA_DEC_CTAS": "148"},
    "dec_two_stages": {"BDLORA_DEC_STAGES": "2"},
    "dec_min_4_kblocks": {"BDLORA_DEC_MINKB": "4"},
    "dec_grid_37": {"BDLORA_DEC_CTAS": "37"},
    "dec_no_cluster_global_fixup": {"BDLORA_DEC_CLUSTER": "0"},
    "dec_cluster_max_8": {"BDLORA_DEC_CLUSTER": "8"},
    "dec_cuda_core_shrink": {"BDLORA_DEC_TC_SHRINK": "0"},
}


@pytest.mark.parametrize("name", sorted(DEC_VARIANTS))
def test_decode_kernel_under_schedule_variant(name):
    env = dict(os.environ, **DEC_VARIANTS[name])
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_decode.py"), "-m", "gpu",
                        "-x", "-q", "-k", DEC_SUBSET, "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-15:])
    assert r.returncode == 0, f"{name} {DEC_VARIANTS[name]}:\n{tail}"
    assert " passed" in tail, tail


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_parity_under_schedule_variant(name):
    env = dict(os.environ, **VARIANTS[name])
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-x", "-q", "-k", SUBSET, "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-15:])
    assert r.returncode == 0, f"{name} {VARIANTS[name]}:\n{tail}"
    assert " passed" in tail, tail
