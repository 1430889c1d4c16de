"""The bench's algorithmic byte / FLOP accounting (paper_2510_23346_b200/accounting.py, which feeds
roofline.achieved) pinned to the paper's closed forms held by the oracle (CPU only).

* Summed over the N devices, the per-device factor elements of BD-LoRA are the adapter's non-zeros
  ("# parameters" rows), those of S-LoRA the dense factor, and NFS-LoRA carries N copies of
  A_1 and B_2 ("N times more memory ... for A_1 and B_2").
* The per-device LoRA FLOPs of an MLP pair are the paper's "# operations" column, 2 S x (# parameters)
  per device."""
import pytest

from oracle import accounting as oacc
from paper_2510_23346_b200 import accounting as pacc

SHAPES = [(4096, 14336), (8192, 28672), (256, 512)]


@pytest.mark.parametrize("d_h,d_i", SHAPES)
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("r", [8, 16, 64])
def test_factor_elements_sum_to_paper_parameter_counts(d_h, d_i, n, r):
    col = sum(pacc.factor_elems("column", "bd", d_h, [d_i], n, r) for _ in range(n))
    row = sum(pacc.factor_elems("row", "bd", d_i, [d_h], n, r) for _ in range(n))
    assert col == oacc.params_bd_column(d_h, d_i, r, n)
    assert row == oacc.params_bd_row(d_i, d_h, r, n)
    assert sum(pacc.factor_elems("column", "slora", d_h, [d_i], n, r) for _ in range(n)) == oacc.params_dense(d_h, d_i, r)
    assert sum(pacc.factor_elems("row", "slora", d_i, [d_h], n, r) for _ in range(n)) == oacc.params_dense(d_i, d_h, r)
    # NFS: A_1 and B_2 replicated on every device, A_2 and B_1 sharded like the base weight
    nfs_col = sum(pacc.factor_elems("column", "nfs", d_h, [d_i], n, r) for _ in range(n))
    nfs_row = sum(pacc.factor_elems("row", "nfs", d_i, [d_h], n, r) for _ in range(n))
    assert nfs_col == oacc.params_dense(d_h, d_i, r) + (n - 1) * d_h * r
    assert nfs_row == oacc.params_dense(d_i, d_h, r) + (n - 1) * r * d_h


@pytest.mark.parametrize("d_h,d_i", SHAPES)
@pytest.mark.parametrize("n", [1, 2, 8])
@pytest.mark.parametrize("method", ["bd", "slora"])
def test_lora_flops_match_paper_operations_column(d_h, d_i, n, method):
    r, S = 16, 37
    toks = [r] * S
    base_col = 2 * S * d_h * (d_i // n)
    base_row = 2 * S * (d_i // n) * d_h
    lora = (pacc.proj_flops("column", method, d_h, [d_i], n, toks) - base_col) + \
        (pacc.proj_flops("row", method, d_i, [d_h], n, toks) - base_row)
    # S-LoRA: 2 S 2 (d_H + d_I) r / N; BD (at its own rank): 2 S 2 (d_H + d_I / N) r / N
    ref = oacc.mlp_lora_flops_per_device(S, d_h, d_i, n, r, method)
    assert lora == ref


def test_ids_and_activations_in_bytes():
    # bf16 weight shard + activations in/out + one adapter's shards + int32 ids
    b = pacc.proj_bytes("column", "bd", 4096, [4096, 1024, 1024], 1, 1, [16])
    assert b == 2 * (4096 * 6144 + 4096 + 6144 + 3 * 4096 * 16 + 16 * (4096 + 1024 + 1024)) + 4
