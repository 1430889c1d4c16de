"""fp64 CPU oracle for BD-LoRA's tensor-parallel multi-adapter LoRA layer.

TEST INFRASTRUCTURE ONLY: importable by `tests/`, `__graft_entry__.smoke()` and
`bench.py` (cpu_baseline and --impl reference legs).  The product package
`paper_2510_23346_b200` never imports it; this package never imports the product.
See oracle/lora.py for the method and its citations, oracle/accounting.py for the
paper's closed-form counts.
"""
from . import accounting, lora  # noqa: F401
