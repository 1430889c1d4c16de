#!/bin/bash
# Quick GPU iteration: selected parity tests, the decode micro-benchmark, a per-CTA trace.
# usage: scripts/gpu_quick.sh TAG "pytest -k expr"
TAG=${1:-q}
K=${2:-decode_lora or integer_mode or full_size}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -15 > gpurun_out/pytest_${TAG}.txt
timeout 300 python scripts/micro_gemm.py > gpurun_out/micro_${TAG}.txt 2>&1
for s in "4096 4096 1 fused" "28672 4096 1 fused"; do timeout 60 python scripts/trace_gemm.py $s; done > gpurun_out/trace_${TAG}.txt 2>&1
