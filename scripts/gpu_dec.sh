#!/bin/bash
# Decode-kernel iteration: its parity tests, the default bench line, and a TP-emulated per-projection table.
TAG=${1:-d}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/pytest_dec_${TAG}.txt
if grep -q " passed" gpurun_out/pytest_dec_${TAG}.txt && ! grep -q "failed\|error" gpurun_out/pytest_dec_${TAG}.txt; then
  timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
  if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
fi
