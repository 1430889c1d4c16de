#!/bin/bash
# Default bench line + the other workloads (parity-test configs, exploration only).
TAG=${1:-all}
mkdir -p gpurun_out
timeout 500 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
for w in 70b-decode-bs1-r32 70b-decode-bs64-r32 70b-multitenant 8b-prefill-1024-r64; do
  timeout 500 python bench.py --steps 20 --warmup 3 --workload $w --skip-cpu > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
done
