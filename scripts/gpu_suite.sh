#!/bin/bash
# the whole -m gpu suite with per-test durations, then the 64-token decode micro / bench lines
TAG=${1:-su}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
START=$(date +%s)
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 2>&1 | tail -60 > gpurun_out/pytest_all_${TAG}.txt
echo "suite wall $(( $(date +%s) - START )) s" >> gpurun_out/pytest_all_${TAG}.txt
timeout 300 python scripts/dec_micro.py 1280 8192 64 4 8192 1024 64 4 7168 8192 64 4 8192 3584 64 4 > gpurun_out/micro_${TAG}.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --workload 70b-decode-bs64-r32 --skip-cpu --decode-layers 0 \
  > gpurun_out/bench_${TAG}_bs64.json 2> gpurun_out/bench_${TAG}_bs64.err
