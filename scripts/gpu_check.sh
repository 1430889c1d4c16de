#!/bin/bash
# One GPU round-trip: parity tests, a bench line, and an ncu launch list (eager, serialized).
# usage: scripts/gpu_check.sh TAG [pytest-args]
TAG=${1:-run}
shift
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -15 | tee gpurun_out/pytest_${TAG}.txt
fi
timeout 400 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -3 gpurun_out/bench_${TAG}.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-graph --skip-slora \
    --skip-tp-emulation --skip-cpu ${BENCH_ARGS} > /dev/null 2>&1
fi
