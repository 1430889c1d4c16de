#!/bin/bash
# decode + prefill parity, 64-token micro, prefill / decode bench lines
TAG=${1:-it2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_prefill.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_${TAG}.txt
timeout 300 python scripts/dec_micro.py 1280 8192 64 4 8192 1024 64 4 > gpurun_out/micro_${TAG}.txt 2>&1
for k in 0 1 2 3; do timeout 120 python scripts/proj_profile.py llama-3.1-8b $k 8 1024 64 1 single >> gpurun_out/prefill_${TAG}.txt 2>&1; done
for wl in 8b-prefill-1024-r64 8b-prefill-8x128-r64 70b-decode-bs64-r32 70b-multitenant; do
  timeout 400 python bench.py --steps 20 --warmup 3 --workload $wl --skip-cpu --decode-layers 0 \
    > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
done
