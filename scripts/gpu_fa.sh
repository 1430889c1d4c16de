#!/bin/bash
TAG=${1:-fa}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_ar.py tests/test_gpu_decode.py tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_fa_${TAG}.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fused_ar.py -m gpu -q -p no:cacheprovider -k "every_projection and 1-8 or 8b_bs1_every_projection and 3-2 or vs_oracle and 1-1-2 or v_precomputed or straddling" > gpurun_out/san_mem_dec_${TAG}.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider -k "every_projection" > gpurun_out/san_race_dec_${TAG}.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider -k "every_projection" > gpurun_out/san_sync_dec_${TAG}.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu --decode-layers 0 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
