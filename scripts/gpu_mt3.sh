#!/bin/bash
# multi-adapter decode A/B: early vs late PDL trigger of the shrink; traces, tests, bench lines
TAG=${1:-mt}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_dec_${TAG}.txt
R="8,16,32,64,128"
for late in 0 1; do
  for k in 0 1 2 3; do BDLORA_SHRINK_LATE_TRIGGER=$late TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 $R 128 uniform >> gpurun_out/trace_${TAG}_late$late.txt 2>&1; done
  for n in 1 2; do BDLORA_SHRINK_LATE_TRIGGER=$late TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b 2 $n 64 $R 128 uniform >> gpurun_out/trace_${TAG}_late$late.txt 2>&1; done
done
timeout 300 python scripts/dec_micro.py 1280 8192 64 4 8192 1024 64 4 > gpurun_out/micro_${TAG}.txt 2>&1
for wl in 70b-multitenant 70b-decode-bs64-r32; do
  timeout 400 python bench.py --steps 20 --warmup 3 --workload $wl --skip-cpu --decode-layers 0 \
    > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
done
