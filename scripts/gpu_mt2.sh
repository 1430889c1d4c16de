#!/bin/bash
# multi-adapter decode: decode tests, traced projections (TP8 / TP2 / TP1), launch list, bench lines
TAG=${1:-mt}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_dec_${TAG}.txt
R="8,16,32,64,128"
for k in 0 1 2 3; do TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 $R 128 uniform >> gpurun_out/trace_${TAG}.txt 2>&1; done
for n in 1 2; do TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b 2 $n 64 $R 128 uniform >> gpurun_out/trace_${TAG}.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mt_${TAG}.csv python scripts/proj_profile.py llama-3.1-70b 0 8 64 $R 128 uniform 4 > /dev/null 2>&1
for wl in 70b-multitenant 70b-decode-bs64-r32; do
  timeout 400 python bench.py --steps 20 --warmup 3 --workload $wl --skip-cpu --decode-layers 0 \
    > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
done
