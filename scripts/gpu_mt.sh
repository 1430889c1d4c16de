#!/bin/bash
# multi-adapter decode diagnosis: decode tests, traced projections, ncu full of the shrink and the LM 3 GEMM
TAG=${1:-mt}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_dec_${TAG}.txt
R="8,16,32,64,128"
for k in 0 1 2 3; do TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 $R 128 uniform >> gpurun_out/trace_${TAG}.txt 2>&1; done
for n in 1 2; do TRACE=1 timeout 120 python scripts/proj_profile.py llama-3.1-70b 2 $n 64 $R 128 uniform >> gpurun_out/trace_${TAG}.txt 2>&1; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_shrink -s 3 -c 1 \
  -o gpurun_out/prof_shrink_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 0 8 64 $R 128 uniform 4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 3 -c 1 \
  -o gpurun_out/prof_lm3_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 0 8 64 $R 128 uniform 4 > /dev/null 2>&1
