#!/bin/bash
# Profiles committed under profiles/: (1) the launch list of one eager layer step of the bench workload,
# (2) ncu --set full of the dominant kernel (gate_up's fused decode GEMM) and of the O projection's.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-graph --skip-slora \
  --skip-tp-emulation --skip-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_lora_gemm -s 3 -c 1 \
  -o gpurun_out/prof_gateup_${TAG} -f python scripts/profile_one.py 28672 4096 1 16 fwd > gpurun_out/prof_gateup_${TAG}.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_lora_gemm -s 3 -c 1 \
  -o gpurun_out/prof_o_${TAG} -f python scripts/profile_one.py 4096 4096 1 16 fwd > gpurun_out/prof_o_${TAG}.log 2>&1
