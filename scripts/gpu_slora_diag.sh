#!/bin/bash
# S-LoRA multi-tenant TP8 expand diagnosis: timings + launch list + ncu --set full of the row expand (lora 4)
TAG=${1:-sd}
mkdir -p gpurun_out
for k in 0 1 2 3; do
  SHARDING=slora timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 8,16,32,64,128 128 uniform >> gpurun_out/slora_${TAG}.txt 2>&1
  timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 8,16,32,64,128 128 uniform >> gpurun_out/slora_${TAG}.txt 2>&1
done
SHARDING=slora timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_slora_o_${TAG}.csv python scripts/proj_profile.py llama-3.1-70b 1 8 64 8,16,32,64,128 128 uniform 3 > /dev/null 2>&1
SHARDING=slora timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 3 -c 1 \
  -o gpurun_out/prof_slora_o_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 1 8 64 8,16,32,64,128 128 uniform 4 > /dev/null 2>&1
