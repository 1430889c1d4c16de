#!/bin/bash
# T = 17..64 decode diagnosis: 70B TP8 projection shapes (column-pool emulation, r/N = 4) at T = 16 / 64,
# with and without LoRA; launch list; ncu --set full of the T = 64 QKV launch.
TAG=${1:-d64}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1
timeout 300 python scripts/dec_micro.py 1280 8192 64 4 1280 8192 16 4 8192 1024 64 4 7168 8192 64 4 8192 3584 64 4 \
  > gpurun_out/micro_${TAG}.txt 2>&1
NOLORA=1 timeout 300 python scripts/dec_micro.py 1280 8192 64 4 8192 1024 64 4 7168 8192 64 4 \
  > gpurun_out/micro_nolora_${TAG}.txt 2>&1
for k in 0 1 2 3; do timeout 120 python scripts/profile_mt.py $k 8 64 >> gpurun_out/mt_${TAG}.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mt_${TAG}.csv python scripts/profile_mt.py 0 8 64 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 5 -c 1 \
  -o gpurun_out/prof_qkv64_${TAG} -f python scripts/dec_micro.py 1280 8192 64 4 > gpurun_out/prof_qkv64_${TAG}.log 2>&1
