#!/bin/bash
# ncu --set full of the lean decode kernel on one shape: python scripts/profile_one.py M K T rank fwd
TAG=${1:-p}; M=${2:-4096}; K=${3:-512}; R=${4:-2}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 2 -c 1 \
  -o gpurun_out/prof_dec_${TAG} -f python scripts/profile_one.py $M $K 1 $R fwd > gpurun_out/prof_dec_${TAG}.log 2>&1
