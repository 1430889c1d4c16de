#!/bin/bash
# Sweep a decode-kernel knob over the bench's layer (TP1 + TP-emulated); one JSON summary line per value.
# usage: scripts/dec_sweep.sh TAG VAR v1 v2 ...
TAG=$1; VAR=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  env $VAR=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu --skip-slora --decode-layers 0 ${BENCH_ARGS} 2>/dev/null | tail -1 | \
    python -c "
import json,sys
d=json.loads(sys.stdin.read())
row={'$VAR':'$v','tp1':round(d['layer_us'],1),'proj':{k:round(x,1) for k,x in d['proj_us'].items()}}
for k,x in (d.get('tp_emulated_1gpu') or {}).items(): row[k]=(round(x['bd']['us_per_layer'],1),{p:round(u,1) for p,u in x['bd']['proj_us'].items()})
print(json.dumps(row))" >> gpurun_out/sweep_${TAG}.txt
done
