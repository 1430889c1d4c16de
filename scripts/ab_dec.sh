#!/bin/bash
# Same-box A/B of two library builds on the bench's default layer + TP-emulated layers.
# usage: put the other build at paper_2510_23346_b200/libbdlora_old.so
cd $GRAFT_REPO_ROOT
L=paper_2510_23346_b200
cp $L/libbdlora.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp $L/libbdlora_old.so $L/libbdlora.so; else cp /tmp/new.so $L/libbdlora.so; fi
  r=$(BDLORA_AB_OLD_LIB=1 timeout 300 python bench.py --steps 30 --warmup 5 --skip-cpu --skip-slora --decode-layers 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print(round(d['layer_us'],1), {k: round(v['bd']['us_per_layer'],1) for k,v in d['tp_emulated_1gpu'].items()})")
  echo "$v $r"
done > gpurun_out/ab_dec.txt
cp /tmp/new.so $L/libbdlora.so
