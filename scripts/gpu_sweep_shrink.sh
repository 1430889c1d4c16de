#!/bin/bash
# shrink launch sweep: CTAs per SM x PDL trigger, 70B multi-tenant TP8 projections (graph-timed)
TAG=${1:-sw}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || exit 1
R="8,16,32,64,128"
for late in 0 1; do for per in 1 2 4 8; do
  echo "late=$late per_sm=$per" >> gpurun_out/sweep_${TAG}.txt
  for k in 0 1 2 3; do BDLORA_SHRINK_LATE_TRIGGER=$late BDLORA_SHRINK_CTAS_PER_SM=$per timeout 120 python scripts/proj_profile.py llama-3.1-70b $k 8 64 $R 128 uniform 2>&1 | sed 's/ranks=.*uniform://; s/last=.*//' >> gpurun_out/sweep_${TAG}.txt; done
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_shrink -s 3 -c 1 \
  -o gpurun_out/prof_shrink_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 1 8 64 $R 128 uniform 4 > /dev/null 2>&1
