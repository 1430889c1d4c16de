#!/bin/bash
# A/B of the decode schedules on ONE box: bench layer step under env toggles, 2 repetitions each.
# usage: scripts/ab_layer.sh TAG "ENV1" "ENV2" ...   (each ENV is e.g. "BDLORA_CLUSTER=0 BDLORA_LOCAL=0")
TAG=$1; shift
mkdir -p gpurun_out
out=gpurun_out/ab_${TAG}.txt
: > $out
for rep in 1 2; do
  for e in "$@"; do
    line=$(env $e timeout 300 python bench.py --steps 30 --warmup 5 --skip-slora --skip-tp-emulation --skip-cpu ${BENCH_ARGS} 2>/dev/null | tail -1)
    python - "$e" "$line" >> $out <<'PY'
import json, sys
e, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(f"{e:45s} layer {d['layer_us']:6.1f}  " + "  ".join(f"{k} {v:5.1f}" for k, v in d['proj_us'].items()) + f"  e2e {d['e2e']['ms_per_step']*1e3:6.1f}")
except Exception as ex:
    print(e, "FAILED", ex, line[:200])
PY
  done
done
cat $out
