#!/bin/bash
# Sweep the decode ring depth (BDLORA_STAGES) on the fused trace + the layer bench.
for ns in 2 3 4 6 10; do
  echo "== stages $ns"
  BDLORA_STAGES=$ns python scripts/trace_gemm.py 6144 4096 1 fused 2>/dev/null | sed -n '1p;5,9p;16,17p'
  BDLORA_STAGES=$ns python bench.py --steps 20 --warmup 5 --skip-tp-emulation --skip-cpu --skip-slora 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', round(d['layer_us'],1), {k: round(v,1) for k,v in d['proj_us'].items()})"
done
