mkdir -p gpurun_out
timeout 400 python bench.py --steps 30 --warmup 5 --skip-cpu > gpurun_out/full_def.json 2>/dev/null
BDLORA_LOCAL=0 timeout 400 python bench.py --steps 30 --warmup 5 --skip-cpu > gpurun_out/full_l0.json 2>/dev/null
BDLORA_LOCAL_MAXKB=24 timeout 400 python bench.py --steps 30 --warmup 5 --skip-cpu > gpurun_out/full_l24.json 2>/dev/null
