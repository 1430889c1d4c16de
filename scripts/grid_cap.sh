# per-SM streaming bandwidth vs number of CTAs (BDLORA_GRID_CAP), gate_up and O shapes, decode T=1
mkdir -p gpurun_out
for c in 148 112 74 48 37; do
  BDLORA_GRID_CAP=$c python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import scripts.micro_gemm as m
for M, K in [(28672, 4096), (4096, 4096)]:
    r = m.run(M, K, 1, lora=False)
    print(os.environ["BDLORA_GRID_CAP"], M, K, "us_fwd_nolora %.1f" % r["us_fwd_nolora"], "GB/s %.0f" % (M*K*2/r["us_fwd_nolora"]/1e3), flush=True)
PY
done > gpurun_out/grid_cap.txt 2>&1
