timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_lora_gemm_kernel -s 5 -c 1 \
  -o gpurun_out/prof_prefill_gateup_tp1_r2h -f python scripts/proj_profile.py llama-3.1-8b 2 1 1024 64 1 single 3 > gpurun_out/prof_pf.log 2>&1
