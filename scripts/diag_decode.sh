mkdir -p gpurun_out
python scripts/micro_gemm.py > gpurun_out/micro.txt 2>&1
for s in "4096 4096 1 fused" "6144 4096 1 fused" "28672 4096 1 fused" "4096 14336 1 fused"; do python scripts/trace_gemm.py $s; done > gpurun_out/trace.txt 2>&1
