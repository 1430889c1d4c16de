for rep in 1 2; do
for k in 0 1 2 3; do SHARDING=slora python scripts/proj_profile.py llama-3.1-70b $k 8 64 8,16,32,64,128 128 uniform >> gpurun_out/mt_time8.txt 2>&1; done
for k in 0 1 2 3; do python scripts/proj_profile.py llama-3.1-70b $k 8 64 8,16,32,64,128 128 uniform >> gpurun_out/mt_time8.txt 2>&1; done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "downward" 2>&1 | tail -2 > gpurun_out/pt_x8.txt
