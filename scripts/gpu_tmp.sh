bash scripts/gpu_round.sh r2e test bench
timeout 400 python bench.py --steps 20 --warmup 3 --workload 70b-decode-bs64-r32 --skip-cpu --decode-layers 0 > gpurun_out/bench_r2e_70b-decode-bs64-r32.json 2> gpurun_out/bench_r2e_bs64.err
