bash scripts/gpu_round.sh r2f test bench
