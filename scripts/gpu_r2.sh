#!/bin/bash
# Round-2 GPU round trip: new parity tests first (no -x: see every failure), then the whole -m gpu suite,
# a default bench line, and compute-sanitizer on small configs.
# usage: scripts/gpu_r2.sh TAG [what...]   what: new all bench san
TAG=${1:-r2}
shift
WHAT=${@:-new all bench san}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
for w in $WHAT; do
  case $w in
    new)
      timeout 900 python -m pytest tests/test_gpu_parity_prefill.py tests/test_gpu_paths.py -m gpu -q \
        -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest_new_${TAG}.txt ;;
    all)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest_all_${TAG}.txt ;;
    bench)
      timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err ;;
    san)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 600 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py smoke \
          > gpurun_out/san_${tool}_smoke_${TAG}.txt 2>&1
      done
      timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q \
        -p no:cacheprovider -k "decode_lora_schedules and (0-1-1 or 3-8-12) or multitenant or prefill_token_tiles" \
        > gpurun_out/san_memcheck_tests_${TAG}.txt 2>&1
      timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q \
        -p no:cacheprovider -k "tiny_config0 or integer_mode_bit_exact_decode" \
        > gpurun_out/san_racecheck_tests_${TAG}.txt 2>&1 ;;
  esac
done
