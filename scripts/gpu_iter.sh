#!/bin/bash
# Iteration round trip: build, the decode GPU tests (+ the variant test), T = 64 micro timings, multi-tenant
# per-projection timings, and bench lines of the T = 64 workloads.  usage: scripts/gpu_iter.sh TAG [what...]
TAG=${1:-it}
shift
WHAT=${@:-test micro bench}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || { cat gpurun_out/build_${TAG}.txt; exit 1; }
for w in $WHAT; do
  case $w in
    test)
      timeout 900 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_dec_${TAG}.txt ;;
    variants)
      timeout 900 python -m pytest tests/test_gpu_env_variants.py -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_var_${TAG}.txt ;;
    all)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_all_${TAG}.txt ;;
    micro)
      timeout 300 python scripts/dec_micro.py 1280 8192 64 4 8192 1024 64 4 7168 8192 64 4 8192 3584 64 4 > gpurun_out/micro_${TAG}.txt 2>&1
      for k in 0 1 2 3; do timeout 120 python scripts/profile_mt.py $k 8 64 >> gpurun_out/mt_${TAG}.txt 2>&1; done ;;
    bench)
      for wl in 70b-decode-bs64-r32 70b-multitenant; do
        timeout 400 python bench.py --steps 20 --warmup 3 --workload $wl --skip-cpu --decode-layers 0 \
          > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
      done ;;
    launches)
      timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/launches_mt_${TAG}.csv python scripts/profile_mt.py 0 8 64 > /dev/null 2>&1 ;;
  esac
done
