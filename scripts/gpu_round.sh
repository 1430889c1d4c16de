#!/bin/bash
# One GPU round trip: the whole -m gpu suite, the default bench line, every other workload, and the
# launch list of one eager layer step.  usage: scripts/gpu_round.sh TAG [what...]  what: test bench wl launches
TAG=${1:-r2}
shift
WHAT=${@:-test bench wl launches profile}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1
for w in $WHAT; do
  case $w in
    test)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_all_${TAG}.txt
      timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.txt 2>&1 ;;
    bench)
      timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err ;;
    wl)
      for wl in 70b-decode-bs1-r32 70b-decode-bs64-r32 70b-multitenant 70b-multitenant-zipf 70b-multitenant-distinct \
                8b-prefill-1024-r8 8b-prefill-1024-r64 8b-prefill-1024-r256 8b-prefill-8x128-r64 \
                8b-decode-bs1-r16-64resident 8b-decode-bs1-bd32-vs-slora16; do
        timeout 400 python bench.py --steps 20 --warmup 3 --workload $wl --skip-cpu --decode-layers 0 \
          > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
      done ;;
    launches)
      timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-graph --skip-slora \
        --skip-tp-emulation --skip-cpu --decode-layers 0 > /dev/null 2>&1 ;;
    profile)
      # ncu --set full of the dominant kernel (8B gate_up decode GEMM, T = 1) and of the 70B multi-tenant
      # TP8 gate_up (lora 4); launch lists of the 8B prefill TP8 chain and of the multi-tenant TP8 QKV chain
      timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 3 -c 1 \
        -o gpurun_out/prof_gateup_${TAG} -f python scripts/profile_one.py 28672 4096 1 16 fwd > /dev/null 2>&1
      timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 3 -c 1 \
        -o gpurun_out/prof_mt_gateup_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 2 8 64 8,16,32,64,128 128 uniform 4 > /dev/null 2>&1
      ONLY=expand SHARDING=slora timeout 300 ncu --set full --clock-control none --import-source on -k regex:dec_lora -s 3 -c 1 \
        -o gpurun_out/prof_slora_gateup_${TAG} -f python scripts/proj_profile.py llama-3.1-70b 2 8 64 8,16,32,64,128 128 uniform 4 > /dev/null 2>&1
      timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
        --clock-control none --csv --log-file gpurun_out/launches_prefill_${TAG}.csv \
        python scripts/proj_profile.py llama-3.1-8b 2 8 1024 64 1 single 3 > /dev/null 2>&1
      timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/launches_mt_${TAG}.csv python scripts/proj_profile.py llama-3.1-70b 0 8 64 8,16,32,64,128 128 uniform 3 > /dev/null 2>&1
      for k in 0 1 2 3; do timeout 120 python scripts/proj_profile.py llama-3.1-8b $k 8 1024 64 1 single >> gpurun_out/prefill_${TAG}.txt 2>&1; done ;;
  esac
done
