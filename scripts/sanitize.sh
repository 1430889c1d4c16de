#!/bin/bash
# compute-sanitizer tier: memcheck, racecheck and synccheck over small GPU parity tests that
# reach every kernel family -- lean decode (T = 1 / 16, K-local LoRA, cluster DSMEM reduce), 64-token tiles,
# the multi-adapter shrink + tensor-core expand (lora 4), the v-precomputed expand, prefill tcgen05 tiles
# (route + shrink + GEMM), the fused row all-reduce over emulated peers, segments, Alg. 2 at N = 1.
# usage: scripts/sanitize.sh TAG   -> gpurun_out/sanitize_TAG_<tool>.txt
TAG=${1:-r2}
mkdir -p gpurun_out
TESTS=(
  "tests/test_gpu_parity.py::test_column_bd_tiny_config0"
  "tests/test_gpu_parity.py::test_segments_bit_exact"
  "tests/test_gpu_parity.py::test_integer_mode_bit_exact_decode"
  "tests/test_gpu_parity.py::test_prefill_token_tiles"
  "tests/test_gpu_parity.py::test_alg2_column_forward_gather"
  "tests/test_gpu_decode.py::test_decode_multi_token_multi_adapter"
  "tests/test_gpu_decode.py::test_decode_slice_straddling_tiles"
  "tests/test_gpu_decode.py::test_decode_bn64_integer_bit_exact"
  "tests/test_gpu_decode.py::test_decode_multi_adapter_integer_bit_exact"
  "tests/test_gpu_decode.py::test_decode_v_precomputed_mode"
  "tests/test_gpu_fused_ar.py::test_fused_row_allreduce_integer_bit_exact"
  "tests/test_gpu_paths.py::test_slora_entry_points_integer_bit_exact"
)
for tool in memcheck racecheck synccheck; do
  OUT=gpurun_out/sanitize_${TAG}_${tool}.txt
  echo "== compute-sanitizer --tool $tool" > $OUT
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  START=$(date +%s)
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest -q -p no:cacheprovider -x "${TESTS[@]}" >> $OUT 2>&1
  echo "exit $? wall $(( $(date +%s) - START )) s" >> $OUT
done
