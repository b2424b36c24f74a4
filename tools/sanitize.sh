#!/bin/bash
# compute-sanitizer over the small-shape GPU parity tests of every kernel
# family: the fused map+partition-reduce stream with its ticketed finisher
# tail (cooperative + PDL launches), the stand-alone finish / stage-2 / tree
# kernels, reduce_cl vector folds, pi, the TMA Sobel, the tcgen05 GEMMs and
# the word-start flags. Logs: gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
SEL_PARITY="fused_map_reduce or segment_reduce_bitexact or tree_reduce or many_short or isum_golden or fig3 or c1_pipeline or c2_small or pi_vs_oracle or sobel_golden or many_partitions or graph_step_matches"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 97 --target-processes all \
    python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "$SEL_PARITY" \
    tests/test_gpu_gemm.py::test_gemm_matches_oracle_small tests/test_gpu_gemm.py::test_gemm_f32_golden_tight \
    tests/test_wordcount.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
