#!/bin/bash
# compute-sanitizer over small instances of every kernel family (SURVEY §5:
# race detection / memory checking).  Reports under gpurun_out/sanitize_*.log
mkdir -p gpurun_out
SEL=${SEL:-"test_edge_matches_golden or (test_edge_fused_vs_oracle and (shape1 or shape2)) or test_edge_gaussian_variants or (test_edge_threshold_cases and inf) or (test_cava_matches_oracle and shape0) or (test_srad_matches_oracle and (shape0 or shape6)) or (test_euler_matches_oracle_bitwise and wh0) or test_euler_fast_path_fallback_bitwise or test_bfs_matches_reference_interpreter or test_bfs_deep_chain or (test_backprop_matches_oracle and 1000) or (test_matmul_tcgen05_within_fp32_bound and shape0) or test_matmul_identity_and_zero_k or test_euler_emulated_slabs"}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
