#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over the small -m gpu
# parity cases (RMAT <= 14, hand-built graphs): every kernel of libseraph.so
# runs at least once (K1 all gates + hub chunks + source blocks, K3 push,
# tail loop, census/compaction, K8, streaming ring, device build/generator).
# Logs go to gpurun_out/sanitizer_<tool>.log; run under gpurun.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SAN=/usr/local/cuda/bin/compute-sanitizer
SEL="test_run_bfs_two_vertex or test_dense_pull_counts or test_weak_dormancy or test_metrics_partition \
or test_fixpoint_law_random or test_mode_independence or test_predictors_preserve or test_rmat_matrix_all_modes \
or test_streaming_matches_resident or test_pagerank_known_answers or test_pagerank_rmat_vs_oracle \
or test_sparse_pass_chains or test_pull_source_blocked or test_pagerank_source_blocked \
or test_frontier_queue or test_sssp_saturating or test_sssp_zero_weight or test_deferred_push \
or test_device_build_bit_exact or test_device_generate_graph or test_sharded_rounds_loopback_world \
or test_group_pagestream_run_multi_device or test_out_of_core_traversal_adjacency_budget \
or test_sharded_run_graph_and_device_built_shards or test_k2_device_reentry_loop \
or test_pagerank_rmat18_relative or test_k1_list_variant"
SEL_RACE="test_fixpoint_law_random or test_pagerank_known_answers or test_sparse_pass_chains \
or test_dense_pull_counts or test_pull_source_blocked or test_frontier_queue \
or test_pagerank_rmat_vs_oracle or test_k2_device_reentry_loop or test_pagerank_source_blocked or test_k1_list_variant"
for tool in memcheck racecheck synccheck; do
  extra=""
  sel="$SEL"
  [ "$tool" != memcheck ] && sel="$SEL_RACE"
  [ "$tool" = memcheck ] && extra="--leak-check no --padding 32"
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout "${SAN_TIMEOUT:-1500}" $SAN --tool $tool $extra --error-exitcode 17 \
      --target-processes all --print-limit 50 \
      python -m pytest tests/test_engine_gpu.py -q -x -p no:cacheprovider -k "$sel" \
      > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.log
  tail -3 gpurun_out/sanitizer_$tool.log
done
