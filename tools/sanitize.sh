#!/bin/bash
# compute-sanitizer over small configurations of the CUDA path (memcheck / racecheck /
# synccheck / initcheck).  Logs -> gpurun_out/sanitize_<tool>.log; summary lines to stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_parity.py::test_parity_small_blocks_many_events tests/test_gpu_evict.py::test_evict_parity tests/test_gpu_replica.py::test_replicated_layer_in_process tests/test_gpu_labels.py tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_budget.py::test_budgeted_commit_parity[22-250-3-80-0.3-True] tests/test_gpu_budget.py::test_budgeted_tiered_cascade_parity[31-budgets0-1-60-0.08-12] tests/test_gpu_prefetch.py::test_staged_host_pipeline_parity[mixed-True] tests/test_gpu_rule_groups.py"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
