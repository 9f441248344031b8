#!/bin/bash
# compute-sanitizer over the GPU parity suite (run under gpurun; one GPU).
# memcheck: every -m gpu unit + pipeline test at golden sizes; racecheck /
# synccheck (shared-memory hazards, barrier misuse): the unit goldens and the
# small integrated_map / multisection goldens (racecheck is ~100x slower).
# Tag: $1.  Logs: gpurun_out/sanitize_<tool>_<tag>.log
T=${1:-rX}
O=gpurun_out
mkdir -p $O
CS="compute-sanitizer --target-processes all --print-limit 200 --error-exitcode 97"
export CUDA_MODULE_LOADING=EAGER  # lazy loading reports a benign cuKernelGetFunction API error
UNITS="total_cost or block_weights or hem_rounds or match_coarse or level_stack or contract_matches or conn_golden or lp_golden or rebalance_golden or apply_moves or refine_golden or ggg_golden or partitioner_golden or multisection_golden or integrated_map_small"
timeout 2400 $CS --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py \
  -m gpu -q -p no:randomly > $O/sanitize_memcheck_$T.log 2>&1; echo "memcheck rc=$?" >> $O/sanitize_memcheck_$T.log
for tool in racecheck synccheck; do
  timeout 1500 $CS --tool $tool python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$UNITS" \
    > $O/sanitize_${tool}_$T.log 2>&1; echo "$tool rc=$?" >> $O/sanitize_${tool}_$T.log
done
tail -3 $O/sanitize_*_$T.log
