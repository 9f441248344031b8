#!/bin/bash
# Probe run: new GPU tests, per-launch refinement trace at 2^22, refinement
# launch list with warps-active / DRAM, config 3 keep vs strip.  Tag: $1
T=${1:-rX}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_envelope.py tests/test_gpu_isolated.py tests/test_gpu_runtime.py -m gpu -q -rfE > $O/tests_new_$T.log 2>&1; tail -3 $O/tests_new_$T.log
GIM_TRACE_REFINE=1 timeout 300 python scripts/ncu_target.py --mode step --logn 22 > /dev/null 2> $O/trace_refine_$T.txt; wc -l $O/trace_refine_$T.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size \
  --clock-control none --csv --log-file $O/launches_refine_$T.csv -k regex:k_refine \
  python scripts/ncu_target.py --mode step --logn 22 > /dev/null 2>&1; wc -l $O/launches_refine_$T.csv
PYTHONPATH=. timeout 900 python scripts/probe_configs.py --which rmat --rmat-scale 22 --reps 2 --isolated strip keep > $O/cfg3_$T.txt 2>&1; tail -5 $O/cfg3_$T.txt
