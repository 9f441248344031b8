#!/bin/bash
# Round-2 check on one B200: GPU tests, bench line (rgg 2^22), reference arm,
# sanitizer spot checks.  Tag: $1.
T=${1:-rX}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rfE -x > $O/tests_$T.log 2>&1; tail -3 $O/tests_$T.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_$T.json 2> $O/bench_$T.err; tail -c 600 $O/bench_$T.json; tail -3 $O/bench_$T.err
if [ -n "$WITH_REF" ]; then
  timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err
  tail -c 1500 $O/bench_ref_$T.json
fi
if [ -n "$WITH_SAN" ]; then
  CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 97"
  CUDA_MODULE_LOADING=EAGER timeout 900 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q \
    -k "ggg_golden or partitioner_golden or multisection_golden or integrated_map_small" > $O/san_race_$T.log 2>&1
  echo "racecheck rc=$?" >> $O/san_race_$T.log; tail -4 $O/san_race_$T.log
fi
