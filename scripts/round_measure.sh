#!/bin/bash
# End-of-round measurement set (run under gpurun): GPU tests, bench lines
# (2^20 with cpu_baseline, 2^22), reference arm, ncu launch list of one map,
# ncu full captures of the level-0 refinement and of the level-0 coarsening
# kernels, DRAM traffic of the refinement launches; WITH_CONFIGS=1 adds
# configs 3 and 4.  Tag: $1 (e.g. r1g).
T=${1:-rX}
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests_$T.log 2>&1; tail -2 $O/tests_$T.log
timeout 400 python bench.py > $O/bench_$T.json 2> $O/bench_$T.err
timeout 300 python bench.py --logn 22 --no-cpu > $O/bench22_$T.json 2> $O/bench22_$T.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$T.csv python scripts/ncu_target.py --mode step --logn 20 > /dev/null 2>&1
for l in 20 22; do
  timeout 300 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_refine --clock-control none --csv --log-file $O/traffic_rgg${l}_$T.csv \
    python scripts/ncu_target.py --mode step --logn $l > /dev/null 2>&1
done
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_refine_fused -c 1 -o $O/refine0_$T python scripts/ncu_target.py --mode refine0 --logn 22 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"k_hem_pref_tpv|k_row_tpv|k_row_compact" -c 3 -o $O/coarsen0_$T python scripts/ncu_target.py --mode lp --logn 22 > /dev/null 2>&1
if [ -n "$WITH_CONFIGS" ]; then  # BASELINE configs 3 and 4 (R-MAT generation alone takes ~80 s)
  PYTHONPATH=. timeout 900 python scripts/probe_configs.py --which rmat grid3d --rmat-scale 22 --reps 2 \
    > $O/configs_$T.txt 2>&1
fi
ls $O | grep $T
