#!/bin/bash
# ncu evidence for the round-2 bench line (one GPU; never under the timed
# bench): launch list of one 2^22 map, DRAM traffic of the refinement
# launches at 2^22 / 2^20 (-> profiles/ncu_traffic.json), full-set captures
# of the level-0 refinement and the level-0 coarsening kernels exported as CSV.
T=${1:-rX}
O=gpurun_out
mkdir -p $O
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$T.csv python scripts/ncu_target.py --mode step --logn 22 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_$T.csv > $O/launch_summary_$T.txt 2>/dev/null; head -12 $O/launch_summary_$T.txt
for l in 22 20; do
  timeout 400 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_refine_fused --clock-control none --csv --log-file $O/traffic_rgg${l}_$T.csv \
    python scripts/ncu_target.py --mode step --logn $l > /dev/null 2>&1
  python scripts/ncu_traffic.py $O/traffic_rgg${l}_$T.csv lp_eval rgg$l
done
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_refine_fused -c 1 -o $O/refine0_$T python scripts/ncu_target.py --mode refine0 --logn 22 > /dev/null 2>&1
ncu -i $O/refine0_$T.ncu-rep --page raw --csv > $O/ncu_refine0_rgg22_$T.csv 2>/dev/null; rm -f $O/refine0_$T.ncu-rep
timeout 600 ncu --profile-from-start off --set full --clock-control none \
  -k regex:"k_hem_pref_tpv|k_row_warp|k_row_compact" -c 3 -o $O/coarsen0_$T python scripts/ncu_target.py --mode step --logn 22 > /dev/null 2>&1
ncu -i $O/coarsen0_$T.ncu-rep --page raw --csv > $O/ncu_coarsen0_rgg22_$T.csv 2>/dev/null; rm -f $O/coarsen0_$T.ncu-rep
ls -la $O | grep $T
