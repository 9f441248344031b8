#!/bin/bash
# A/B of an environment knob on the bench workload: "VAR=value" settings in $SETS
for set in "" ${SETS}; do
  env $set timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --replica-jobs 0 2>/dev/null | python -c "
import sys,json,statistics as S
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph=d['step_phases_ms']['coarsen/initial/refine']
print('[$set] ms/map',round(d['ms_per_step'],2),'median coarsen/initial/refine',[round(S.median(x[i] for x in ph),2) for i in range(3)],'parity',d['parity']['assignment_identical'])"
done
