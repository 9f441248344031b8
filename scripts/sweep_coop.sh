#!/bin/bash
# refinement grid sizing at the bench workload: device ms per map and the
# refine phase for several GIM_COOP_VPC (vertices per CTA of cooperative
# grids; fewer CTAs = cheaper barriers and less per-CTA O(k) work)
for gv in ${GVS:-128 256 512 1024 2048}; do
  GIM_COOP_VPC=$gv timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --replica-jobs 0 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph=d['step_phases_ms']['coarsen/initial/refine']
import statistics as S
print('COOP_VPC=$gv ms/map',round(d['ms_per_step'],2),'coarsen/initial/refine medians',[round(S.median(x[i] for x in ph),2) for i in range(3)], 'J ok', d['parity']['assignment_identical'])"
done
