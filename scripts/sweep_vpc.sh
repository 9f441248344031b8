#!/bin/bash
# sweep the refinement grid sizing knobs on integrated_map (fan-out on)
for cv in ${CVS:-128 256 512}; do
  for gv in ${GVS:-32 128 512 1024}; do
    echo "CLUSTER_VPC=$cv COOP_VPC=$gv"
    GIM_CLUSTER_VPC=$cv GIM_COOP_VPC=$gv PYTHONPATH=. python scripts/probe_im.py --logn ${LOGNS:-20 22} --oracle 0 --reps 3 2>&1 \
      | grep '"rep": 2' | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); print(' logn',d['logn'],'wall',round(d['wall_s']*1e3,1),'coarsen',round(d['ms_coarsen'],1),'initial',round(d['ms_initial'],1),'refine',round(d['ms_refine'],1))"
  done
done
