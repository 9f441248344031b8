#!/bin/bash
# run probe_im (fan-out on) under several environment settings: VAR=vals
# usage: ENVS="GIM_SMEM_MAXN=0 GIM_SMEM_MAXN=4096" LOGNS="20 22" bash scripts/sweep_env.sh
for e in ${ENVS}; do
  echo "$e"
  env $e PYTHONPATH=. python scripts/probe_im.py --logn ${LOGNS:-20 22} --oracle 0 --reps 3 --no-host 2>&1 \
    | grep '"rep": 2' | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); print(' logn',d['logn'],'wall',round(d['wall_s']*1e3,1),'coarsen',round(d['ms_coarsen'],1),'initial',round(d['ms_initial'],1),'refine',round(d['ms_refine'],1))"
done
