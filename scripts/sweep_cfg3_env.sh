#!/bin/bash
# Config 3 (R-MAT scale 22, H=4:8:8) under environment settings: wall and
# coarsen / initial / refine ms per map, J (must not change).  The graph is
# cached in /tmp between runs.  usage: SETS="A=1 B=2,C=3" scripts/sweep_cfg3_env.sh
export PYTHONPATH=.
for set in "" ${SETS}; do
  env $(echo "$set" | tr ',' ' ') timeout 600 python scripts/probe_configs.py --which rmat --reps ${REPS:-2} \
    --cache /tmp/rmat22.npz 2>/dev/null | python -c "
import sys, json
rows = [json.loads(l) for l in sys.stdin if l.startswith('{')]
print('[$set]', [(round(d['wall_ms']), d['ms_coarsen'], d['ms_initial'], d['ms_refine'], d['J']) for d in rows])"
done
