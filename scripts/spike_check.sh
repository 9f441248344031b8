PYTHONPATH=. python scripts/probe_im.py --logn 22 --oracle 0 --reps 6 --seeds 0 --no-host 2>&1 | python -c "
import sys,json
print([round(json.loads(l)['wall_s']*1e3,1) for l in sys.stdin if l.startswith('{')])"
nvidia-smi --query-gpu=clocks.sm --format=csv,noheader -lms 100 > /dev/null &
P=$!
PYTHONPATH=. python scripts/probe_im.py --logn 22 --oracle 0 --reps 6 --seeds 0 --no-host 2>&1 | python -c "
import sys,json
print('smi', [round(json.loads(l)['wall_s']*1e3,1) for l in sys.stdin if l.startswith('{')])"
kill $P
