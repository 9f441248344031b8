#!/bin/bash
# Round-2 measurement set on one B200 (tag $1): GPU tests, smoke, bench lines
# (default = rgg 2^22 with cpu_baseline + config 5; config 2 at 2^20),
# reference arm, METIS loader timing.  ncu captures: scripts/r2_ncu.sh.
T=${1:-rX}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rfE > $O/tests_$T.log 2>&1; tail -2 $O/tests_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; tail -1 $O/smoke_$T.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_$T.json 2> $O/bench_$T.err; tail -c 300 $O/bench_$T.json; echo
timeout 600 python bench.py --logn 20 --steps 20 --warmup 5 --no-cpu --replica-jobs 0 > $O/bench20_$T.json 2> $O/bench20_$T.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err; tail -c 300 $O/bench_ref_$T.json; echo
timeout 1200 python scripts/bench_metis.py --logn 22 > $O/metis_$T.json 2> $O/metis_$T.err; cat $O/metis_$T.json
