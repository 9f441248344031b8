"""Initial-phase breakdown at the bench workload: runs two maps (warm-up, then
seed 0) with GIM_TRACE_MS set by the caller; prints the stats' phase split."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_12196_b200 import device as D  # noqa: E402
from paper_2510_12196_b200.generators import gen_rgg  # noqa: E402

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = gen_rgg(1 << logn, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
for s in (1, 0):
    print(f"==== map seed {s}", file=sys.stderr, flush=True)
    _, _, st = D.integrated_map_device(dg, (4, 8, 6), (1, 10, 100), 0.03, s)
    torch.cuda.synchronize()
    print(f"seed {s}: coarsen {st['ms_coarsen']:.2f} initial {st['ms_initial']:.2f} "
          f"refine {st['ms_refine']:.2f} ms", file=sys.stderr, flush=True)
