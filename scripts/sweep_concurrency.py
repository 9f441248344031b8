"""Config 5 on one GPU: 64 mapping seeds of the rgg 2^22 instance with 1..6
concurrent maps (streams / host threads) -> aggregate edges/s per setting."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12196_b200 import device as D  # noqa: E402
from paper_2510_12196_b200.generators import gen_rgg  # noqa: E402
from paper_2510_12196_b200.replicas import DeviceRunner  # noqa: E402

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = gen_rgg(1 << logn, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
for conc in (1, 2, 3, 4, 6):
    r = DeviceRunner(dg, conc)
    r.warm()
    out = r.run(list(range(64)))
    wall = out["t_end"] - out["t_start"]
    print(json.dumps({"concurrency": conc, "maps": len(out["jobs"]), "wall_s": wall,
                      "edges_per_s": len(out["jobs"]) * g.m / wall,
                      "balanced": all(j["balanced"] for j in out["jobs"])}), flush=True)
