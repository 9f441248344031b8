"""Run the deep-hierarchy envelope cases one by one (CUDA_LAUNCH_BLOCKING=1
recommended) and report the first failing call."""
import sys
import traceback
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12196_b200 import integrated_map  # noqa: E402
from paper_2510_12196_b200.generators import HostGraph  # noqa: E402

z = np.load(Path(__file__).resolve().parents[1] / "tests/golden/scale_envelope.npz")


class T:
    pass


for i in range(int(z["count"])):
    if str(z[f"{i}/kind"]) != "deep":
        continue
    g = HostGraph(z[f"{i}/offsets"], z[f"{i}/targets"], z[f"{i}/weights"], z[f"{i}/vweights"])
    t = T()
    t.hierarchy = tuple(int(x) for x in z[f"{i}/hierarchy"])
    t.distances = tuple(int(x) for x in z[f"{i}/distances"])
    try:
        m = integrated_map(g, t, 0.03, 0, coarsest_factor=int(z[f"{i}/coarsest_factor"]))
        print(i, "ok", np.array_equal(m.assignment, z[f"{i}/assignment"]), flush=True)
    except Exception:  # noqa: BLE001
        print(i, "FAILED", t.hierarchy, flush=True)
        traceback.print_exc()
