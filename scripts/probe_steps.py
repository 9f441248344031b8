"""The bench's timed loop with host timers beside the events (GIM_TRACE_MS=1
adds the library's own host split): where does an outlier step's time go?"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12196_b200 import device as D  # noqa: E402
from paper_2510_12196_b200.generators import gen_rgg  # noqa: E402

H, DIST = (4, 8, 6), (1, 10, 100)
g = gen_rgg(1 << 22, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for w in range(3):
    D.integrated_map_device(dg, H, DIST, 0.03, 10**6 + w)
torch.cuda.synchronize()
for step in range(6):
    flush.fill_(step & 0xff)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    t0 = time.perf_counter()
    _, _, st = D.integrated_map_device(dg, H, DIST, 0.03, step)
    t1 = time.perf_counter()
    b.record(s)
    b.synchronize()
    print(f"step {step}: events {a.elapsed_time(b):.2f} ms host call {1e3 * (t1 - t0):.2f} ms "
          f"ms_total {st['ms_total']:.2f}", file=sys.stderr, flush=True)
