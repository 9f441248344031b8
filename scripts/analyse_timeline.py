"""Analyse a chrome trace from probe_timeline.py: per time window, GPU busy
(union of kernel intervals), kernel count, host runtime-API time."""
import json
import sys
from collections import defaultdict


def union_len(iv):
    iv.sort()
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if ce is None or s > ce:
            if ce is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if ce is not None:
        tot += ce - cs
    return tot


def main(path, nwin=20):
    tr = json.load(open(path))
    ev = [e for e in tr["traceEvents"] if e.get("ph") == "X"]
    ker = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    rt = [e for e in ev if e.get("cat") == "cuda_runtime"]
    t0 = min(e["ts"] for e in ker)
    t1 = max(e["ts"] + e["dur"] for e in ker)
    W = (t1 - t0) / nwin
    print(f"span {(t1 - t0) / 1e3:.2f} ms, kernels {len(ker)}, runtime calls {len(rt)}")
    names = defaultdict(float)
    for i in range(nwin):
        a, b = t0 + i * W, t0 + (i + 1) * W
        iv = [(max(a, e["ts"]), min(b, e["ts"] + e["dur"])) for e in ker
              if e["ts"] < b and e["ts"] + e["dur"] > a]
        busy = union_len(iv)
        nk = sum(1 for e in ker if a <= e["ts"] < b)
        top = defaultdict(float)
        for e in ker:
            if e["ts"] < b and e["ts"] + e["dur"] > a:
                top[e["name"].split("(")[0].split("<")[0][-28:]] += min(b, e["ts"] + e["dur"]) - max(a, e["ts"])
        t3 = sorted(top.items(), key=lambda kv: -kv[1])[:3]
        print(f"[{(a - t0) / 1e3:7.2f} ms] busy {busy / W:5.1%} kernels {nk:5d}  " +
              "  ".join(f"{k}:{v / 1e3:.2f}" for k, v in t3))
    for e in ker:
        names[e["name"].split("(")[0][-40:]] += e["dur"]
    print("device time by kernel (ms, summed over streams):")
    for k, v in sorted(names.items(), key=lambda kv: -kv[1])[:15]:
        print(f"  {k:40s} {v / 1e3:8.3f}")
    by = defaultdict(lambda: [0, 0.0])
    for e in rt:
        by[e["name"]][0] += 1
        by[e["name"]][1] += e["dur"]
    print("runtime API (count, ms summed over threads):")
    for k, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:10]:
        print(f"  {k:30s} {c:6d} {t / 1e3:8.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
