"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count and device time, total device time."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def main(path, top=30):
    rows = load(path)
    by = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
        name = r["Kernel Name"].split("(")[0].split("<")[0]
        by[name][0] += 1
        by[name][1] += v
        tot += v
    print(f"launches {sum(c for c, _ in by.values())}  device time {tot/1e3:.3f} ms")
    print(f"{'kernel':48s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k:48s} {c:8d} {t/1e3:9.3f} {t/tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
