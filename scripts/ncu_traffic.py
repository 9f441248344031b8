"""Per-launch DRAM traffic of the dominant kernel class from an ncu capture
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:k_refine_fused --csv` over one serialised map, ncu_target.py --mode
step): writes/updates profiles/ncu_traffic.json {class: {workload: {...}}}."""
import csv
import io
import json
import sys
from collections import defaultdict
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def main(path, cls, workload):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(dict)
    for r in rows:
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        per[r["ID"]][r["Metric Name"]] = v
    launches = [p for p in per.values() if "dram__bytes_read.sum" in p]
    tot = sum(p["dram__bytes_read.sum"] + p["dram__bytes_write.sum"] for p in launches)
    big = max(launches, key=lambda p: p.get("gpu__time_duration.sum", 0.0))
    out = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
    data = json.loads(out.read_text()) if out.exists() else {}
    data.setdefault(cls, {})[workload] = {
        "launches": len(launches),
        "dram_bytes_per_launch": tot / len(launches),
        "largest_launch_dram_bytes": big["dram__bytes_read.sum"] + big["dram__bytes_write.sum"],
        "largest_launch_ms_ncu": big.get("gpu__time_duration.sum"),
        "source": Path(path).name,
    }
    out.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data[cls][workload]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
